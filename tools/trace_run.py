"""Per-CTA timeline of one decode layer (globaltimer stamps, see shadowkv_trace_buffer).

python tools/trace_run.py [--config c2] [--layers 4]  -> prints phase statistics (us, relative to
the score kernel's first CTA) for score / select / sparse-attn CTAs of the last traced layer."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace, binding as bd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--raw-epi", action="store_true", help="score events 8-11 hold clock64 deltas")
ap.add_argument("--slots", type=int, default=1, help="trace this many consecutive layers (steady state)")
ap.add_argument("--vc-rho", type=float, default=None, help="value cache on, queries drifting with this rho")
ap.add_argument("--q-len", type=int, default=1, help="s_q query tokens per call")
args = ap.parse_args()
args.layers = max(args.layers, args.slots)
os.environ["SKV_TRACE_SLOTS"] = str(args.slots)
cfg = synth.CONFIGS[args.config]
shape = Shape.from_config(cfg, steps=64, q_len=args.q_len)
inv, rot, il = synth.rope_table(cfg)
rope = RopeTable(inv, rot, il)
ws = alloc_workspace(shape)
states = []
for l in range(args.layers):
    inp = synth.gen_layer(cfg, 99, layer=l, device="cuda")
    st = LayerState(shape, value_cache=args.vc_rho is not None)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    st.build(rope.struct, ws)
    states.append(st)
out = torch.empty(cfg.batch, cfg.n_q_heads, args.q_len, 128, dtype=torch.bfloat16, device="cuda")
SLOT = 4 * 4096 * 16
tr = torch.zeros(args.slots * SLOT, dtype=torch.int64, device="cuda")
first = args.layers - args.slots
sis = [[synth.gen_step(cfg, 99, l, step, device="cuda") for l in range(args.layers)] for step in range(6)]
if args.q_len > 1:
    for step in range(6):
        for l in range(args.layers):
            si = sis[step][l]
            sis[step][l] = {n: si[n].unsqueeze(2).repeat(1, 1, args.q_len, 1).contiguous() for n in si}
if args.vc_rho is not None:
    for l in range(args.layers):
        qd = synth.gen_q_drift(cfg, 99, l, 6, args.vc_rho, device="cuda")
        for step in range(6):
            sis[step][l]["q"] = qd[step]
for step in range(6):
    for l, st in enumerate(states):
        si = sis[step][l]
        if step == 5 and l == first:
            torch.cuda.synchronize()
            tr.zero_()
            bd.shadowkv_trace_buffer(tr)
        st.decode(rope.struct, si["q"], si["k_new"], si["v_new"], step * args.q_len, out, ws)
    if step == 5:
        torch.cuda.synchronize()
        bd.shadowkv_trace_buffer(None)
T = tr.view(args.slots, 4, 4096, 16).cpu().numpy().astype(np.float64)
if args.vc_rho is not None:
    st_ = states[-1].cache_stats()
    print(f"value cache: last-step hit rate {st_[..., 2].sum().item() / (cfg.batch * cfg.n_kv_heads * cfg.budget):.3f}")
g0 = T[0, 0][T[0, 0][:, 0] > 0][:, 0].min()
if args.slots > 1:
    print("== per-layer milestones (us from the first traced layer's score start)")
    print("   layer  score_start pdl_rel  score_end  sel_start  pub(cand)  first_issue  p50_issue  last_V_in  merge_end  last_sparse_done")
    for sl in range(args.slots):
        t = T[sl]
        def col(k, e, f):
            c = t[k][:, e]; c = c[c > 0]
            return f(c - g0) / 1e3 if len(c) else float("nan")
        print(f"   {sl:5d}  {col(0, 0, np.min):10.2f} {col(0, 15, np.min):8.2f} {col(0, 1, np.max):9.2f} {col(1, 0, np.min):10.2f} "
              f"{col(1, 5, np.max):10.2f} {col(2, 2, np.min):11.2f} {col(2, 2, np.median):10.2f} "
              f"{col(2, 5, np.max):10.2f} {col(3, 1, np.max):10.2f} {col(2, 8, np.max):10.2f}")
t = T[args.slots - 1]
t0 = t[0][t[0][:, 0] > 0][:, 0].min()
names = {0: ["start", "end", "tile0_in", "tile1_in", "tile2_in", "tile3_in", "setup_smem", "setup_done", "epi_t0", "epi_t1", "epi_t2", "epi_t3", "mma0_issued", "epi_loop_done", "flushed", "pdl_released"], 1: ["start", "pdl_done", "lse", "z_hist", "sync1", "cand_scan", "sync2", "end", "gathered", "ranked", "B_found", "pass1_done", "emitted", "nseg", "loaded_max", "exp_sum"],
         3: ["merge_start", "merge_done", "ml_ready", "o_issued", "weights"],
         2: ["start", "pdl_done", "issued", "AB_in", "logits", "V_in", "partial_done", "merge_end", "pv_done", "synced", "exit"]}
for kid, kn in [(0, "score"), (1, "select"), (2, "sparse_attn"), (3, "merge")]:
    m = t[kid]
    rows = m[m[:, 0] > 0]
    print(f"== {kn}: {len(rows)} CTAs")
    for e, en in enumerate(names[kid]):
        col = rows[:, e]
        col = col[col > 0]
        if len(col):
            r = (col - t0) / 1e3
            print(f"   {en:14s} n={len(r):4d} min={r.min():8.2f} p50={np.median(r):8.2f} p90={np.percentile(r, 90):8.2f} max={r.max():8.2f} us")

if args.raw_epi:
    m = t[0][:148]
    for e, nm in zip(range(8, 12), ["wait_acc_full", "tmem_ld", "arrive", "compute_store"]):
        c = m[:, e]; c = c[c > 0]
        if len(c):
            print(f"   epi tile2 {nm:14s} cycles p50={np.median(c):8.0f} p90={np.percentile(c, 90):8.0f} max={c.max():8.0f}")
