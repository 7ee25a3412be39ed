"""Ragged batches (per-request context lengths) through the C ABI vs the oracle.

Every request b of a batch padded to ctx_len has its own length s_b: its own chunk grid, outliers,
window tail (R8 per request) and decode positions.  The oracle runs each request alone on its own
s_b tokens (slices of the same seeded inputs); the GPU runs the whole padded batch in one call.
Build: landmarks within 1 bf16 ulp (R13), outlier sets valid under the min-cos tie rule (R12),
window tail keys within 1 ulp and values bit-exact.  Decode: the usual selection / key / output
tolerances (R1, R23) per request, over two steps, from identical state bytes.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import shadowkv_oracle as O
from tests.parity import assert_bf16_close, check_decode, f64, outliers_valid

pytestmark = pytest.mark.gpu

C1 = synth.CONFIGS["c1"]
CASES = {
    "llama_b3": (C1.replace(batch=3, ctx_len=4096, budget=8), [4096, 3001, 2053], [0, 1, 2]),
    "glm_g16_b2": (C1.replace(batch=2, n_q_heads=32, n_kv_heads=2, rope="glm", ctx_len=2048, budget=12),
                   [1500, 2048], [0, 1]),
    "b32_sub_batch_chains": (C1.replace(batch=32, n_q_heads=8, n_kv_heads=2, ctx_len=1024, budget=8, n_outlier=2),
                             [1024 - 20 * i for i in range(32)], [0, 13, 31]),
}


@pytest.mark.parametrize("name,q_len,value_cache", [(n, 1, False) for n in CASES] +
                         [("llama_b3", 2, True), ("b32_sub_batch_chains", 4, True)])
def test_ragged_batch_parity(name, q_len, value_cache):
    """(+ s_q > 1 query tokens and the value cache on the same ragged batch: every NEXT-3 / NEXT-1
    feature at once; with the cache, results are also bit-identical to a cache-less twin)."""
    from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace
    cfg, lens, sample = CASES[name]
    steps, seed = (3 if value_cache else 2), 11
    c, o, w, k = cfg.chunk, cfg.n_outlier, cfg.window_ctx, cfg.budget
    inp = synth.gen_layer(cfg, seed)
    inv, rot, il = synth.rope_table(cfg)
    shape = Shape.from_config(cfg, steps=steps, ctx_lens=lens, q_len=q_len)
    st = LayerState(shape, value_cache=value_cache)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    rope = RopeTable(inv, rot, il)
    ws = alloc_workspace(shape)
    st.build(rope.struct, ws)
    torch.cuda.synchronize()
    A64, B64, V64 = f64(inp["A"]), f64(inp["B"]), f64(inp["V"])
    ost = {}
    gids = st.outlier_ids.cpu().numpy()
    bf = torch.bfloat16
    for b in sample:
        sb = lens[b]
        ob = O.build(A64[b:b + 1, :sb], B64[b:b + 1], V64[b:b + 1, :, :sb], inv, rot, il, c, o, w, shape.window_cap)
        n_c, w_eff = ob.n_c, ob.w_eff
        assert_bf16_close(f64(st.landmarks[b, :, :n_c]), ob.landmarks[0], what=f"landmarks b={b}")
        for h in range(cfg.n_kv_heads):
            assert outliers_valid(gids[b, h], ob.mincos[0, h], o), f"outliers b={b} h={h}"
        assert_bf16_close(f64(st.K_win[b, :, :w_eff]), ob.K_win[0, :, :w_eff], what=f"window keys b={b}")
        assert np.array_equal(f64(st.V_win[b, :, :w_eff]), ob.V_win[0, :, :w_eff]), f"window values b={b}"
        ost[b] = ob
        # identical state bytes for decode parity (R13): the oracle's build output for this request
        st.landmarks[b, :, :n_c].copy_(torch.from_numpy(ob.landmarks[0]).to(bf))
        st.outlier_ids[b].copy_(torch.from_numpy(ob.outlier_ids[0]).to(torch.int32))
        st.K_out[b].copy_(torch.from_numpy(ob.K_out[0]).to(bf)); st.V_out[b].copy_(torch.from_numpy(ob.V_out[0]).to(bf))
        st.K_win[b].copy_(torch.from_numpy(ob.K_win[0]).to(bf)); st.V_win[b].copy_(torch.from_numpy(ob.V_win[0]).to(bf))
    twin = None
    if value_cache:
        twin = LayerState(shape, V_host=st.V_host)
        for n in ("A", "B", "landmarks", "outlier_ids", "K_out", "V_out", "K_win", "V_win"):
            getattr(twin, n).copy_(getattr(st, n))
    one = cfg.replace(batch=1)
    qd = synth.gen_q_drift(cfg, seed, 0, steps * q_len, 0.97)           # drifting: the cache gets hits
    for call in range(steps):
        step = call * q_len
        toks = [synth.gen_step(cfg, seed, 0, step + i) for i in range(q_len)]
        for i, t in enumerate(toks):
            t["q"] = qd[step + i]
        if q_len == 1:
            si = toks[0]
        else:
            si = {n: torch.stack([t[n] for t in toks], dim=2) for n in ("q", "k_new", "v_new")}
        out = torch.empty(si["q"].shape, dtype=bf, device="cuda")
        sel = torch.empty(cfg.batch, cfg.n_kv_heads, k, dtype=torch.int32, device="cuda")
        dbg = torch.empty(cfg.batch, cfg.n_kv_heads, k * c, cfg.head_dim, dtype=bf, device="cuda")
        st.decode(rope.struct, si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda(), step, out, ws,
                  sel_ids=sel, dbg_keys=dbg)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
        if twin is not None:
            out2 = torch.empty_like(out)
            sel2 = torch.empty_like(sel)
            twin.decode(rope.struct, si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda(), step, out2, ws,
                        sel_ids=sel2)
            torch.cuda.synchronize()
            assert torch.equal(out, out2) and torch.equal(sel, sel2), "value cache changed a ragged result"
        for b in sample:
            sb = lens[b]
            run = lambda st0, sel_=None, b=b, sb=sb: O.decode_step(
                st0, A64[b:b + 1, :sb], B64[b:b + 1], V64[b:b + 1, :, :sb], f64(si["q"][b:b + 1]),
                f64(si["k_new"][b:b + 1]), f64(si["v_new"][b:b + 1]), step, k, inv, rot, il, c, sel=sel_)
            st_prev = ost[b]
            oo, os_, oz, ok, ost[b] = run(st_prev)
            assert sel[b].max().item() < ost[b].n_c, "selected a chunk past the request's own grid"
            check_decode(one, f64(out[b:b + 1]), sel[b:b + 1].cpu().numpy(), f64(dbg[b:b + 1]), oo, os_, oz, ok,
                         rerun=lambda s_, st_prev=st_prev, run=run: run(st_prev, s_))
    if value_cache:
        assert int(st.cache_stats()[..., 3].sum()) > 0, "drifting queries produced no cache hits"


def test_ragged_graph_replay_matches_per_call():
    """The graph-replayable entry point (device step counter) on a ragged batch with s_q = 2 and low-rank
    generated keys: one captured graph replayed over three calls reproduces per-call decoding bit for bit."""
    from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace
    cfg, lens, _ = CASES["llama_b3"]
    q_len, calls, seed = 2, 3, 13
    inp = synth.gen_layer(cfg, seed)
    inv, rot, il = synth.rope_table(cfg)
    shape = Shape.from_config(cfg, steps=calls, ctx_lens=lens, q_len=q_len)
    rope = RopeTable(inv, rot, il)
    ws = alloc_workspace(shape)
    st = LayerState(shape, lowrank_gen=True)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    st.build(rope.struct, ws)
    torch.cuda.synchronize()
    win0 = (st.K_win.clone(), st.V_win.clone())
    ins = []
    for call in range(calls):
        toks = [synth.gen_step(cfg, seed, 0, call * q_len + i) for i in range(q_len)]
        ins.append({n: torch.stack([t[n] for t in toks], dim=2).cuda() for n in ("q", "k_new", "v_new")})
    ref = []
    for call, si in enumerate(ins):
        out = torch.empty(si["q"].shape, dtype=torch.bfloat16, device="cuda")
        st.decode(rope.struct, si["q"], si["k_new"], si["v_new"], call * q_len, out, ws)
        torch.cuda.synchronize()
        ref.append(out.clone())
    st.K_win.copy_(win0[0]); st.V_win.copy_(win0[1]); st.A_gen.zero_()
    qb, kb, vb = (ins[0][n].clone() for n in ("q", "k_new", "v_new"))
    ob = torch.empty_like(ref[0])
    step_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            st.decode_dev(rope.struct, qb, kb, vb, step_dev, (calls - 1) * q_len, ob, ws, stream=side)
            step_dev.add_(q_len)
        torch.cuda.synchronize()
        step_dev.fill_(0)
        st.K_win.copy_(win0[0]); st.V_win.copy_(win0[1]); st.A_gen.zero_()
        torch.cuda.synchronize()
        for call, si in enumerate(ins):
            qb.copy_(si["q"]); kb.copy_(si["k_new"]); vb.copy_(si["v_new"])
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(ob, ref[call]), f"graph replay differs at call {call}"
