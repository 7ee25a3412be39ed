"""Bit-reproducibility check: the same decode call repeated on one layer state gives identical outputs.

python tools/determinism.py <config> <reps>   (SKV_SPLIT / SKV_SERIALIZE honoured)"""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace
name = sys.argv[1]; reps = int(sys.argv[2])
cfg = synth.CONFIGS[name]
shape = Shape.from_config(cfg, steps=2)
inp = synth.gen_layer(cfg, 7, device="cuda")
st = LayerState(shape); st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
rope = RopeTable(*synth.rope_table(cfg)); ws = alloc_workspace(shape)
st.build(rope.struct, ws); torch.cuda.synchronize(); del inp
si = synth.gen_step(cfg, 7, 0, 0)
q, kn, vn = si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda()
outs = []
tag = f"{name} split={os.environ.get('SKV_SPLIT')} serial={os.environ.get('SKV_SERIALIZE')}"
for r in range(reps):
    out = torch.empty(cfg.batch, cfg.n_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    t0 = time.time()
    try:
        st.decode(rope.struct, q, kn, vn, 0, out, ws)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(tag, "rep", r, "FAILED after", round(time.time() - t0, 2), "s:", str(e)[:120], flush=True)
        sys.exit(1)
    outs.append(out.clone())
    print(tag, "rep", r, "ok", round(time.time() - t0, 3), "s", flush=True)
diffs = [int((o.view(torch.int16) != outs[0].view(torch.int16)).sum()) for o in outs]
print(tag, "mismatching elements vs first:", diffs, flush=True)
for r, o in enumerate(outs):
    bad = (o.view(torch.int16) != outs[0].view(torch.int16)).any(-1).nonzero().tolist()
    if bad:
        print(tag, "rep", r, "differing (b, hq) rows:", bad[:40], "... total", len(bad), flush=True)
