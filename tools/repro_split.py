"""Minimal multi-layer decode loop (for sanitizer runs): python tools/repro_split.py [config] [layers] [steps]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
S = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = synth.CONFIGS[name]
shape = Shape.from_config(cfg, steps=S + 1)
rope = RopeTable(*synth.rope_table(cfg))
ws = alloc_workspace(shape)
states = []
for l in range(L):
    inp = synth.gen_layer(cfg, 5, layer=l, device="cuda")
    st = LayerState(shape)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    st.build(rope.struct, ws)
    states.append(st)
    del inp
torch.cuda.synchronize()
out = torch.empty(cfg.batch, cfg.n_q_heads, 128, dtype=torch.bfloat16, device="cuda")
for step in range(S):
    for l, st in enumerate(states):
        si = synth.gen_step(cfg, 5, l, step, device="cuda")
        st.decode(rope.struct, si["q"], si["k_new"], si["v_new"], step, out, ws)
torch.cuda.synchronize()
print("ok", out.float().abs().mean().item())
