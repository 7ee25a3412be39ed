"""Does replaying a captured CUDA graph of one 32-layer decode step beat stream launches? (c2)"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace  # noqa: E402
cfg = synth.CONFIGS["c2"]
L = 32
shape = Shape.from_config(cfg, steps=4096)
rope = RopeTable(*synth.rope_table(cfg))
ws = alloc_workspace(shape)
states = []
for l in range(L):
    inp = synth.gen_layer(cfg, 1234, layer=l, device="cuda")
    st = LayerState(shape); st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    st.build(rope.struct, ws); states.append(st); del inp
sis = [synth.gen_step(cfg, 1234, l, 0, device="cuda") for l in range(L)]
out = torch.empty(L, cfg.batch, cfg.n_q_heads, 128, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.Stream()
def step(i):
    for l, st in enumerate(states):
        st.decode(rope.struct, sis[l]["q"], sis[l]["k_new"], sis[l]["v_new"], i % 4000, out[l], ws,
                  stream=torch.cuda.current_stream())
with torch.cuda.stream(s):
    for i in range(5): step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [step(5) for _ in range(100)]; e1.record(); torch.cuda.synchronize()
    print("stream launches: %.3f ms/step" % (e0.elapsed_time(e1) / 100))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step(6)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0.record(); [g.replay() for _ in range(100)]; e1.record(); torch.cuda.synchronize()
    print("graph replay:    %.3f ms/step" % (e0.elapsed_time(e1) / 100))
