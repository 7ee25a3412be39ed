"""Time Alg 1's device build (shadowkv_build_cache) of one c2 layer: python tools/build_probe.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = synth.CONFIGS[os.environ.get("CFG", "c2")]
shape = Shape.from_config(cfg, steps=64)
rope = RopeTable(*synth.rope_table(cfg))
ws = alloc_workspace(shape)
inp = synth.gen_layer(cfg, 1234, layer=0, device="cuda")
st = LayerState(shape)
st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
ts = []
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st.build(rope.struct, ws); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{cfg.name} build_cache: median {ts[len(ts) // 2]:.3f} ms, min {ts[0]:.3f} ms over {reps}")
