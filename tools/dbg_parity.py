import numpy as np, torch, sys
sys.path.insert(0, '.')
import synth
from tests.parity import Problem
from paper_2410_21465_b200.state import ws_ptr
cfg = synth.CONFIGS["c1"]
P = Problem(cfg, seed=0, steps=4)
ost = P.oracle_build(); P.load_state_from_oracle(ost)
si = P.step_inputs(0)
gout, gsel, gkeys = P.gpu_decode(0, si)
oout, osel, oz, okeys, ost = P.oracle_decode(ost, 0, si)
S = P.shape; b, hq, hk, n_c, k, wcap = 1, 32, 8, S.n_c, 8, S.window_cap
al = lambda x: (x + 255) // 256 * 256
off = al(b * hk * 5 * 4)
o_log = off; off += al(b * hq * n_c * 4)
o_part = off; off += al(b * hq * 64 * 8)
o_z = off; off += al(b * hk * n_c * 4)
o_sel = off; off += al(b * hk * k * 4)
o_rest = off; off += al(b * hk * k * 4)
n_sel_u = (k + 7) // 8 + 1; n_out_u = (4 * 8 + 63) // 64; n_win_max = (wcap + 63) // 64
n_split_alloc = n_sel_u + n_out_u + n_win_max
o_op = off; off += al(b * hq * n_split_alloc * 128 * 4)
o_ml = off
n_split = n_sel_u + n_out_u + 1
base = ws_ptr(P.ws) - P.ws.data_ptr()
raw = P.ws[base:].cpu()
def arr(o, n, dt): return raw[o:o + n * 4].view(dt).numpy()
sel = arr(o_sel, hk * k, torch.int32).reshape(hk, k); rest = arr(o_rest, hk * k, torch.int32).reshape(hk, k)
print("def list h0", sel[0], "rest h0", rest[0], "oracle sel", osel[0, 0])
op = arr(o_op, hq * n_split * 128, torch.float32).reshape(hq, n_split, 128)
ml = arr(o_ml, hq * n_split * 2, torch.float32).reshape(hq, n_split, 2)
for h in range(4):
    print("qhead", h, "ml", np.round(ml[h], 3).tolist(), "o norms", np.round(np.linalg.norm(op[h], axis=1), 3))
for h in range(4):
    m = ml[h, :, 0]; l = ml[h, :, 1]; M = m.max(); w = np.exp(m - M)
    o = (w[:, None] * op[h]).sum(0) / (w * l).sum()
    print("qhead", h, "merge-from-partials vs oracle", np.abs(o - oout[0, h]).max(), "gpu vs oracle", np.abs(gout[0, h] - oout[0, h]).max())
print("counters+flags", raw[:160].view(torch.int32).numpy()[:40])
