"""Low-rank storage of generated keys (P:196 footnote) through the C ABI vs the oracle.

With skv_layer.A_gen, decode's k_new is the PRE-RoPE key; the kernels store it as one rank-r row
a = sum_h k'_h B_h^T and attend with RoPE_t(a B_h).  The oracle applies the footnote's formula
(oracle.lowrank_generated_keys) and runs its ordinary decode step with those keys: outputs and
selections must agree within the decode tolerances (R1, R23) over three consecutive calls, and the
stored rows must equal the oracle's bf16(a) within one bf16 ulp (fp32 vs fp64 sums, R13).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import shadowkv_oracle as O
from tests.parity import Problem, assert_bf16_close, f64

pytestmark = pytest.mark.gpu

C1 = synth.CONFIGS["c1"]
CASES = {
    "c1": C1,
    "g8_ragged_tail": C1.replace(n_q_heads=32, n_kv_heads=4, ctx_len=4100, budget=20),
    "glm_g16_interleaved": C1.replace(n_q_heads=32, n_kv_heads=2, rope="glm"),
}


@pytest.mark.parametrize("name,q_len", [("c1", 1), ("c1", 2), ("g8_ragged_tail", 2), ("glm_g16_interleaved", 1)])
def test_lowrank_generated_keys_parity(name, q_len):
    cfg = CASES[name]
    P = Problem(cfg, seed=12, steps=3, q_len=q_len, lowrank_gen=True)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    s = cfg.ctx_len
    for call in range(3):
        step = call * q_len
        si = P.step_inputs(step)                           # k_new: pre-RoPE keys of the new tokens
        gout, gsel, gkeys = P.gpu_decode(step, si)
        kp = f64(si["k_new"])
        kp4 = kp if kp.ndim == 4 else kp[:, :, None]
        a, keys = O.lowrank_generated_keys(kp4, P.B64, s + step + np.arange(q_len), P.inv, P.rot, P.il)
        si_o = dict(si)
        si_o["k_new"] = torch.from_numpy(keys if kp.ndim == 4 else keys[:, :, 0])
        _, ost = P.check(ost, step, si_o, (gout, gsel, gkeys))
        assert_bf16_close(f64(P.st.A_gen[:, step:step + q_len]), a, abs_slack=1e-6, what="A_gen rows")
