"""GPU value-chunk cache (DESIGN R26) through the C ABI, against the oracle.

* Outputs and selections with the cache are bit-identical to the same GPU path without it (cached
  values are bit copies), and match the fp64 oracle within the decode tolerances (R1, R23).
* The per-step hit counts the kernels report equal, bit-exact, the oracle's least-recently-selected
  cache (capacity C = k and C = 3k, oracle.ValueChunkCache) replayed over the GPU's own selection trace,
  and the oracle's own trace wherever the two selections agree.
* Queries drift (synth.gen_q_drift, R27) so consecutive selections overlap.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import shadowkv_oracle as O
from tests.parity import Problem, check_decode

pytestmark = pytest.mark.gpu

C1 = synth.CONFIGS["c1"]
CASES = {
    "c1_k16": C1.replace(ctx_len=2048, budget=16),
    "g16_multi_unit": C1.replace(n_q_heads=32, n_kv_heads=2, rope="glm", ctx_len=8192, budget=40, n_outlier=6),
    "g1_batch2_ragged": C1.replace(batch=2, n_q_heads=8, n_kv_heads=8, ctx_len=3001, budget=12),
    "b32_sub_batch_chains": C1.replace(batch=32, n_q_heads=8, n_kv_heads=2, ctx_len=1024, budget=8, n_outlier=2),
}


def _drift_inputs(cfg, seed, steps, rho):
    qs = synth.gen_q_drift(cfg, seed, 0, steps, rho)
    out = []
    for t in range(steps):
        si = synth.gen_step(cfg, seed, 0, t)
        si["q"] = qs[t]
        out.append(si)
    return out


def _twin_without_cache(P):
    """A second GPU layer state holding the same bytes, without a value cache."""
    from paper_2410_21465_b200 import LayerState
    ref = LayerState(P.shape, V_host=P.st.V_host)
    for n in ("A", "B", "landmarks", "outlier_ids", "K_out", "V_out", "K_win", "V_win"):
        getattr(ref, n).copy_(getattr(P.st, n))
    return ref


@pytest.mark.parametrize("cap", [1, 3])
@pytest.mark.parametrize("name", list(CASES))
def test_value_cache_parity_and_hits(name, cap):
    cfg = CASES[name]
    steps = 8
    C = cap * cfg.budget
    P = Problem(cfg, seed=5, steps=steps, value_cache=True, vc_capacity=C)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    P.st.vc_dir.zero_(); P.st.vc_stats.zero_(); P.st.vc_slots.zero_()
    ref = _twin_without_cache(P)
    b, hk, k = cfg.batch, cfg.n_kv_heads, cfg.budget
    gtrace = [[[] for _ in range(hk)] for _ in range(b)]
    otrace = [[[] for _ in range(hk)] for _ in range(b)]
    total = 0
    for t, si in enumerate(_drift_inputs(cfg, 5, steps, 0.97)):
        gout, gsel, gkeys = P.gpu_decode(t, si)
        rout, rsel, _ = P.gpu_decode(t, si, st=ref)
        assert np.array_equal(gout, rout) and np.array_equal(gsel, rsel), f"cache changed the result at step {t}"
        ost0 = ost
        oout, osel, oz, okeys, ost = P.oracle_decode(ost, t, si)
        check_decode(cfg, gout, gsel, gkeys, oout, osel, oz, okeys,
                     rerun=lambda s_, ost0=ost0, t=t, si=si: P.oracle_decode(ost0, t, si, sel=s_))
        stats = P.st.cache_stats().numpy()
        assert (stats[..., 0] == t + 1).all()                      # one generation per decode step
        for bi in range(b):
            for h in range(hk):
                gtrace[bi][h].append(gsel[bi, h])
                otrace[bi][h].append(osel[bi, h])
                want = O.replay_hits(gtrace[bi][h], C)
                assert stats[bi, h, 2] == want[-1], f"step {t} b={bi} h={h}: gpu hits {stats[bi, h, 2]} != {want[-1]}"
                assert stats[bi, h, 3] == want.sum()
                if all(np.array_equal(x, y) for x, y in zip(gtrace[bi][h], otrace[bi][h])):
                    assert stats[bi, h, 2] == O.replay_hits(otrace[bi][h], C)[-1]
        total = int(stats[..., 3].sum())
    assert total > 0, "drifting queries produced no cache hits"
    P.gpu_build()                                                  # a new prefill resets the cache
    assert (P.st.cache_stats().numpy() == 0).all()


def test_value_cache_graph_replay():
    """One captured CUDA graph (device step, value cache inside) replayed over drifting steps gives the
    per-call results bit for bit, and the same hit counts."""
    cfg = CASES["c1_k16"]
    steps = 6
    P = Problem(cfg, seed=9, steps=steps, value_cache=True)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    win0 = (P.st.K_win.clone(), P.st.V_win.clone())
    P.st.vc_dir.zero_(); P.st.vc_stats.zero_(); P.st.vc_slots.zero_()
    inputs = _drift_inputs(cfg, 9, steps, 0.97)
    ref_out, ref_hits = [], []
    for t, si in enumerate(inputs):
        gout, _, _ = P.gpu_decode(t, si)
        ref_out.append(gout)
        ref_hits.append(P.st.cache_stats().numpy()[..., 2].copy())
    P.st.K_win.copy_(win0[0]); P.st.V_win.copy_(win0[1])
    P.st.vc_dir.zero_(); P.st.vc_stats.zero_(); P.st.vc_slots.zero_()
    c = cfg
    q_b = inputs[0]["q"].cuda().clone(); k_b = inputs[0]["k_new"].cuda().clone(); v_b = inputs[0]["v_new"].cuda().clone()
    out_b = torch.empty(c.batch, c.n_q_heads, c.head_dim, dtype=torch.bfloat16, device="cuda")
    step_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            P.st.decode_dev(P.rope.struct, q_b, k_b, v_b, step_dev, steps - 1, out_b, P.ws, stream=side)
            step_dev.add_(1)
        torch.cuda.synchronize()
        P.st.vc_dir.zero_(); P.st.vc_stats.zero_(); P.st.vc_slots.zero_(); step_dev.fill_(0)   # capture does not execute; be explicit
        torch.cuda.synchronize()
        for t, si in enumerate(inputs):
            q_b.copy_(si["q"]); k_b.copy_(si["k_new"]); v_b.copy_(si["v_new"])
            g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(out_b.double().cpu().numpy(), ref_out[t]), f"graph replay differs at step {t}"
            assert np.array_equal(P.st.cache_stats().numpy()[..., 2], ref_hits[t])
