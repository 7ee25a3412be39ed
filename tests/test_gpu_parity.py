"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on identical seeded inputs.

Tolerances: selection bit-exact except score ties within 1e-5 in z (R1);
outputs <= 2e-2 max-abs; rebuilt keys <= 1e-2 relative; stored bf16 state <= 1 ulp (R13);
value copies bit-exact.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import shadowkv_oracle as O
from tests.parity import (Problem, assert_bf16_close, check_decode, f64, outliers_valid)

pytestmark = pytest.mark.gpu

C1 = synth.CONFIGS["c1"]
CASES = {
    "c1": C1,
    "glm_g16_interleaved": C1.replace(n_q_heads=32, n_kv_heads=2, rope="glm"),
    "g1_batch2": C1.replace(batch=2, n_q_heads=8, n_kv_heads=8, ctx_len=2048, budget=4),
    "g2_rank64": C1.replace(n_q_heads=16, n_kv_heads=8, rank=64, ctx_len=1536),
    "g8_ragged": C1.replace(n_q_heads=32, n_kv_heads=4, ctx_len=4100, budget=20),
    "full_budget": C1.replace(ctx_len=1040, n_outlier=3, budget=(1040 - 16) // 8 - 3),
    "no_outliers": C1.replace(ctx_len=2048, n_outlier=0, budget=16, window_ctx=0),
    "multi_tile_k": C1.replace(ctx_len=16384, budget=40, n_outlier=9, window_ctx=64),
}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU parity tests need a CUDA device (run via gpurun)")


def _build_checks(P, ost):
    c = P.cfg
    assert_bf16_close(f64(P.st.landmarks), ost.landmarks, what="landmarks")
    gids = P.st.outlier_ids.cpu().numpy()
    for bi in range(c.batch):
        for h in range(c.n_kv_heads):
            if c.n_outlier == 0:
                continue
            assert outliers_valid(gids[bi, h], ost.mincos[bi, h], c.n_outlier), (bi, h, gids[bi, h], ost.outlier_ids[bi, h])
            if np.array_equal(gids[bi, h], ost.outlier_ids[bi, h]):
                assert_bf16_close(f64(P.st.K_out[bi, h]), ost.K_out[bi, h], what="K_out")
                np.testing.assert_array_equal(f64(P.st.V_out[bi, h]), ost.V_out[bi, h])
    w = P.shape.w_eff
    assert_bf16_close(f64(P.st.K_win[:, :, :w]), ost.K_win[:, :, :w], what="K_win")
    np.testing.assert_array_equal(f64(P.st.V_win[:, :, :w]), ost.V_win[:, :, :w])


@pytest.mark.parametrize("name", list(CASES))
def test_build_parity(name):
    P = Problem(CASES[name], seed=0)
    P.gpu_build()
    _build_checks(P, P.oracle_build())


def test_build_parity_given_K_rope():
    P = Problem(C1.replace(ctx_len=2048), seed=3, K_rope=True)
    P.gpu_build()
    _build_checks(P, P.oracle_build())


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("seed", [0, 1])
def test_decode_parity_identical_state(name, seed):
    """Oracle-built state bytes fed to both decoders; 3 consecutive steps (window grows)."""
    P = Problem(CASES[name], seed=seed, steps=4)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    for step in range(3):
        si = P.step_inputs(step)
        gout, gsel, gkeys = P.gpu_decode(step, si)
        _, ost = P.check(ost, step, si, (gout, gsel, gkeys))
        slot = P.shape.w_eff + step
        np.testing.assert_array_equal(f64(P.st.K_win[:, :, slot]), f64(si["k_new"]))
        np.testing.assert_array_equal(f64(P.st.V_win[:, :, slot]), f64(si["v_new"]))


@pytest.mark.parametrize("name", ["c1", "glm_g16_interleaved", "g1_batch2", "multi_tile_k"])
def test_decode_parity_cuda_core_score(name, monkeypatch):
    """Same parity check with the CUDA-core score kernel (fallback when TMA tensor maps are unavailable)."""
    monkeypatch.setenv("SKV_NO_TC", "1")
    P = Problem(CASES[name], seed=4, steps=2)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    for step in range(2):
        si = P.step_inputs(step)
        gout, gsel, gkeys = P.gpu_decode(step, si)
        _, ost = P.check(ost, step, si, (gout, gsel, gkeys))


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("name", ["c1", "glm_g16_interleaved", "multi_tile_k"])
def test_decode_parity_select_fallback(name, mode, monkeypatch):
    """The exact radix-select fallback of a3 (taken for pathological score distributions): forced
    before (1) or after (2) the definite chunks are published."""
    monkeypatch.setenv("SKV_SELECT_FALLBACK", mode)
    P = Problem(CASES[name], seed=6, steps=2)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    for step in range(2):
        si = P.step_inputs(step)
        gout, gsel, gkeys = P.gpu_decode(step, si)
        _, ost = P.check(ost, step, si, (gout, gsel, gkeys))


@pytest.mark.parametrize("name", ["c1", "glm_g16_interleaved", "g8_ragged"])
def test_end_to_end_build_then_decode(name):
    """GPU build -> GPU decode vs oracle build -> oracle decode (states may differ by 1 bf16 ulp)."""
    P = Problem(CASES[name], seed=5)
    P.gpu_build()
    ost = P.oracle_build()
    c = P.cfg
    g = c.n_q_heads // c.n_kv_heads
    overlap, total, exact = 0, 0, 0
    for step in range(2):
        si = P.step_inputs(step)
        gout, gsel, gkeys = P.gpu_decode(step, si)
        ost0 = ost
        oout, osel, oz, okeys, ost = P.oracle_decode(ost, step, si)
        # outputs on every head: the oracle's own where the sets agree, else the oracle on the GPU's set
        oout_g = P.oracle_decode(ost0, step, si, sel=gsel)[0]
        for bi in range(c.batch):
            for h in range(c.n_kv_heads):
                overlap += len(set(gsel[bi, h]) & set(osel[bi, h])); total += c.budget
                same = np.array_equal(gsel[bi, h], osel[bi, h])
                exact += same
                ref = oout if same else oout_g
                err = np.abs(gout[bi, h * g:(h + 1) * g] - ref[bi, h * g:(h + 1) * g]).max()
                assert err <= 2e-2, (err, bi, h, same)
    assert overlap >= 0.97 * total and exact >= 1


def test_full_size_c2_layer():
    """BASELINE configs[1] at full size (128K, 48 outliers, k = 256), the bench's launch configuration:
    GPU build vs oracle build, then decode on identical state bytes."""
    cfg = synth.CONFIGS["c2"]
    P = Problem(cfg, seed=1234, steps=2)
    P.gpu_build()
    ost = P.oracle_build()
    _build_checks(P, ost)
    P.load_state_from_oracle(ost)
    si = P.step_inputs(0)
    gout, gsel, gkeys = P.gpu_decode(0, si)
    P.check(ost, 0, si, (gout, gsel, gkeys))


def test_decode_deterministic_and_unpinned_rejected():
    from paper_2410_21465_b200 import LayerState, binding as bd
    P = Problem(C1, seed=2)
    P.gpu_build()
    si = P.step_inputs(0)
    a = P.gpu_decode(0, si)
    for _ in range(4):                     # bit-identical across repeats (no timing-dependent order)
        b = P.gpu_decode(0, si)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    bad = LayerState(P.shape, V_host=torch.empty(P.shape.batch, C1.n_kv_heads, C1.ctx_len, 128,
                                                 dtype=torch.bfloat16).pin_memory())
    bad.V_host = torch.empty(P.shape.batch, C1.n_kv_heads, C1.ctx_len, 128, dtype=torch.bfloat16)  # pageable
    with pytest.raises(bd.ShadowKVError, match="SKV_ESTATE"):
        bad.build(P.rope.struct, P.ws)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_sampled(name):
    """The other BASELINE configs at full size in the bench's launch configuration (whole per-GPU batch
    in one call: c3 64 x 122K, c4 1M ctx with k = 2048, c5 GLM 12 x 256K with g = 16).  The oracle
    cannot build the whole batch in seconds, so it builds + decodes sampled requests (first, last) from
    the same generator inputs; the GPU state of those requests is then replaced by the oracle's bytes
    so the decode comparison runs on identical state (as in test_decode_parity_identical_state)."""
    from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace
    cfg = synth.CONFIGS[name]
    shape = Shape.from_config(cfg, steps=2)
    inp = synth.gen_layer(cfg, 7, device="cuda")                 # generator output, not the CUDA path's
    st = LayerState(shape)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    inv, rot, il = synth.rope_table(cfg)
    rope = RopeTable(inv, rot, il)
    ws = alloc_workspace(shape)
    st.build(rope.struct, ws)
    torch.cuda.synchronize()
    sample = sorted({0, cfg.batch - 1})
    A64 = f64(inp["A"][sample]); B64 = f64(inp["B"][sample]); V64 = f64(inp["V"][sample].cpu())
    del inp
    ost = O.build(A64, B64, V64, inv, rot, il, cfg.chunk, cfg.n_outlier, cfg.window_ctx, shape.window_cap)
    bf = torch.bfloat16
    for j, bi in enumerate(sample):
        assert_bf16_close(f64(st.landmarks[bi]), ost.landmarks[j], what=f"landmarks b={bi}")
        gids = st.outlier_ids[bi].cpu().numpy()
        for h in range(cfg.n_kv_heads):
            assert outliers_valid(gids[h], ost.mincos[j, h], cfg.n_outlier)
        st.landmarks[bi].copy_(torch.from_numpy(ost.landmarks[j]).to(bf))
        st.outlier_ids[bi].copy_(torch.from_numpy(ost.outlier_ids[j]).to(torch.int32))
        st.K_out[bi].copy_(torch.from_numpy(ost.K_out[j]).to(bf)); st.V_out[bi].copy_(torch.from_numpy(ost.V_out[j]).to(bf))
        st.K_win[bi].copy_(torch.from_numpy(ost.K_win[j]).to(bf)); st.V_win[bi].copy_(torch.from_numpy(ost.V_win[j]).to(bf))
    si = synth.gen_step(cfg, 7, 0, 0)
    out = torch.empty(cfg.batch, cfg.n_q_heads, cfg.head_dim, dtype=bf, device="cuda")
    sel = torch.empty(cfg.batch, cfg.n_kv_heads, cfg.budget, dtype=torch.int32, device="cuda")
    dbg = torch.empty(cfg.batch, cfg.n_kv_heads, cfg.budget * cfg.chunk, cfg.head_dim, dtype=bf, device="cuda")
    st.decode(rope.struct, si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda(), 0, out, ws, sel_ids=sel, dbg_keys=dbg)
    torch.cuda.synchronize()
    oout, osel, oz, okeys, _ = O.decode_step(ost, A64, B64, V64, f64(si["q"][sample]), f64(si["k_new"][sample]),
                                             f64(si["v_new"][sample]), 0, cfg.budget, inv, rot, il, cfg.chunk)
    sub = cfg.replace(batch=len(sample))
    rerun = lambda s_: O.decode_step(ost, A64, B64, V64, f64(si["q"][sample]), f64(si["k_new"][sample]),
                                     f64(si["v_new"][sample]), 0, cfg.budget, inv, rot, il, cfg.chunk, sel=s_)
    check_decode(sub, f64(out[sample]), sel[sample].cpu().numpy(), f64(dbg[sample]), oout, osel, oz, okeys,
                 rerun=rerun)
    assert torch.isfinite(out.float()).all()                      # the unsampled requests ran too


@pytest.mark.parametrize("name", ["c1", "g8_ragged"])
def test_decode_step_dev_and_graph_replay(name):
    """shadowkv_decode_step_dev (step read on the device, grid sized for max_step) and one captured CUDA
    graph replayed across steps give bit-identical outputs to shadowkv_decode_step."""
    P = Problem(CASES[name], seed=8, steps=5)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    c = P.cfg
    max_step = 3
    steps = [P.step_inputs(s) for s in range(4)]
    ref = []
    for s, si in enumerate(steps):
        out = torch.empty(c.batch, c.n_q_heads, c.head_dim, dtype=torch.bfloat16, device="cuda")
        P.st.decode(P.rope.struct, si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda(), s, out, P.ws)
        ref.append(out.clone())
    step_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
    for s, si in enumerate(steps):                        # device step, plain launches
        step_dev.fill_(s)
        out = torch.empty_like(ref[0])
        P.st.decode_dev(P.rope.struct, si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda(), step_dev, max_step,
                        out, P.ws)
        torch.cuda.synchronize()
        assert torch.equal(out, ref[s]), f"step_dev decode differs at step {s}"
    q_b = steps[0]["q"].cuda().clone(); k_b = steps[0]["k_new"].cuda().clone(); v_b = steps[0]["v_new"].cuda().clone()
    out_b = torch.empty_like(ref[0])
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        step_dev.fill_(0)
        P.st.decode_dev(P.rope.struct, q_b, k_b, v_b, step_dev, max_step, out_b, P.ws, stream=side)   # warm-up
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            P.st.decode_dev(P.rope.struct, q_b, k_b, v_b, step_dev, max_step, out_b, P.ws, stream=side)
            step_dev.add_(1)
        step_dev.fill_(0)
        for s, si in enumerate(steps):
            q_b.copy_(si["q"]); k_b.copy_(si["k_new"]); v_b.copy_(si["v_new"])
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out_b, ref[s]), f"graph replay differs at step {s}"


@pytest.mark.parametrize("name,q_len", [("c1", 2), ("c1", 4), ("g2_rank64", 8), ("g1_batch2", 2),
                                        ("multi_tile_k", 4)])
def test_decode_parity_multi_query(name, q_len):
    """s_q = q_len query tokens per call (Alg 2's Q[b][h_q][s_q][d], NEXT-3): one shared selection from
    S1 = sum over s_q, causal attention among the new tokens (R28); three calls in a row so the
    window holds earlier multi-token appends."""
    P = Problem(CASES[name], seed=6, steps=3, q_len=q_len)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    for call in range(3):
        step = call * q_len
        si = P.step_inputs(step)
        gout, gsel, gkeys = P.gpu_decode(step, si)
        assert gout.shape == (P.cfg.batch, P.cfg.n_q_heads, q_len, P.cfg.head_dim)
        _, ost = P.check(ost, step, si, (gout, gsel, gkeys))
