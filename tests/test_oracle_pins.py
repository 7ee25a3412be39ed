"""Pins for the CPU oracle (runs without a GPU: -m "not gpu").

Each test ties an oracle function to something other than itself: the paper's
printed worked example, hand-computed cases (tests/golden/), closed forms,
library routines (numpy/scipy/torch) or brute force on tiny inputs.  A plausible
mistake anywhere in the oracle -- a dropped term, wrong sign, wrong index,
transposed operand -- should fail at least one of these.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

from oracle import shadowkv_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


# ---------------------------------------------------------------- bf16 store
def test_bf16_round_hand_cases():
    for x, want in GOLD["bf16_rounding"]["cases"]:
        assert O.bf16_round(np.array([x]))[0] == want, (x, want)


def test_bf16_round_matches_torch_on_fp32_inputs():
    # torch's fp32 -> bf16 conversion is RNE; from an fp32 value it is a single rounding.
    g = torch.Generator().manual_seed(0)
    x = torch.randn(20000, generator=g) * torch.exp(torch.randn(20000, generator=g) * 3)
    want = x.to(torch.bfloat16).double().numpy()
    got = O.bf16_round(x.double().numpy())
    np.testing.assert_array_equal(got, want)


# ---------------------------------------------------------------- partition
def test_partition_examples():
    assert O.partition(4096, 8, 16) == (510, 16)
    assert O.partition(4100, 8, 16) == (510, 20)      # ragged tail absorbed by the window (R8)
    assert O.partition(131072, 8, 16) == (16382, 16)
    assert O.partition(64, 8, 0) == (8, 0)            # S:192 "s=64, c=8 -> n_c = 8"


# ---------------------------------------------------------------- RoPE
def _rope_complex(x, pos, inv_freq, rot, interleaved):
    """Independent formulation: multiply complex pairs by exp(i phi)."""
    x = np.asarray(x, np.float64)
    phi = (np.asarray(pos).astype(np.float32)[:, None] * np.asarray(inv_freq, np.float32)[None, :])
    rotor = np.exp(1j * phi.astype(np.float32).astype(np.float64))
    out = x.copy()
    if interleaved:
        z = (x[..., 0:rot:2] + 1j * x[..., 1:rot:2]) * rotor
        out[..., 0:rot:2], out[..., 1:rot:2] = z.real, z.imag
    else:
        h = rot // 2
        z = (x[..., :h] + 1j * x[..., h:rot]) * rotor
        out[..., :h], out[..., h:rot] = z.real, z.imag
    return out


def test_rope_position_zero_identity():
    x = np.random.default_rng(0).normal(size=(1, 16))
    inv = np.array([1.0, 0.5, 0.25, 0.125, 0.1, 0.01, 0.001, 1e-4], np.float32)
    np.testing.assert_array_equal(O.rope(x, [0], inv, 16, False), x)


def test_rope_d2_rotates_by_one_radian():
    # d = 2, position 1, inv_freq 1 -> rotation of (x, y) by exactly 1 rad
    out = O.rope(np.array([[1.0, 0.0], [0.0, 1.0]]), [1, 1], np.array([1.0], np.float32), 2, False)
    np.testing.assert_allclose(out, [[math.cos(1), math.sin(1)], [-math.sin(1), math.cos(1)]], atol=1e-15)


@pytest.mark.parametrize("interleaved,rot", [(False, 128), (True, 64), (False, 64)])
def test_rope_matches_complex_rotation(interleaved, rot):
    rng = np.random.default_rng(1)
    x = rng.normal(size=(50, 128))
    pos = rng.integers(0, 2_000_000, size=50)
    inv = (1.0 / 500000.0 ** (np.arange(0, rot, 2) / rot)).astype(np.float32)
    np.testing.assert_allclose(O.rope(x, pos, inv, rot, interleaved),
                               _rope_complex(x, pos, inv, rot, interleaved), atol=1e-12)
    if rot < 128:   # pass-through dims
        np.testing.assert_array_equal(O.rope(x, pos, inv, rot, interleaved)[:, rot:], x[:, rot:])


def test_rope_isometry_and_relative_position():
    rng = np.random.default_rng(2)
    x, y = rng.normal(size=(1, 32)), rng.normal(size=(1, 32))
    inv = (2.0 ** -np.arange(16)).astype(np.float32)           # exact fp32 angles
    r = lambda v, p: O.rope(v, [p], inv, 32, False)[0]
    np.testing.assert_allclose(np.linalg.norm(r(x, 777)), np.linalg.norm(x), rtol=1e-14)
    d1 = r(x, 10) @ r(y, 3)
    d2 = r(x, 107) @ r(y, 100)
    assert abs(d1 - d2) < 1e-12                                 # depends only on p - p'


# ---------------------------------------------------------------- chunk stats / outliers
def test_constant_chunk_landmark_and_cos():
    v = np.random.default_rng(3).normal(size=8)
    grid = np.tile(v, (16, 1))                                  # 2 chunks of c = 8, constant
    C = O.chunk_means(grid, 8)
    np.testing.assert_allclose(C, np.tile(v, (2, 1)), rtol=1e-15)
    np.testing.assert_allclose(O.chunk_min_cos(grid, C, 8), [1.0, 1.0], atol=1e-15)


def test_two_token_chunk_half_angle():
    # c = 2, |x| = |y|, angle theta between them -> cos(mean, x) = cos(theta / 2) (geometry)
    theta = 1.234
    x = np.array([3.0, 0.0]); y = 3.0 * np.array([math.cos(theta), math.sin(theta)])
    grid = np.stack([x, y])
    m = O.chunk_min_cos(grid, O.chunk_means(grid, 2), 2)
    assert abs(m[0] - math.cos(theta / 2)) < 1e-15


def test_zero_norm_gives_minus_one():
    grid = np.ones((8, 4)); grid[5] = 0.0
    assert O.chunk_min_cos(grid, O.chunk_means(grid, 8), 8)[0] == -1.0


def test_planted_antialigned_token_is_sole_outlier():
    # chunk 3 holds one token anti-aligned with its chunk; other chunks constant
    rng = np.random.default_rng(4)
    c, n_c, d = 8, 8, 16
    grid = np.repeat(rng.normal(size=(n_c, d)), c, axis=0)
    others = grid[3 * c + 1: 4 * c]
    grid[3 * c] = -others.mean(axis=0)
    m = O.chunk_min_cos(grid, O.chunk_means(grid, c), c)
    assert m[3] < 0 and np.all(np.delete(m, 3) > 1 - 1e-12)
    assert list(O.smallest_o(m, 1)) == [3]


def test_smallest_o_brute_force_and_ties():
    rng = np.random.default_rng(5)
    for _ in range(50):
        m = rng.normal(size=9)
        o = int(rng.integers(0, 5))
        best = min(itertools.combinations(range(9), o), key=lambda S: sum(m[list(S)]))
        assert list(O.smallest_o(m, o)) == sorted(best)
    m = np.array([0.5, 0.1, 0.1, 0.1, 0.9])
    assert list(O.smallest_o(m, 2)) == [1, 2]                   # ties -> lower index (R12)


# ---------------------------------------------------------------- scoring / selection
def test_normalise_group_max_vs_scipy_softmax():
    rng = np.random.default_rng(6)
    lg = rng.normal(size=(4, 30)) * 3
    mask = np.ones(30, bool); mask[[2, 17]] = False
    z = O.normalise_group_max(lg, mask)
    S = scipy.special.softmax(lg[:, mask], axis=1)              # Softmax over the landmarks only
    np.testing.assert_allclose(np.exp(z[mask]), S.max(axis=0), rtol=1e-12)
    assert np.all(np.isneginf(z[~mask]))


def test_gqa_hand_example():
    ex = GOLD["gqa_hand_example"]
    lg = O.landmark_scores(np.array(ex["q"]), np.array(ex["L"]), ex["d"])
    z = O.normalise_group_max(lg, np.ones(2, bool))
    np.testing.assert_allclose(np.exp(z), ex["S2"], rtol=1e-12)
    assert list(O.arg_topk(z, 1)) == [ex["top1"]]


def test_normalisation_counterexample():
    ex = GOLD["normalisation_counterexample"]
    lg = np.array(ex["logits"])
    z = O.normalise_group_max(lg, np.ones(3, bool))
    np.testing.assert_allclose(np.exp(z), ex["S2"], rtol=1e-6)
    assert list(O.arg_topk(z, 1)) == [ex["top1_normalised"]]
    assert int(np.argmax(lg.max(axis=0))) == ex["top1_raw"]      # raw-logit max would differ (R5)


def test_landmark_scores_scale_and_orientation():
    # P = Q L^T / sqrt(d): entry [hq][j] = <q_hq, L_j> / sqrt(d) -- check one entry by hand
    q = np.array([[1.0, 2.0, 0.0, 0.0], [0.0, 0.0, 3.0, 0.0]])
    L = np.array([[1.0, 1.0, 1.0, 1.0], [0.0, 0.0, 0.0, 2.0], [5.0, 0.0, 0.0, 0.0]])
    P = O.landmark_scores(q, L, 4)
    assert P.shape == (2, 3)
    np.testing.assert_allclose(P, [[1.5, 0.0, 2.5], [1.5, 0.0, 0.0]])


def test_arg_topk_brute_force_ties_and_g1():
    rng = np.random.default_rng(7)
    for _ in range(60):
        n = int(rng.integers(1, 12)); k = int(rng.integers(1, n + 1))
        z = rng.normal(size=n)
        best = max(itertools.combinations(range(n), k), key=lambda S: sum(z[list(S)]))
        assert list(O.arg_topk(z, k)) == sorted(best)
    z = np.array([1.0, 3.0, 3.0, 3.0, 0.0])
    assert list(O.arg_topk(z, 2)) == [1, 2]
    # g = 1: selection == top-k of raw logits (softmax is monotone) via argsort
    lg = rng.normal(size=(1, 40))
    z = O.normalise_group_max(lg, np.ones(40, bool))
    assert list(O.arg_topk(z, 7)) == sorted(np.argsort(-lg[0], kind="stable")[:7])


def test_selection_nested_and_mass_monotone():
    rng = np.random.default_rng(8)
    z = O.normalise_group_max(rng.normal(size=(4, 100)) * 2, np.ones(100, bool))
    prev, prev_mass = set(), 0.0
    for k in range(1, 100):
        sel = set(O.arg_topk(z, k).tolist())
        mass = float(np.exp(z[list(sel)]).sum())
        assert prev <= sel and mass >= prev_mass - 1e-15
        prev, prev_mass = sel, mass


# ---------------------------------------------------------------- rebuild / SVD
def test_jacobi_svd_matches_numpy():
    X = np.random.default_rng(9).normal(size=(20, 7))
    U, s, Vt = O.jacobi_svd(X)
    np.testing.assert_allclose(s, np.linalg.svd(X, compute_uv=False), rtol=1e-12)
    np.testing.assert_allclose((U * s) @ Vt, X, atol=1e-12)
    # Eckart-Young: truncation error = sqrt(sum_{i>r} s_i^2)
    r = 3
    err = np.linalg.norm(X - (U[:, :r] * s[:r]) @ Vt[:r])
    assert abs(err - math.sqrt((np.linalg.svd(X, compute_uv=False)[r:] ** 2).sum())) < 1e-12


@pytest.mark.parametrize("true_rank,r", [(16, 16), (3, 3), (3, 5)])
def test_rebuild_exact_for_rank_deficient_keys(true_rank, r):
    # Alg 1 "A, B <- SVD(K)" over keys flattened across KV heads, Alg 2 rebuild
    rng = np.random.default_rng(10)
    s, hk, d = 40, 2, 8
    K = rng.normal(size=(s, true_rank)) @ rng.normal(size=(true_rank, hk * d))
    U, sig, Vt = O.jacobi_svd(K)
    A = U[:, :r] * sig[:r]
    B = Vt[:r].reshape(r, hk, d).transpose(1, 0, 2)
    inv = (1.0 / 10000 ** (np.arange(0, d, 2) / d)).astype(np.float32)
    tok = np.array([3, 4, 5, 17, 39])
    for h in range(hk):
        got = O.rebuild_keys(A, B[h], tok, inv, d, False)
        want = _rope_complex(K[tok, h * d:(h + 1) * d], tok, inv, d, False)
        np.testing.assert_allclose(got, want, atol=1e-11)


# ---------------------------------------------------------------- attention
def test_softmax_attention_special_cases():
    rng = np.random.default_rng(11)
    q = rng.normal(size=8)
    k1, v1 = rng.normal(size=(1, 8)), rng.normal(size=(1, 8))
    np.testing.assert_allclose(O.softmax_attention(q, k1, v1), v1[0], rtol=1e-15)
    K = np.tile(rng.normal(size=8), (5, 1)); V = rng.normal(size=(5, 8))
    np.testing.assert_allclose(O.softmax_attention(q, K, V), V.mean(axis=0), atol=1e-14)


def test_dense_attention_vs_scipy():
    rng = np.random.default_rng(12)
    q = rng.normal(size=(4, 16)); K = rng.normal(size=(2, 9, 16)); V = rng.normal(size=(2, 9, 16))
    out = O.dense_attention(q, K, V)
    for hq in range(4):
        p = scipy.special.softmax(K[hq // 2] @ q[hq] / 4.0)
        np.testing.assert_allclose(out[hq], p @ V[hq // 2], atol=1e-14)


def _small_problem(seed, s=200, hk=2, g=2, d=16, r=12, c=8, w=5, interleaved=False, rot=None):
    rng = np.random.default_rng(seed)
    rot = rot or d
    A = rng.normal(size=(1, s, r)); B = rng.normal(size=(1, hk, r, d)) / math.sqrt(r)
    V = rng.normal(size=(1, hk, s, d))
    inv = (1.0 / 10000 ** (np.arange(0, rot, 2) / rot)).astype(np.float32)
    return A, B, V, inv, rot, rng


@pytest.mark.parametrize("interleaved,rot,o,w", [(False, 16, 3, 5), (True, 8, 0, 0), (False, 16, 7, 8)])
def test_full_coverage_equals_dense_attention(interleaved, rot, o, w):
    """North-star pin: k = n_L, exact keys (self-check mode) => sparse path == dense attention over all tokens."""
    s, hk, g, d, c = 203, 2, 3, 16, 8
    A, B, V, inv, rot, rng = _small_problem(13, s=s, hk=hk, g=g, d=d, w=w, interleaved=interleaved, rot=rot)
    n_c, w_eff = O.partition(s, c, w)
    st = O.build(A, B, V, inv, rot, interleaved, c, o, w, window_cap=w_eff + 3, store=O.identity_store)
    keys_ctx = np.stack([_rope_complex(A[0] @ B[0, h], np.arange(s), inv, rot, interleaved) for h in range(hk)])
    gen_k, gen_v = [], []
    for step in range(3):
        q = rng.normal(size=(1, hk * g, d)) * 2
        kn = rng.normal(size=(1, hk, d)); vn = rng.normal(size=(1, hk, d))
        gen_k.append(kn[0]); gen_v.append(vn[0])
        out, sel, z, kt, st = O.decode_step(st, A, B, V, q, kn, vn, step, n_c - o, inv, rot, interleaved, c,
                                            store=O.identity_store)
        keys = np.concatenate([keys_ctx, np.stack(gen_k, axis=1)], axis=1)
        vals = np.concatenate([V[0], np.stack(gen_v, axis=1)], axis=1)
        want = O.dense_attention(q[0], keys, vals)
        np.testing.assert_allclose(out[0], want, atol=1e-12)
        for h in range(hk):   # every landmark selected
            assert sorted(set(sel[0, h]) | set(st.outlier_ids[0, h])) == list(range(n_c))


def test_full_coverage_with_given_K_rope():
    s, hk, g, d, c, o, w = 120, 2, 2, 16, 8, 2, 8
    A, B, V, inv, rot, rng = _small_problem(14, s=s, hk=hk, g=g, d=d, w=w)
    # with K_rope given, keys attended are K_rope for outliers/window but the rebuild uses A.B;
    # pass K_rope == RoPE(A.B) built independently -> must equal dense attention.
    Kr = np.stack([_rope_complex(A[0] @ B[0, h], np.arange(s), inv, d, False) for h in range(hk)])[None]
    n_c, w_eff = O.partition(s, c, w)
    st = O.build(A, B, V, inv, d, False, c, o, w, w_eff + 1, K_rope=Kr, store=O.identity_store)
    q = rng.normal(size=(1, hk * g, d)); kn = rng.normal(size=(1, hk, d)); vn = rng.normal(size=(1, hk, d))
    out, *_ = O.decode_step(st, A, B, V, q, kn, vn, 0, n_c - o, inv, d, False, c, store=O.identity_store)
    keys = np.concatenate([Kr[0], kn[0][:, None]], axis=1); vals = np.concatenate([V[0], vn[0][:, None]], axis=1)
    np.testing.assert_allclose(out[0], O.dense_attention(q[0], keys, vals), atol=1e-12)


def test_build_invariants_and_value_copy():
    s, hk, d, c, o, w = 160, 2, 16, 8, 4, 7
    A, B, V, inv, rot, rng = _small_problem(15, s=s, hk=hk, d=d, w=w)
    n_c, w_eff = O.partition(s, c, w)
    st = O.build(A, B, V, inv, d, False, c, o, w, w_eff)
    for h in range(hk):
        ids = st.outlier_ids[0, h]
        assert len(set(ids.tolist())) == o and list(ids) == sorted(ids) and ids.max() < n_c
        tok = (ids[:, None] * c + np.arange(c)).reshape(-1)
        np.testing.assert_array_equal(st.V_out[0, h], V[0, h, tok])         # exact copy
        np.testing.assert_array_equal(st.V_win[0, h], V[0, h, n_c * c:])
        assert np.all(O.bf16_round(st.landmarks[0, h]) == st.landmarks[0, h])  # stored bf16
    st0 = O.build(A, B, V, inv, d, False, c, 0, w, w_eff)
    assert st0.outlier_ids.shape[2] == 0 and st0.K_out.shape[2] == 0


def test_needle_chunk_selected():
    # plant one chunk whose keys align with q -> its landmark dominates -> selected
    s, hk, g, d, c, o, w = 400, 1, 4, 16, 8, 2, 8
    rng = np.random.default_rng(16)
    A, B, V, inv, rot, _ = _small_problem(16, s=s, hk=hk, g=g, d=d, w=w)
    n_c, w_eff = O.partition(s, c, w)
    q = rng.normal(size=(1, g, d))
    Kr = np.stack([_rope_complex(A[0] @ B[0, h], np.arange(s), inv, d, False) for h in range(hk)])[None]
    needle = 23
    Kr[0, 0, needle * c:(needle + 1) * c] = 6.0 * q[0, 1] / np.linalg.norm(q[0, 1]) + 0.01 * rng.normal(size=(c, d))
    st = O.build(A, B, V, inv, d, False, c, o, w, w_eff + 1, K_rope=Kr)
    kn = rng.normal(size=(1, hk, d)); vn = rng.normal(size=(1, hk, d))
    _, sel, z, _, _ = O.decode_step(st, A, B, V, q, kn, vn, 0, 3, inv, d, False, c)
    assert needle in sel[0, 0]
    assert int(np.argmax(z[0, 0])) == needle


def test_equivalent_bandwidth_paper_example():
    ex = GOLD["equivalent_bandwidth"]
    beq = O.equivalent_bandwidth(ex["S"], ex["C"], ex["K"], ex["O"], ex["alpha"], ex["B_gpu"], ex["B_pcie"])
    assert abs(beq / 1e12 - ex["expected_TBps"]) <= ex["abs_tol_TBps"]
    # alpha = 1 limit drops the PCIe term; monotone in alpha and B_PCIe
    lim = O.equivalent_bandwidth(ex["S"], ex["C"], ex["K"], ex["O"], 1.0, ex["B_gpu"], ex["B_pcie"])
    assert abs(lim - 2 * ex["S"] * ex["B_gpu"] / (ex["S"] / ex["C"] + 2 * (ex["K"] + ex["O"]) * ex["C"])) < 1e-3
    vals = [O.equivalent_bandwidth(ex["S"], 8, 256, 48, a, 2e12, 31.5e9) for a in np.linspace(0, 1, 11)]
    assert all(b > a for a, b in zip(vals, vals[1:]))


def test_paper_operating_point_arithmetic():
    kc = GOLD["key_compression"]
    assert kc["h_kv_times_d"] / kc["rank"] == kc["expected_ratio"]
    of = GOLD["outlier_fraction"]
    frac = of["o"] / O.partition(of["s"], of["c"], 16)[0]
    assert of["lo"] <= frac <= of["hi"]


# ---------------------------------------------------------------- s_q > 1 (NEXT-3, Alg 2's Q[b][h_q][s_q][d])
def test_multi_query_sum_hand_example():
    ex = GOLD["multi_query_sum_example"]
    lg = np.array(ex["logits"])
    z = O.normalise_sum_group_max(lg, np.ones(lg.shape[-1], bool))
    np.testing.assert_allclose(np.exp(z), ex["S1"], atol=1e-6)
    assert O.arg_topk(z, 1)[0] == ex["top1"]


def test_multi_query_reduces_to_single_query():
    """s_q = 1: normalise_sum_group_max == normalise_group_max, and the 4-D decode == the 3-D decode."""
    rng = np.random.default_rng(21)
    lg = rng.normal(size=(3, 1, 40)) * 2
    mask = rng.random(40) > 0.2
    np.testing.assert_allclose(O.normalise_sum_group_max(lg, mask)[mask], O.normalise_group_max(lg[:, 0], mask)[mask],
                               atol=1e-12)
    s, hk, g, d, c, o, w = 160, 2, 2, 16, 8, 2, 8
    A, B, V, inv, rot, rng = _small_problem(22, s=s, hk=hk, g=g, d=d, w=w)
    n_c, w_eff = O.partition(s, c, w)
    st = O.build(A, B, V, inv, d, False, c, o, w, w_eff + 2)
    q = rng.normal(size=(1, hk * g, d)); kn = rng.normal(size=(1, hk, d)); vn = rng.normal(size=(1, hk, d))
    o3, s3, z3, k3, _ = O.decode_step(st, A, B, V, q, kn, vn, 1, 5, inv, d, False, c)
    o4, s4, z4, k4, _ = O.decode_step(st, A, B, V, q[:, :, None], kn[:, :, None], vn[:, :, None], 1, 5, inv, d,
                                      False, c)
    np.testing.assert_array_equal(s3, s4)
    np.testing.assert_allclose(o4[:, :, 0], o3, atol=1e-12)
    np.testing.assert_allclose(z4, z3, atol=1e-12)


@pytest.mark.parametrize("sq", [2, 4])
def test_multi_query_full_coverage_equals_causal_dense_attention(sq):
    """k = n_L, exact keys: each of the s_q query tokens == dense attention over the context, the earlier
    generated tokens and the new tokens up to and including itself (causal, R28)."""
    s, hk, g, d, c, o, w = 150, 2, 2, 16, 8, 3, 6
    A, B, V, inv, rot, rng = _small_problem(23, s=s, hk=hk, g=g, d=d, w=w)
    n_c, w_eff = O.partition(s, c, w)
    st = O.build(A, B, V, inv, d, False, c, o, w, w_eff + 2 * sq, store=O.identity_store)
    keys_ctx = np.stack([_rope_complex(A[0] @ B[0, h], np.arange(s), inv, d, False) for h in range(hk)])
    gk, gv = [], []
    for call in range(2):
        step = call * sq
        q = rng.normal(size=(1, hk * g, sq, d)) * 2
        kn = rng.normal(size=(1, hk, sq, d)); vn = rng.normal(size=(1, hk, sq, d))
        out, sel, z, kt, st = O.decode_step(st, A, B, V, q, kn, vn, step, n_c - o, inv, d, False, c,
                                            store=O.identity_store)
        for i in range(sq):
            gk.append(kn[0, :, i]); gv.append(vn[0, :, i])
            keys = np.concatenate([keys_ctx, np.stack(gk, axis=1)], axis=1)
            vals = np.concatenate([V[0], np.stack(gv, axis=1)], axis=1)
            np.testing.assert_allclose(out[0, :, i], O.dense_attention(q[0, :, i], keys, vals), atol=1e-12)


@pytest.mark.parametrize("sq", [1, 2])
def test_given_selection_equals_dense_attention_over_that_set(sq):
    """decode_step(sel=J) (the R23 test hook: oracle evaluated on the GPU's set) attends exactly the
    outlier tokens, the tokens of the chunks in J (any order given) and the window: equal to dense
    attention over that explicit token subset with independently rebuilt keys (self-check mode)."""
    s, hk, g, d, c, o, w = 203, 2, 2, 16, 8, 3, 5
    A, B, V, inv, rot, rng = _small_problem(21, s=s, hk=hk, g=g, d=d, w=w)
    n_c, w_eff = O.partition(s, c, w)
    st = O.build(A, B, V, inv, rot, False, c, o, w, window_cap=w_eff + 4, store=O.identity_store)
    keys_ctx = np.stack([_rope_complex(A[0] @ B[0, h], np.arange(s), inv, rot, False) for h in range(hk)])
    k = 5
    J = np.stack([rng.permutation([j for j in range(n_c) if j not in set(st.outlier_ids[0, h])])[:k]
                  for h in range(hk)])[None]
    q = rng.normal(size=(1, hk * g, sq, d)) * 2 if sq > 1 else rng.normal(size=(1, hk * g, d)) * 2
    kn = rng.normal(size=(1, hk, sq, d)) if sq > 1 else rng.normal(size=(1, hk, d))
    vn = rng.normal(size=(1, hk, sq, d)) if sq > 1 else rng.normal(size=(1, hk, d))
    out, sel, z, kt, _ = O.decode_step(st, A, B, V, q, kn, vn, 0, k, inv, rot, False, c, store=O.identity_store,
                                       sel=J)
    for h in range(hk):
        assert list(sel[0, h]) == sorted(J[0, h])
        toks = sorted({t for j in list(J[0, h]) + list(st.outlier_ids[0, h]) for t in range(j * c, j * c + c)} |
                      set(range(n_c * c, s)))
        for i in range(sq):
            kn_i = kn[0, h, i] if sq > 1 else kn[0, h]
            vn_i = vn[0, h, i] if sq > 1 else vn[0, h]
            gk = np.stack([kn[0, h, t] for t in range(i + 1)]) if sq > 1 else kn_i[None]
            gv = np.stack([vn[0, h, t] for t in range(i + 1)]) if sq > 1 else vn_i[None]
            keys = np.concatenate([keys_ctx[h, toks], gk])
            vals = np.concatenate([V[0, h, toks], gv])
            for j in range(g):
                qq = q[0, h * g + j, i] if sq > 1 else q[0, h * g + j]
                got = out[0, h * g + j, i] if sq > 1 else out[0, h * g + j]
                np.testing.assert_allclose(got, O.dense_attention(qq[None], keys[None], vals[None])[0], atol=1e-12)
        # the rebuilt keys are reported in the ascending order of the given set
        tk = [t for j in sorted(J[0, h]) for t in range(j * c, j * c + c)]
        np.testing.assert_allclose(kt[0, h], keys_ctx[h, tk], atol=1e-12)
