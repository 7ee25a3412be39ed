"""Pins for the oracle's value-chunk cache (DESIGN R26).

Each pin ties ``oracle.ValueChunkCache`` to something other than itself: SPEC's worked examples,
a closed form (capacity = k reduces LRU to "the previous selection"), an independent recount of
the least-recently-selected definition straight from the trace, and the i.i.d. steady state k/n.
"""
import numpy as np
import pytest

from oracle import shadowkv_oracle as O


def test_same_id_twice_is_hit():
    """'same id fetched twice consecutively -> second fetch is a hit'."""
    c = O.ValueChunkCache(4)
    assert not c.fetch([7])[0]
    assert c.fetch([7])[0]


def test_capacity_zero_always_misses():
    """'capacity 0 -> every fetch is a miss'."""
    c = O.ValueChunkCache(0)
    for _ in range(5):
        assert not c.fetch([1, 2, 3]).any()
    assert c.hit_rate() == 0.0


def _trace(rng, n, k, steps, drift):
    """Selection trace with temporal locality: each step keeps ~drift of the previous set."""
    cur = rng.choice(n, k, replace=False)
    out = [np.sort(cur)]
    for _ in range(steps - 1):
        keep = cur[rng.random(k) < drift]
        rest = np.setdiff1d(np.arange(n), keep)
        cur = np.concatenate([keep, rng.choice(rest, k - len(keep), replace=False)])
        out.append(np.sort(cur))
    return out


@pytest.mark.parametrize("seed", range(4))
def test_capacity_k_hits_equal_previous_overlap(seed):
    """Closed form: with capacity = k and k-sized selections the cache after step t holds exactly
    S_t, so hits_t = |S_t & S_{t-1}| (the GPU implements this case with ping-pong slot buffers)."""
    rng = np.random.default_rng(seed)
    n, k = 200, 16
    tr = _trace(rng, n, k, 60, 0.6)
    hits = O.replay_hits(tr, k)
    want = [0] + [len(np.intersect1d(tr[t], tr[t - 1])) for t in range(1, len(tr))]
    np.testing.assert_array_equal(hits, want)


def _recount(trace, capacity):
    """Least-recently-selected, restated from the trace alone: before call t the cache holds the
    `capacity` previously selected ids with the largest (last selection time, id)."""
    out = []
    for t, ids in enumerate(trace):
        last = {}
        for u in range(t):
            for j in trace[u]:
                last[int(j)] = u
        resident = set(sorted(last, key=lambda j: (last[j], j), reverse=True)[:capacity])
        out.append(np.array([int(j) in resident for j in ids]))
    return out


@pytest.mark.parametrize("capacity", [0, 3, 8, 13, 40])
def test_lru_matches_event_by_event_recount(capacity):
    """S:146 '[DERIVED: independent recount oracle over the same trace]', at capacities below,
    equal to and above k, with a varying request size."""
    rng = np.random.default_rng(capacity)
    n = 30
    trace = [np.sort(rng.choice(n, int(rng.integers(1, 9)), replace=False)) for _ in range(80)]
    c = O.ValueChunkCache(capacity)
    got = [c.fetch(ids) for ids in trace]
    want = _recount(trace, capacity)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
    assert c.hits == sum(int(w.sum()) for w in want)
    assert c.requested == sum(len(t) for t in trace)


def test_iid_uniform_steady_state_is_k_over_n():
    """i.i.d. uniform k-subsets of n chunks, capacity k -> hit rate ~ k/n
    (E|S_t & S_{t-1}| = k^2/n)."""
    rng = np.random.default_rng(11)
    n, k, steps = 64, 8, 4000
    trace = [rng.choice(n, k, replace=False) for _ in range(steps)]
    hits = O.replay_hits(trace, k)
    rate = hits[1:].sum() / (k * (steps - 1))
    assert abs(rate - k / n) < 0.01, rate


def test_replay_is_deterministic():
    """S:150 'Replaying the identical selection trace twice yields identical stats'."""
    rng = np.random.default_rng(5)
    tr = _trace(rng, 100, 10, 50, 0.5)
    np.testing.assert_array_equal(O.replay_hits(tr, 10), O.replay_hits(tr, 10))


def test_hit_rate_feeds_equivalent_bandwidth():
    """B_eq rises with alpha; alpha = 0.6 (Fig 3c) reproduces the paper's 7.2 TB/s
    while alpha = 0 gives the uncached figure (S=128K, K=256, O=48, A100 bandwidths)."""
    b0 = O.equivalent_bandwidth(131072, 8, 256, 48, 0.0, 2e12, 31.5e9)
    b6 = O.equivalent_bandwidth(131072, 8, 256, 48, 0.6, 2e12, 31.5e9)
    # closed form of the denominator at alpha = 0: 16384 + 4864 + 2048 * 2e12 / 31.5e9
    assert b0 == pytest.approx(2 * 131072 * 2e12 / (16384 + 4864 + 2048 * 2e12 / 31.5e9), rel=1e-12)
    assert 7.1e12 < b6 < 7.3e12 and b0 < b6


def test_drift_queries_recipe():
    """synth.gen_q_drift (DESIGN R27): stationary N(0, tau^2) marginals and lag-1 correlation rho."""
    import synth
    import torch
    cfg = synth.CONFIGS["c1"]
    for rho in (0.0, 0.9):
        q = synth.gen_q_drift(cfg, 3, 0, 400, rho).float()
        assert abs(q.std().item() - 2.0) < 0.05
        a, b = q[1:].flatten(), q[:-1].flatten()
        corr = torch.corrcoef(torch.stack([a, b]))[0, 1].item()
        assert abs(corr - rho) < 0.02, (rho, corr)
