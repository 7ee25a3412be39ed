"""Multi-GPU shards on one GPU: the per-rank slice of a layer's state -- by request,
or by KV head with A replicated -- decoded alone through the C ABI gives the same output, selection and
rebuilt-key bytes as the unsharded call, which itself is checked against the oracle.

Bit-identity holds because every result of a (request, KV head) is computed from that unit's data in
an order that does not depend on the rest of the batch: the score kernel writes one softmax partial
per 128-landmark tile and k_select merges a head's tiles in a fixed order (no per-CTA segments), the
select cluster, the attention units and the merge are per (request, KV head).  So on N GPUs each rank
reproduces its share of the single-GPU result exactly, with no collective.
"""
import numpy as np
import pytest
import torch

import synth
from paper_2410_21465_b200 import alloc_workspace, shard
from tests.parity import Problem, f64

pytestmark = pytest.mark.gpu

C1 = synth.CONFIGS["c1"]


def _decode(st, rope, ws, q, kn, vn, step):
    c = st.shape
    out = torch.empty(q.shape, dtype=torch.bfloat16, device="cuda")
    sel = torch.empty(c.batch, c.n_kv_heads, c.budget, dtype=torch.int32, device="cuda")
    dbg = torch.empty(c.batch, c.n_kv_heads, c.budget * c.chunk, c.head_dim, dtype=torch.bfloat16, device="cuda")
    st.decode(rope, q, kn, vn, step, out, ws, sel_ids=sel, dbg_keys=dbg)
    torch.cuda.synchronize()
    return out, sel, dbg


def _check_shards(st, rope, si, full, world, step=0):
    cfg = st.shape
    g = cfg.n_q_heads // cfg.n_kv_heads
    q, kn, vn = si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda()
    covered = 0.0
    for rank in range(world):
        pl = shard.plan(cfg.batch, cfg.n_q_heads, cfg.n_kv_heads, rank, world)
        sub = shard.shard_state(st, pl)
        ws = alloc_workspace(sub.shape)
        (r0, r1), (h0, h1) = pl.requests, pl.kv_heads
        qs = q[r0:r1, h0 * g:h1 * g].contiguous()
        ks, vs = kn[r0:r1, h0:h1].contiguous(), vn[r0:r1, h0:h1].contiguous()
        out, sel, dbg = _decode(sub, rope, ws, qs, ks, vs, step)
        assert torch.equal(out, full[0][r0:r1, h0 * g:h1 * g]), f"rank {rank}/{world} ({pl.mode}): output differs"
        assert torch.equal(sel, full[1][r0:r1, h0:h1]), f"rank {rank}/{world}: selection differs"
        assert torch.equal(dbg, full[2][r0:r1, h0:h1]), f"rank {rank}/{world}: rebuilt keys differ"
        covered += shard.tokens_this_rank(pl, cfg.n_kv_heads)
    assert abs(covered - cfg.batch) < 1e-9


CASES = {
    "request_c1x4": (C1.replace(batch=4), [2, 4]),
    "kv_head_c1": (C1, [2, 4, 8]),
    "kv_head_glm_g16": (C1.replace(n_q_heads=32, n_kv_heads=2, rope="glm"), [2]),
    "request_multi_tile": (C1.replace(batch=3, ctx_len=16384, budget=40, n_outlier=9, window_ctx=64), [3]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_shards_bit_identical_and_oracle_checked(name):
    cfg, worlds = CASES[name]
    P = Problem(cfg, seed=31, steps=2)
    ost = P.oracle_build()
    P.load_state_from_oracle(ost)
    si = P.step_inputs(0)
    q, kn, vn = si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda()
    full = _decode(P.st, P.rope.struct, P.ws, q, kn, vn, 0)
    P.check(ost, 0, si, (f64(full[0]), full[1].cpu().numpy(), f64(full[2])))      # the unsharded call vs oracle
    for world in worlds:
        _check_shards(P.st, P.rope.struct, si, full, world)


def test_ragged_request_shards():
    """Ragged batch (per-request lengths, R29) split by request: each shard carries its own lengths."""
    from paper_2410_21465_b200 import LayerState, RopeTable, Shape
    cfg = C1.replace(batch=4, ctx_len=4096)
    lens = [4096, 3001, 2053, 3800]
    shape = Shape.from_config(cfg, steps=2, ctx_lens=lens)
    inp = synth.gen_layer(cfg, 33)
    st = LayerState(shape)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    inv, rot, il = synth.rope_table(cfg)
    rope = RopeTable(inv, rot, il)
    ws = alloc_workspace(shape)
    st.build(rope.struct, ws)
    si = synth.gen_step(cfg, 33, 0, 0)
    full = _decode(st, rope.struct, ws, si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda(), 0)
    _check_shards(st, rope.struct, si, full, 2)
    _check_shards(st, rope.struct, si, full, 4)


def test_c3_request_shards_full_size():
    """BASELINE configs[2] at full size (64 x 122K, the bench's whole-batch launch incl. the 4 sub-batch
    chains): the shards of ranks 0 and N-1 for N = 2 and 8 reproduce the single-GPU result's bytes."""
    from paper_2410_21465_b200 import LayerState, RopeTable, Shape
    cfg = synth.CONFIGS["c3"]
    shape = Shape.from_config(cfg, steps=2)
    inp = synth.gen_layer(cfg, 7, device="cuda")
    st = LayerState(shape)
    st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); st.V_host.copy_(inp["V"])
    del inp
    inv, rot, il = synth.rope_table(cfg)
    rope = RopeTable(inv, rot, il)
    ws = alloc_workspace(shape)
    st.build(rope.struct, ws)
    si = synth.gen_step(cfg, 7, 0, 0)
    q, kn, vn = si["q"].cuda(), si["k_new"].cuda(), si["v_new"].cuda()
    full = _decode(st, rope.struct, ws, q, kn, vn, 0)
    g = cfg.n_q_heads // cfg.n_kv_heads
    for world in (2, 8):
        for rank in (0, world - 1):
            pl = shard.plan(cfg.batch, cfg.n_q_heads, cfg.n_kv_heads, rank, world)
            sub = shard.shard_state(st, pl)
            (r0, r1) = pl.requests
            out, sel, dbg = _decode(sub, rope.struct, alloc_workspace(sub.shape), q[r0:r1].contiguous(),
                                    kn[r0:r1].contiguous(), vn[r0:r1].contiguous(), 0)
            assert torch.equal(out, full[0][r0:r1]) and torch.equal(sel, full[1][r0:r1])
            assert torch.equal(dbg, full[2][r0:r1])
