"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path: sharding plan and the
max-over-ranks / sum-over-ranks job throughput that bench.py reports.  No GPU needed."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_21465_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for n in (1, 7, 64, 131):
        for world in (1, 2, 3, 8):
            if n < world:
                continue
            parts = [shard.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def test_plan_modes():
    p = shard.plan(64, 32, 8, rank=3, world=8)          # c3 on 8 GPUs: 8 requests each
    assert p.mode == "request" and p.requests == (24, 32) and p.batch == 8 and p.n_kv_heads == 8
    p = shard.plan(1, 32, 8, rank=1, world=4)           # c2 on 4 GPUs: 2 KV heads (8 q heads) each
    assert p.mode == "kv_head" and p.kv_heads == (2, 4) and p.q_heads == (8, 16)
    with pytest.raises(ValueError):
        shard.plan(1, 32, 2, rank=0, world=4)           # 2 KV heads cannot feed 4 ranks


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = shard.plan(64, 32, 8, rank, world)
        step_s = 0.010 + 0.005 * rank                   # rank 1 is the slow one
        tps = shard.job_tokens_per_s(p.batch, step_s)
        t = torch.tensor([tps, shard.max_over_ranks(step_s), float(p.requests[0])], dtype=torch.float64)
        gathered = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        if rank == 0:
            out.put([g.tolist() for g in gathered])
    finally:
        dist.destroy_process_group()


def test_two_rank_job_throughput_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks agree: 64 tokens per step over the slowest rank's 15 ms
    for tps, tmax, _ in res:
        assert abs(tmax - 0.015) < 1e-12
        assert abs(tps - 64 / 0.015) < 1e-6
    assert [r[2] for r in res] == [0.0, 32.0]


def test_tokens_per_rank_sum_to_the_batch():
    """Request sharding: each rank's requests; KV-head sharding (batch < world): each rank's fraction of the
    request's heads; either way the shares sum to the job's batch (bench.py's strong-scaling tokens/s)."""
    for batch, hq, hk, world in [(64, 32, 8, 8), (64, 32, 8, 3), (1, 32, 8, 4), (1, 32, 8, 8), (1, 32, 2, 2)]:
        shares = [shard.tokens_this_rank(shard.plan(batch, hq, hk, r, world), hk) for r in range(world)]
        assert abs(sum(shares) - batch) < 1e-12
        if batch < world:
            assert all(abs(x - 1.0 / world) < 1e-12 for x in shares) or hk % world
