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


def _bench_dry(*extra):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", *extra], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout                       # rank 0 alone prints
    return lines[0]


def test_bench_gpus_2_self_launches_two_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run, 127.0.0.1);
    c3 defaults to strong scaling (64 requests split 64/n): each rank owns 32 requests and the
    ranks' token shares sum to the job's batch."""
    out = _bench_dry("--gpus", "2", "--config", "c3")
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    assert sorted(tuple(p["requests"]) for p in out["ranks"]) == [(0, 32), (32, 64)]
    assert out["tokens_per_step"] == 64


def test_bench_gpus_2_c2_weak_and_kv_head_split():
    """c2 defaults to weak scaling (one 128K request per GPU); --scaling strong splits its 8 KV heads."""
    out = _bench_dry("--gpus", "2", "--config", "c2")
    assert out["n_gpus"] == 2 and out["scaling"] == "weak" and out["tokens_per_step"] == 2
    out = _bench_dry("--gpus", "2", "--config", "c2", "--scaling", "strong")
    assert sorted(tuple(p["kv_heads"]) for p in out["ranks"]) == [(0, 4), (4, 8)]
    assert all(p["mode"] == "kv_head" for p in out["ranks"]) and abs(out["tokens_per_step"] - 1.0) < 1e-12
