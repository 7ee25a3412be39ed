"""Multi-GPU plumbing for the decode path (host logic only; no data-path collective).

ShadowKV's per-layer decode step is independent per request and per KV head (Alg 2, P:160-185:
every tensor is indexed by b and h_kv; the only cross-head object is the shared A of a request).
So the path shards with no exchange step:

  * by request: rank r owns requests [r*B/N, (r+1)*B/N)   (c3: 64 requests over N GPUs)
  * by KV head when the batch is smaller than the world: rank r owns KV heads [r*H/N, (r+1)*H/N)
    of every request (A replicated; its q heads follow the GQA map hq -> floor(hq/g), R2)

torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only for the start barrier, the
max-over-ranks step time and the token count; never on the data path.
"""
from __future__ import annotations

import dataclasses

import torch


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of n units: rank gets [lo, hi)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return n * rank // world, n * (rank + 1) // world


@dataclasses.dataclass(frozen=True)
class Plan:
    mode: str              # "request" or "kv_head"
    requests: tuple        # (lo, hi) request range owned by this rank
    kv_heads: tuple        # (lo, hi) KV-head range owned by this rank
    q_heads: tuple         # (lo, hi) query-head range (GQA map)

    @property
    def batch(self) -> int:
        return self.requests[1] - self.requests[0]

    @property
    def n_kv_heads(self) -> int:
        return self.kv_heads[1] - self.kv_heads[0]

    @property
    def n_q_heads(self) -> int:
        return self.q_heads[1] - self.q_heads[0]


def plan(batch: int, n_q_heads: int, n_kv_heads: int, rank: int, world: int) -> Plan:
    """Request sharding when batch >= world, else KV-head sharding (every rank gets >= 1 unit)."""
    g = n_q_heads // n_kv_heads
    if batch >= world:
        r = shard_range(batch, rank, world)
        return Plan("request", r, (0, n_kv_heads), (0, n_q_heads))
    if batch * n_kv_heads < world:
        raise ValueError(f"{batch} requests x {n_kv_heads} KV heads cannot feed {world} ranks")
    if batch != 1:
        raise ValueError("KV-head sharding is defined for a single request (batch < world => batch 1 here)")
    h = shard_range(n_kv_heads, rank, world)
    return Plan("kv_head", (0, 1), h, (h[0] * g, h[1] * g))


def tokens_this_rank(p: Plan, n_kv_heads: int) -> float:
    """This rank's share of the job's decode tokens per step: its requests, or, under KV-head sharding,
    the fraction of the request's heads it computes (the ranks' shares sum to the batch)."""
    return p.batch * p.n_kv_heads / n_kv_heads


def max_over_ranks(value: float, device=None) -> float:
    """Step time of the whole job = the slowest rank (timing rule)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def job_tokens_per_s(tokens_this_rank: float, step_s_this_rank: float, device=None) -> float:
    """Whole-job decode tokens/s: all ranks' tokens per step / max-over-ranks step time."""
    return sum_over_ranks(tokens_this_rank, device) / max_over_ranks(step_s_this_rank, device)


def shard_state(state, p: Plan):
    """The shard of one layer's state a rank owns under plan p, as VIEWS of `state`'s tensors (no copy):
    requests [lo, hi) (every tensor's leading dim), or, for a single request, KV heads [lo, hi) with A
    replicated.  The views are contiguous, so they can be handed to the C ABI as they are;
    on a real N-GPU run each rank allocates exactly these shapes itself.  Returns a LayerState."""
    import dataclasses as dc

    from .state import LayerState
    S = state.shape
    r0, r1 = p.requests
    h0, h1 = p.kv_heads
    if p.mode == "kv_head" and S.batch != 1:
        raise ValueError("KV-head shards are views of a single-request state")
    lens = S.ctx_lens[r0:r1] if S.ctx_lens is not None else None
    shape = dc.replace(S, batch=r1 - r0, n_kv_heads=h1 - h0, n_q_heads=(h1 - h0) * (S.n_q_heads // S.n_kv_heads),
                       ctx_lens=lens)
    req = lambda t: None if t is None else t[r0:r1]
    head = lambda t: None if t is None else t[r0:r1, h0:h1]
    t = dict(A=req(state.A), B=head(state.B), landmarks=head(state.landmarks), outlier_ids=head(state.outlier_ids),
             K_out=head(state.K_out), V_out=head(state.V_out), K_win=head(state.K_win), V_win=head(state.V_win),
             V_host=head(state.V_host), A_gen=req(state.A_gen), vc_values=head(state.vc_values),
             vc_dir=head(state.vc_dir), vc_stats=head(state.vc_stats), vc_slots=head(state.vc_slots),
             vc_capacity=state.vc_capacity)
    for k, v in t.items():
        if isinstance(v, torch.Tensor) and not v.is_contiguous():
            raise ValueError(f"shard view of {k} is not contiguous")
    return LayerState.from_tensors(shape, state.A.device, **t)
