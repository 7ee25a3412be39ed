"""Layer-state allocation for the C ABI (plumbing: torch allocates, the library computes).

``Shape`` mirrors skv_dims; ``LayerState`` owns one layer's device tensors (A, B, landmarks,
outliers, window) plus the pinned, device-mapped host value cache V_host ("Offload the
rest of values to the CPU").  No arithmetic of the method lives here.
"""
from __future__ import annotations

import dataclasses

import torch

from . import binding as bd


@dataclasses.dataclass(frozen=True)
class Shape:
    batch: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ctx_len: int
    rank: int
    chunk: int
    n_outlier: int
    budget: int
    window_ctx: int
    window_cap: int
    q_len: int = 1          # s_q query tokens per decode call (Alg 2's Q[b][h_q][s_q][d])
    ctx_lens: tuple | None = None   # ragged batch: per-request context lengths (ctx_len = the padded length)

    @property
    def n_c(self) -> int:          # grid chunks (window absorbs the ragged tail, DESIGN R8)
        return (self.ctx_len - self.window_ctx) // self.chunk

    @property
    def w_eff(self) -> int:
        return self.ctx_len - self.n_c * self.chunk

    def dims(self, lens_host=None, lens_dev=None) -> bd.SkvDims:
        """skv_dims; a ragged shape needs its host / device length tensors (LayerState holds them)."""
        return bd.dims_struct(self.batch, self.n_q_heads, self.n_kv_heads, self.head_dim, self.ctx_len,
                              self.rank, self.chunk, self.n_outlier, self.budget, self.window_ctx,
                              self.window_cap, self.q_len, lens_host, lens_dev)

    @classmethod
    def from_config(cls, cfg, steps: int = 64, batch: int | None = None, q_len: int = 1,
                    ctx_lens=None) -> "Shape":
        """`steps` decode calls of `q_len` tokens each fit in the window.  ctx_lens: per-request
        lengths of a ragged batch (cfg.ctx_len is then the padded length)."""
        s, w, c = cfg.ctx_len, cfg.window_ctx, cfg.chunk
        w_eff = s - ((s - w) // c) * c
        if ctx_lens is not None:
            ctx_lens = tuple(int(x) for x in ctx_lens)
            # the largest per-request tail; also the padded length's own (shape.dims() without the length
            # arrays, e.g. for the workspace size, validates against it)
            w_eff = max([w_eff] + [x - ((x - w) // c) * c for x in ctx_lens])
        return cls(cfg.batch if batch is None else batch, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, s,
                   cfg.rank, c, cfg.n_outlier, cfg.budget, w, w_eff + steps * q_len, q_len, ctx_lens)


def alloc_workspace(shape: Shape, device="cuda") -> torch.Tensor:
    bd.ensure_init(device)
    n = bd.shadowkv_workspace_bytes(shape.dims())
    return torch.zeros(n + 256, dtype=torch.uint8, device=device)     # ABI: zero-filled before first use


def ws_ptr(ws: torch.Tensor) -> int:
    p = ws.data_ptr()
    return (p + 255) & ~255


class LayerState:
    """One layer's tensors for the whole per-GPU batch."""

    def __init__(self, shape: Shape, device="cuda", V_host: torch.Tensor | None = None,
                 value_cache: bool = False, lowrank_gen: bool = False, vc_capacity: int = 0):
        self.shape = S = shape
        bd.ensure_init(device)                          # shadowkv_init for this device (once)
        b, hk, d = S.batch, S.n_kv_heads, S.head_dim
        self.lens_host = self.lens_dev = None
        if S.ctx_lens is not None:                      # ragged batch: host + device length arrays
            self.lens_host = torch.tensor(S.ctx_lens, dtype=torch.int32)
            self.lens_dev = self.lens_host.to(device)
        bf = torch.bfloat16
        self.A = torch.empty(b, S.ctx_len, S.rank, dtype=bf, device=device)
        self.B = torch.empty(b, hk, S.rank, d, dtype=bf, device=device)
        self.landmarks = torch.empty(b, hk, S.n_c, d, dtype=bf, device=device)
        self.outlier_ids = torch.empty(b, hk, max(S.n_outlier, 1), dtype=torch.int32, device=device)
        oc = max(S.n_outlier * S.chunk, 1)
        self.K_out = torch.empty(b, hk, oc, d, dtype=bf, device=device)
        self.V_out = torch.empty(b, hk, oc, d, dtype=bf, device=device)
        self.K_win = torch.zeros(b, hk, S.window_cap, d, dtype=bf, device=device)
        self.V_win = torch.zeros(b, hk, S.window_cap, d, dtype=bf, device=device)
        if V_host is None:
            V_host = torch.empty(b, hk, S.ctx_len, d, dtype=bf, pin_memory=True)
        assert V_host.is_pinned() and V_host.shape == (b, hk, S.ctx_len, d)
        self.V_host = V_host
        # optional GPU-resident value-chunk cache (skv_layer.vc_*, DESIGN R26): C = vc_capacity (0: k) value
        # slots per (request, KV head), the chunk directory, the hit counters and the per-slot state
        # optional low-rank generated keys (skv_layer.A_gen, NEXT-4): one rank-r row per generated token
        self.A_gen = torch.zeros(b, S.window_cap, S.rank, dtype=bf, device=device) if lowrank_gen else None
        self.vc_values = self.vc_dir = self.vc_stats = self.vc_slots = None
        self.vc_capacity = 0
        if value_cache:
            C = vc_capacity or S.budget
            self.vc_capacity = C
            self.vc_values = torch.empty(b, hk, C, S.chunk, d, dtype=bf, device=device)
            self.vc_dir = torch.zeros(b, hk, S.n_c, dtype=torch.int64, device=device)
            self.vc_stats = torch.zeros(b, hk, 4, dtype=torch.int64, device=device)
            self.vc_slots = torch.zeros(b, hk, C + S.budget, dtype=torch.int64, device=device)

    @classmethod
    def from_tensors(cls, shape: Shape, device, **tensors) -> "LayerState":
        """A LayerState over caller-provided tensors (e.g. shard views, shard.shard_state); no allocation
        except the ragged-length arrays."""
        self = cls.__new__(cls)
        self.shape = shape
        bd.ensure_init(device)
        self.lens_host = self.lens_dev = None
        if shape.ctx_lens is not None:
            self.lens_host = torch.tensor(shape.ctx_lens, dtype=torch.int32)
            self.lens_dev = self.lens_host.to(device)
        for k in ("A", "B", "landmarks", "outlier_ids", "K_out", "V_out", "K_win", "V_win", "V_host", "A_gen",
                  "vc_values", "vc_dir", "vc_stats", "vc_slots"):
            setattr(self, k, tensors.get(k))
        self.vc_capacity = int(tensors.get("vc_capacity", 0))
        return self

    def layer(self) -> bd.SkvLayer:
        return bd.layer_struct(self.A, self.B, self.landmarks, self.outlier_ids, self.K_out, self.V_out,
                               self.K_win, self.V_win, self.V_host, self.vc_values, self.vc_dir, self.vc_stats,
                               self.A_gen, self.vc_slots, self.vc_capacity)

    def cache_stats(self):
        """-> int64 [b][h_kv][4] {generation, -, hits in the last step, hits in total} (synchronises)."""
        return None if self.vc_stats is None else self.vc_stats.cpu()

    def dims(self) -> bd.SkvDims:
        return self.shape.dims(self.lens_host, self.lens_dev)

    def build(self, rope: bd.SkvRope, workspace: torch.Tensor, K_rope: torch.Tensor | None = None, stream=None):
        bd.shadowkv_build_cache(self.dims(), rope, self.layer(), K_rope, ws_ptr(workspace), stream)

    def decode(self, rope: bd.SkvRope, q, k_new, v_new, step: int, out, workspace, sel_ids=None,
               dbg_keys=None, stream=None):
        bd.shadowkv_decode_step(self.dims(), rope, self.layer(), q, k_new, v_new, step, out, sel_ids,
                                dbg_keys, ws_ptr(workspace), stream)


    def decode_dev(self, rope: bd.SkvRope, q, k_new, v_new, step_dev, max_step: int, out, workspace,
                   sel_ids=None, dbg_keys=None, stream=None):
        """Graph-replayable decode: the step index is read on the device from step_dev (int32 tensor)."""
        bd.shadowkv_decode_step_dev(self.dims(), rope, self.layer(), q, k_new, v_new, step_dev, max_step, out,
                                    sel_ids, dbg_keys, ws_ptr(workspace), stream)


class RopeTable:
    """Device copy of the model's fp32 inv_freq table + layout flags (skv_rope)."""

    def __init__(self, inv_freq, rotary_dim: int, interleaved: bool, device="cuda"):
        self.inv_freq = torch.as_tensor(inv_freq, dtype=torch.float32).to(device).contiguous()
        self.rotary_dim, self.interleaved = int(rotary_dim), bool(interleaved)
        self.struct = bd.rope_struct(self.rotary_dim, self.interleaved, self.inv_freq)


def factorize(K_pre: torch.Tensor, rank: int, stream=None):
    """Alg 1 "A, B <- SVD(K)" on the GPU through shadowkv_factorize.
    K_pre: device bf16 [b][h_kv][s][d] -> (A bf16 [b][s][r], B bf16 [b][h_kv][r][d], sigma fp32 [b][r])."""
    b, hk, s, d = K_pre.shape
    bd.ensure_init(K_pre.device)
    dims = bd.dims_struct(b, hk, hk, d, s, rank, 8, 0, 1, 0, 1)
    n = bd.shadowkv_factorize_workspace_bytes(dims)
    ws = torch.empty(n + 256, dtype=torch.uint8, device=K_pre.device)
    A = torch.empty(b, s, rank, dtype=torch.bfloat16, device=K_pre.device)
    B = torch.empty(b, hk, rank, d, dtype=torch.bfloat16, device=K_pre.device)
    sigma = torch.empty(b, rank, dtype=torch.float32, device=K_pre.device)
    bd.shadowkv_factorize(dims, K_pre.contiguous(), A, B, sigma, ws_ptr(ws), stream)
    return A, B, sigma
