"""Seeded synthetic inputs for ShadowKV decode (the ONLY module both sides share).

This module holds no arithmetic of the method: it draws the raw inputs that
PAPER.md Alg. 1 / Alg. 2 take -- the low-rank
pre-RoPE factors A, B, the values V, the query q and the current-token K, V --
plus the model's RoPE frequency table (model configuration, not the paper's
method).  The oracle (``oracle/``), the CUDA path's tests and ``bench.py`` all
consume the same bytes from here.

Recipe:
  * A [b][s][r]: stationary AR(1) walk over token index t with rho = 0.9 per
    rank channel (adjacent-token similarity, PAPER.md:103 and Fig. 3b), drawn
    as its truncated MA(inf) form with 256 taps (rho^256 ~ 2e-12), unit
    variance.  In ~0.3 % of 8-token chunks one token is replaced by an
    independent N(0, I) draw (planted outliers).
  * B [b][h_kv][r][d]: N(0, 1/r)  -> key entries ~ unit variance.
  * V [b][h_kv][s][d]: N(0, 1).
  * q [b][h_q][d]: N(0, tau^2), tau = 2.  k_new, v_new [b][h_kv][d]: N(0, 1).
  * Temporally correlated queries (value-cache runs, DESIGN R27): q_t = rho q_{t-1} +
    sqrt(1 - rho^2) tau eps_t per (request, q head), stationary N(0, tau^2) marginals; rho sets
    how much consecutive selections overlap (the paper's Fig 3c hit rate).
  * Everything is rounded to bf16 once.
  * RoPE tables: Llama-3.1 (base 5e5, llama3 scaling, halves layout, full d)
    for the Llama shapes; GLM-4 (rotary_dim 64, interleaved, base 1e4*1e4).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

__all__ = ["Config", "CONFIGS", "rope_table", "gen_layer", "gen_step", "gen_q_drift", "stream_seed"]


@dataclasses.dataclass(frozen=True)
class Config:
    """Raw workload numbers of one BASELINE.json config."""
    name: str
    batch: int          # requests per GPU
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ctx_len: int        # s
    rank: int           # r
    chunk: int          # c
    n_outlier: int      # o
    budget: int         # k (selected chunks per KV head)
    window_ctx: int     # w (context tail kept exact)
    n_layers: int
    rope: str           # "llama3" | "glm"

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: single layer, 4K (oracle in seconds)
    "c1": Config("c1", 1, 32, 8, 128, 4096, 160, 8, 4, 8, 16, 1, "llama3"),
    # configs[1]: Llama-3.1-8B shape, 32 layers, batch 1, 128K, 1 B200 (the bench workload)
    "c2": Config("c2", 1, 32, 8, 128, 131072, 160, 8, 48, 256, 16, 32, "llama3"),
    # configs[2]: batch 64 x 122K (124928 = 122*1024), split by batch over GPUs
    "c3": Config("c3", 64, 32, 8, 128, 124928, 160, 8, 48, 244, 16, 32, "llama3"),
    # configs[3]: Llama-3-8B-1M, 1M context, one request per GPU
    "c4": Config("c4", 1, 32, 8, 128, 1048576, 160, 8, 48, 2048, 16, 32, "llama3"),
    # configs[4]: GLM-4-9B-1M shape (32 q / 2 KV heads), 256K, 12 requests per GPU
    "c5": Config("c5", 12, 32, 2, 128, 262144, 160, 8, 48, 512, 16, 40, "glm"),
}


def stream_seed(seed: int, *keys: int) -> int:
    """Deterministic 63-bit seed for an independent stream (splitmix64 chain)."""
    x = (seed * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    for k in keys:
        x = (x ^ ((k + 0x632BE59BD9B4E019) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        x = z ^ (z >> 31)
    return x & 0x7FFFFFFFFFFFFFFF


def rope_table(cfg: Config):
    """Model RoPE configuration -> (inv_freq fp32 [rotary_dim/2], rotary_dim, interleaved).

    Llama-3.1 "llama3" rope scaling (factor 8, low 1, high 4, original 8192,
    base 500000) and GLM-4-9B-1M (rotary_dim = head_dim/2, interleaved pairs,
    base 10000 * rope_ratio 10000).  These are model configs (PAPER.md is
    silent); both sides receive this exact fp32 table.
    """
    d = cfg.head_dim
    if cfg.rope == "llama3":
        rot = d
        base, factor, lo, hi, orig = 500000.0, 8.0, 1.0, 4.0, 8192.0
        inv = 1.0 / (base ** (np.arange(0, rot, 2, dtype=np.float64) / rot))
        wavelen = 2.0 * math.pi / inv
        lo_wl, hi_wl = orig / lo, orig / hi
        out = np.where(wavelen > lo_wl, inv / factor, inv)
        smooth = (orig / wavelen - lo) / (hi - lo)
        smoothed = (1.0 - smooth) * out / factor + smooth * out
        medium = (wavelen >= hi_wl) & (wavelen <= lo_wl)
        out = np.where(medium, smoothed, out)
        return out.astype(np.float32), rot, False
    if cfg.rope == "glm":
        rot = d // 2
        base = 10000.0 * 10000.0
        inv = 1.0 / (base ** (np.arange(0, rot, 2, dtype=np.float64) / rot))
        return inv.astype(np.float32), rot, True
    if cfg.rope == "plain":  # textbook base-10000 table, halves layout (tests)
        rot = d
        inv = 1.0 / (10000.0 ** (np.arange(0, rot, 2, dtype=np.float64) / rot))
        return inv.astype(np.float32), rot, False
    raise ValueError(cfg.rope)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _ar1_rows(n_rows: int, width: int, rho: float, g: torch.Generator, device) -> torch.Tensor:
    """Stationary AR(1) rows (unit variance) via the 256-tap truncated MA(inf) form."""
    taps = 256
    eps = torch.randn(width, n_rows + taps - 1, generator=g, device=device, dtype=torch.float32)
    w = (math.sqrt(1.0 - rho * rho) * rho ** torch.arange(taps - 1, -1, -1, dtype=torch.float64))
    w = w.to(device=device, dtype=torch.float32).view(1, 1, taps).expand(width, 1, taps).contiguous()
    out = torch.nn.functional.conv1d(eps.unsqueeze(0), w, groups=width).squeeze(0)  # [width][n_rows]
    return out.t().contiguous()


def gen_layer(cfg: Config, seed: int, layer: int = 0, device="cpu", batch: int | None = None,
              outlier_frac: float = 0.003):
    """Draw one layer's prefill-side inputs for ``batch`` requests.

    Returns dict of bf16 tensors on ``device``: A [b][s][r], B [b][h_kv][r][d],
    V [b][h_kv][s][d].  (The caller moves V to pinned host memory.)
    """
    b = cfg.batch if batch is None else batch
    s, r, d, hk, c = cfg.ctx_len, cfg.rank, cfg.head_dim, cfg.n_kv_heads, cfg.chunk
    A = torch.empty(b, s, r, dtype=torch.bfloat16, device=device)
    B = torch.empty(b, hk, r, d, dtype=torch.bfloat16, device=device)
    V = torch.empty(b, hk, s, d, dtype=torch.bfloat16, device=device)
    for i in range(b):
        g = _gen(stream_seed(seed, layer, i, 1), device)
        a = _ar1_rows(s, r, 0.9, g, device)
        n_ch = s // c
        n_plant = max(1, int(round(outlier_frac * n_ch)))
        ch = torch.randperm(n_ch, generator=g, device=device)[:n_plant]
        off = torch.randint(0, c, (n_plant,), generator=g, device=device)
        a[ch * c + off] = torch.randn(n_plant, r, generator=g, device=device)
        A[i] = a.to(torch.bfloat16)
        B[i] = (torch.randn(hk, r, d, generator=g, device=device) / math.sqrt(r)).to(torch.bfloat16)
        V[i] = torch.randn(hk, s, d, generator=g, device=device).to(torch.bfloat16)
    return {"A": A, "B": B, "V": V}


def gen_step(cfg: Config, seed: int, layer: int = 0, step: int = 0, device="cpu",
             batch: int | None = None, tau: float = 2.0):
    """Draw one decode step's inputs: q [b][h_q][d] (post-RoPE), k_new/v_new [b][h_kv][d]."""
    b = cfg.batch if batch is None else batch
    g = _gen(stream_seed(seed, layer, step, 2), device)
    q = (tau * torch.randn(b, cfg.n_q_heads, cfg.head_dim, generator=g, device=device)).to(torch.bfloat16)
    kn = torch.randn(b, cfg.n_kv_heads, cfg.head_dim, generator=g, device=device).to(torch.bfloat16)
    vn = torch.randn(b, cfg.n_kv_heads, cfg.head_dim, generator=g, device=device).to(torch.bfloat16)
    return {"q": q, "k_new": kn, "v_new": vn}


def gen_q_drift(cfg: Config, seed: int, layer: int, steps: int, rho: float, device="cpu",
                batch: int | None = None, tau: float = 2.0) -> torch.Tensor:
    """Queries of ``steps`` consecutive decode steps as a stationary AR(1) process over the step
    index (fp32, rounded to bf16 once): q_0 ~ N(0, tau^2); q_t = rho q_{t-1} + sqrt(1-rho^2) tau eps_t.
    Returns bf16 [steps][b][h_q][d].  rho = 0 gives independent queries (like gen_step's)."""
    b = cfg.batch if batch is None else batch
    g = _gen(stream_seed(seed, layer, 3), device)
    shape = (b, cfg.n_q_heads, cfg.head_dim)
    out = torch.empty((steps,) + shape, dtype=torch.bfloat16, device=device)
    cur = tau * torch.randn(shape, generator=g, device=device)
    for t in range(steps):
        if t:
            cur = rho * cur + math.sqrt(1.0 - rho * rho) * tau * torch.randn(shape, generator=g, device=device)
        out[t] = cur.to(torch.bfloat16)
    return out
