"""CPU oracle for ShadowKV's per-layer decode-time sparse attention (fp64, numpy).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_2410_21465_b200/``)
and imports nothing from it.

Every function follows PAPER.md (arXiv 2410.21465, LaTeX source) step by step;
"P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "Rn" = the reading register
in DESIGN.md (= SURVEY.md §8(c)).  All arithmetic is float64; bf16 inputs are
widened exactly.  ``store`` models where the product stores bf16: bf16
round-to-nearest-even in parity mode, the identity in self-check mode.

Pins (tests/test_oracle_*.py) tie each function to something other than itself:
closed forms, brute force on tiny inputs, library routines, the paper's 7.2 TB/s
worked example and the full-coverage == dense-attention equivalence.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "bf16_round", "identity_store", "partition", "rope", "chunk_means", "chunk_min_cos",
    "smallest_o", "build", "BuildState", "landmark_scores", "normalise_group_max",
    "arg_topk", "rebuild_keys", "decode_step", "dense_attention", "softmax_attention",
    "equivalent_bandwidth", "jacobi_svd", "ValueChunkCache", "replay_hits", "factorize", "normalise_sum_group_max", "lowrank_generated_keys",
]


# ----------------------------------------------------------------------------
# storage precision
# ----------------------------------------------------------------------------
def bf16_round(x):
    """Round float64 values to the nearest bfloat16 (ties to even), returned as float64.

    bf16 keeps 8 significant bits.  frexp gives x = m * 2**e with 0.5 <= |m| < 1;
    m * 2**8 is rounded half-to-even (np.rint) and scaled back.  Exact for the
    normal range (all values this path produces); no overflow handling needed.
    """
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)


def identity_store(x):
    """Self-check mode: no storage rounding (pure fp64)."""
    return np.asarray(x, dtype=np.float64)


# ----------------------------------------------------------------------------
# partition (R8) and RoPE (R15)
# ----------------------------------------------------------------------------
def partition(s: int, c: int, w: int):
    """R8: n_c = floor((s - w) / c) grid chunks; the window is [n_c*c, s), w_eff = s - n_c*c >= w."""
    n_c = (s - w) // c
    return n_c, s - n_c * c


def rope(x, pos, inv_freq, rotary_dim: int, interleaved: bool):
    """Rotary position embedding of rows ``x[..., T, d]`` at integer positions ``pos[T]``.

    Angle phi_{t,i} = fl32(fl32(t) * inv_freq[i]) (float32 product, as HF builds
    ``inv_freq (x) position``), cos/sin in float64 (R15).  Halves layout pairs
    (x_i, x_{i+rot/2}); interleaved layout pairs (x_{2i}, x_{2i+1}); dims >= rot
    pass through.  Rotation: (a, b) -> (a cos - b sin, b cos + a sin).
    """
    x = np.asarray(x, dtype=np.float64)
    pos = np.asarray(pos)
    half = rotary_dim // 2
    phi = (pos.astype(np.float32)[:, None] * np.asarray(inv_freq, dtype=np.float32)[None, :])
    phi = phi.astype(np.float32).astype(np.float64)           # [T][half]
    cos, sin = np.cos(phi), np.sin(phi)
    out = x.copy()
    if interleaved:
        a, b = x[..., 0:rotary_dim:2], x[..., 1:rotary_dim:2]
        out[..., 0:rotary_dim:2] = a * cos - b * sin
        out[..., 1:rotary_dim:2] = b * cos + a * sin
    else:
        a, b = x[..., :half], x[..., half:rotary_dim]
        out[..., :half] = a * cos - b * sin
        out[..., half:rotary_dim] = b * cos + a * sin
    return out


# ----------------------------------------------------------------------------
# Algorithm 1 (pre-filling)
# ----------------------------------------------------------------------------
def chunk_means(keys_grid, c: int):
    """Alg 1 "C <- Reduce(K^RoPE)": C_j = (1/c) sum_{t in chunk j} k_t.  keys_grid [n_c*c][d]."""
    n_c = keys_grid.shape[0] // c
    return keys_grid.reshape(n_c, c, -1).sum(axis=1) / c


def chunk_min_cos(keys_grid, means, c: int):
    """Alg 1 "S <- CosineSimilarity(C, K^RoPE)" then Min over the chunk.

    m_j = min_{t in j} <C_j, k_t> / (|C_j| |k_t|) with the unrounded mean and the
    token included in its own mean (R10, R11); a zero norm gives -1.
    """
    n_c = means.shape[0]
    k = keys_grid.reshape(n_c, c, -1)
    dots = np.einsum("jtd,jd->jt", k, means)
    nk = np.sqrt(np.einsum("jtd,jtd->jt", k, k))
    nc = np.sqrt(np.einsum("jd,jd->j", means, means))[:, None]
    den = nk * nc
    cos = np.where(den > 0, dots / np.where(den > 0, den, 1.0), -1.0)
    return cos.min(axis=1)


def smallest_o(m, o: int):
    """Alg 1 "I <- ArgTopK(-Min(S), o)": the o chunks with smallest m, ties -> lower j (R12), ascending."""
    order = np.lexsort((np.arange(len(m)), m))   # primary key m ascending, then index
    return np.sort(order[:o])


@dataclasses.dataclass
class BuildState:
    """Per-layer artefacts of Alg 1 for a batch (shapes as the C-ABI)."""
    n_c: int
    w_eff: int
    landmarks: np.ndarray     # [b][h_kv][n_c][d]  store(C) on the full chunk grid
    mincos: np.ndarray        # [b][h_kv][n_c]
    outlier_ids: np.ndarray   # [b][h_kv][o] ascending
    K_out: np.ndarray         # [b][h_kv][o*c][d]  store(post-RoPE keys) of outlier chunks
    V_out: np.ndarray         # [b][h_kv][o*c][d]  values of outlier chunks (exact copy)
    K_win: np.ndarray         # [b][h_kv][window_cap][d]
    V_win: np.ndarray         # [b][h_kv][window_cap][d]

    def copy(self):
        return dataclasses.replace(self, **{f.name: np.array(getattr(self, f.name), copy=True)
                                            for f in dataclasses.fields(self)
                                            if isinstance(getattr(self, f.name), np.ndarray)})


def build(A, B, V, inv_freq, rotary_dim, interleaved, c, o, w, window_cap, K_rope=None,
          store=bf16_round):
    """Algorithm 1 for every request b and KV head h.

    A [b][s][r], B [b][h_kv][r][d], V [b][h_kv][s][d], optional K_rope [b][h_kv][s][d].
    Post-RoPE keys are K_rope if given, else RoPE_t(A[t] . B_h) (the rank-r keys the
    factors represent; SVD itself is the caller's, R14).
    """
    A = np.asarray(A, np.float64); B = np.asarray(B, np.float64); V = np.asarray(V, np.float64)
    nb, s, r = A.shape
    hk, d = B.shape[1], B.shape[3]
    n_c, w_eff = partition(s, c, w)
    assert 0 <= o < n_c and window_cap >= w_eff
    L = np.zeros((nb, hk, n_c, d)); M = np.zeros((nb, hk, n_c))
    I = np.zeros((nb, hk, o), np.int64)
    Ko = np.zeros((nb, hk, o * c, d)); Vo = np.zeros((nb, hk, o * c, d))
    Kw = np.zeros((nb, hk, window_cap, d)); Vw = np.zeros((nb, hk, window_cap, d))
    pos = np.arange(s)
    for bi in range(nb):
        for h in range(hk):
            if K_rope is not None:
                keys = np.asarray(K_rope[bi, h], np.float64)
            else:
                keys = rope(A[bi] @ B[bi, h], pos, inv_freq, rotary_dim, interleaved)
            grid = keys[: n_c * c]
            C = chunk_means(grid, c)
            m = chunk_min_cos(grid, C, c)
            ids = smallest_o(m, o)
            L[bi, h] = store(C)
            M[bi, h] = m
            I[bi, h] = ids
            tok = (ids[:, None] * c + np.arange(c)[None, :]).reshape(-1)
            Ko[bi, h] = store(keys[tok])
            Vo[bi, h] = V[bi, h, tok]
            Kw[bi, h, :w_eff] = store(keys[n_c * c:])
            Vw[bi, h, :w_eff] = V[bi, h, n_c * c:]
    return BuildState(n_c, w_eff, L, M, I, Ko, Vo, Kw, Vw)


# ----------------------------------------------------------------------------
# Algorithm 2 (decoding)
# ----------------------------------------------------------------------------
def landmark_scores(q_group, L_h, d):
    """Alg 2 "P <- MatMul(Q, L^T)" scaled by 1/sqrt(d) (R6): [g][n_c]."""
    return (q_group @ L_h.T) / math.sqrt(d)


def normalise_group_max(logits, mask):
    """Alg 2 "S <- Softmax(P/sqrt d)", "S1 <- sum over s_q" (s_q = 1), "S2 <- max_kv_group(S1)".

    Works in the log domain: z_j = max_hq (l_{hq,j} - lse_hq) = log S2_j, where lse_hq is
    over the landmarks (mask True) only (R3, R4, R5).  Masked entries get -inf.
    """
    lg = np.where(mask[None, :], logits, -np.inf)
    mx = lg.max(axis=1, keepdims=True)
    lse = mx + np.log(np.exp(lg - mx).sum(axis=1, keepdims=True))
    z = (lg - lse).max(axis=0)
    return np.where(mask, z, -np.inf)


def normalise_sum_group_max(logits, mask):
    """Alg 2 with s_q >= 1 query tokens: logits [g][s_q][n_c];
    S = Softmax(P/sqrt d) per (q head, query token) over the landmarks, S1 = sum over s_q ("dim=-2"),
    S2 = max over the KV group.  Returns z = log S2 (masked -inf), computed literally in the
    probability domain (fp64): for s_q = 1 it equals normalise_group_max."""
    lg = np.where(mask[None, None, :], logits, -np.inf)
    mx = lg.max(axis=2, keepdims=True)
    S = np.exp(lg - mx)
    S = S / S.sum(axis=2, keepdims=True)
    S1 = S.sum(axis=1)
    S2 = S1.max(axis=0)
    with np.errstate(divide="ignore"):
        return np.where(mask, np.log(S2), -np.inf)


def arg_topk(z, k: int):
    """Alg 2 "I <- ArgTopK(S2, k)": k largest z, ties -> lower index (R12), returned ascending."""
    order = np.lexsort((np.arange(len(z)), -z))
    return np.sort(order[:k])


def rebuild_keys(A_b, B_h, tokens, inv_freq, rotary_dim, interleaved):
    """Alg 2 "K^sparse <- MatMul(Gather(A, I), B)" then RoPE at absolute positions."""
    return rope(A_b[tokens] @ B_h, tokens, inv_freq, rotary_dim, interleaved)


def softmax_attention(q, keys, values):
    """out = sum_t softmax_t(<q, k_t>/sqrt d) v_t, max-subtracted exp, summed in the given order."""
    a = keys @ q / math.sqrt(q.shape[-1])
    p = np.exp(a - a.max())
    return (p[:, None] * values).sum(axis=0) / p.sum()


def decode_step(state: BuildState, A, B, V, q, k_new, v_new, step, k, inv_freq, rotary_dim,
                interleaved, c, store=bf16_round, sel=None):
    """One decode step of Alg 2 + sparse attention (R17, R18).

    q [b][h_q][d] (s_q = 1) or [b][h_q][s_q][d] (Alg 2's Q, NEXT-3; k_new, v_new then
    [b][h_kv][s_q][d]).  Query token i sits at position s + step + i and attends causally to the
    new tokens 0..i (R28); the selection is shared by the s_q tokens (S1 = sum over s_q).
    state is NOT modified; returns (out [b][h_q][d] or [b][h_q][s_q][d], sel [b][h_kv][k],
    z [b][h_kv][n_c], rebuilt keys [b][h_kv][k*c][d] (unrounded), new_state with the window
    slots written).

    sel (optional, [b][h_kv][k] chunk ids): attend these chunks instead of ArgTopK's I (z is still
    computed and returned).  Test hook for R23: where the GPU's set differs from the oracle's only by
    a tie swap within 1e-5 (R1), keys and outputs are compared with the oracle evaluated on the GPU's
    set, which is the same algorithm after step "I <- ArgTopK".
    """
    if np.ndim(q) == 4:
        return _decode_step_multi(state, A, B, V, q, k_new, v_new, step, k, inv_freq, rotary_dim,
                                  interleaved, c, store, sel)
    given = sel
    A = np.asarray(A, np.float64); B = np.asarray(B, np.float64); V = np.asarray(V, np.float64)
    q = np.asarray(q, np.float64); k_new = np.asarray(k_new, np.float64)
    v_new = np.asarray(v_new, np.float64)
    st = state.copy()
    nb, s, _ = A.shape
    hk, d = B.shape[1], B.shape[3]
    hq_n = q.shape[1]
    g = hq_n // hk                         # R2: q head hq uses KV head floor(hq / g)
    n_c, w_eff = st.n_c, st.w_eff
    slot = w_eff + step
    assert slot < st.K_win.shape[2]
    # a7: the current token's K, V join the window before attention (R18)
    st.K_win[:, :, slot] = k_new
    st.V_win[:, :, slot] = v_new
    out = np.zeros((nb, hq_n, d)); sel = np.zeros((nb, hk, k), np.int64)
    Z = np.zeros((nb, hk, n_c)); Kt = np.zeros((nb, hk, k * c, d))
    o = st.outlier_ids.shape[2]
    for bi in range(nb):
        for h in range(hk):
            mask = np.ones(n_c, bool)
            mask[st.outlier_ids[bi, h]] = False          # L = C \ Gather(C, I)
            qg = q[bi, h * g:(h + 1) * g]
            logits = landmark_scores(qg, st.landmarks[bi, h], d)
            z = normalise_group_max(logits, mask)
            ids = arg_topk(z, k) if given is None else np.sort(np.asarray(given[bi][h], np.int64))
            tok = (ids[:, None] * c + np.arange(c)[None, :]).reshape(-1)
            kt = rebuild_keys(A[bi], B[bi, h], tok, inv_freq, rotary_dim, interleaved)
            vt = V[bi, h, tok]                           # Gather(V^CPU, I)
            Z[bi, h] = z; sel[bi, h] = ids; Kt[bi, h] = kt
            # assemble [outliers; sparse; window] and order by absolute position (R17)
            otok = (st.outlier_ids[bi, h][:, None] * c + np.arange(c)[None, :]).reshape(-1)
            wpos = np.array([n_c * c + j if j < w_eff else s + (j - w_eff) for j in range(slot + 1)],
                            dtype=np.int64)
            pos = np.concatenate([otok, tok, wpos])
            keys = np.concatenate([st.K_out[bi, h], kt, st.K_win[bi, h, :slot + 1]])
            vals = np.concatenate([st.V_out[bi, h], vt, st.V_win[bi, h, :slot + 1]])
            order = np.argsort(pos, kind="stable")
            keys, vals = keys[order], vals[order]
            for j in range(g):
                out[bi, h * g + j] = softmax_attention(qg[j], keys, vals)
    return out, sel, Z, Kt, st


def _decode_step_multi(state, A, B, V, q, k_new, v_new, step, k, inv_freq, rotary_dim, interleaved, c,
                       store, sel=None):
    """decode_step for s_q >= 1 query tokens (Alg 2 with Q in R^{b x h_q x s_q x d})."""
    given = sel
    A = np.asarray(A, np.float64); B = np.asarray(B, np.float64); V = np.asarray(V, np.float64)
    q = np.asarray(q, np.float64); k_new = np.asarray(k_new, np.float64)
    v_new = np.asarray(v_new, np.float64)
    st = state.copy()
    nb, s, _ = A.shape
    hk, d = B.shape[1], B.shape[3]
    hq_n, sq = q.shape[1], q.shape[2]
    g = hq_n // hk                         # R2
    n_c, w_eff = st.n_c, st.w_eff
    slot0 = w_eff + step
    assert slot0 + sq <= st.K_win.shape[2]
    for i in range(sq):                    # the s_q current tokens join the window (R18)
        st.K_win[:, :, slot0 + i] = k_new[:, :, i]
        st.V_win[:, :, slot0 + i] = v_new[:, :, i]
    out = np.zeros((nb, hq_n, sq, d)); sel = np.zeros((nb, hk, k), np.int64)
    Z = np.zeros((nb, hk, n_c)); Kt = np.zeros((nb, hk, k * c, d))
    for bi in range(nb):
        for h in range(hk):
            mask = np.ones(n_c, bool)
            mask[st.outlier_ids[bi, h]] = False
            qg = q[bi, h * g:(h + 1) * g]                               # [g][s_q][d]
            logits = np.stack([landmark_scores(qg[:, i], st.landmarks[bi, h], d) for i in range(sq)], axis=1)
            z = normalise_sum_group_max(logits, mask)
            ids = arg_topk(z, k) if given is None else np.sort(np.asarray(given[bi][h], np.int64))
            tok = (ids[:, None] * c + np.arange(c)[None, :]).reshape(-1)
            kt = rebuild_keys(A[bi], B[bi, h], tok, inv_freq, rotary_dim, interleaved)
            vt = V[bi, h, tok]
            Z[bi, h] = z; sel[bi, h] = ids; Kt[bi, h] = kt
            otok = (st.outlier_ids[bi, h][:, None] * c + np.arange(c)[None, :]).reshape(-1)
            for i in range(sq):
                last = slot0 + i                                        # causal among the new tokens
                wpos = np.array([n_c * c + j if j < w_eff else s + (j - w_eff) for j in range(last + 1)],
                                dtype=np.int64)
                pos = np.concatenate([otok, tok, wpos])
                keys = np.concatenate([st.K_out[bi, h], kt, st.K_win[bi, h, :last + 1]])
                vals = np.concatenate([st.V_out[bi, h], vt, st.V_win[bi, h, :last + 1]])
                order = np.argsort(pos, kind="stable")
                for j in range(g):
                    out[bi, h * g + j, i] = softmax_attention(qg[j, i], keys[order], vals[order])
    return out, sel, Z, Kt, st


def lowrank_generated_keys(k_pre, B, positions, inv_freq, rotary_dim, interleaved, store=bf16_round):
    """Low-rank storage of generated keys (P:196 footnote): "new pre-RoPE keys K' can be
    stored as K' Psi and projected back with Psi^T when needed", Psi = the right singular matrix of the
    context's pre-RoPE keys.  With the heads concatenated (R14) Psi[(h, j), rho] = B_h[rho, j], so the
    stored state of a generated token is one rank-r row a = sum_h k'_h B_h^T (like a row of A), kept
    at storage precision, and the key attended is RoPE_t(a B_h) at the token's position t.
    k_pre [b][h_kv][n][d] (n generated tokens), B [b][h_kv][r][d], positions [n].
    Returns (a [b][n][r] as stored, keys [b][h_kv][n][d] post-RoPE, unrounded)."""
    k_pre = np.asarray(k_pre, np.float64); B = np.asarray(B, np.float64)
    nb, hk, n, d = k_pre.shape
    a = store(np.einsum("bhnd,bhrd->bnr", k_pre, B))
    keys = np.zeros((nb, hk, n, d))
    for bi in range(nb):
        for h in range(hk):
            keys[bi, h] = rope(a[bi] @ B[bi, h], np.asarray(positions), inv_freq, rotary_dim, interleaved)
    return a, keys


# ----------------------------------------------------------------------------
# references used by the pins
# ----------------------------------------------------------------------------
def dense_attention(q, keys, values):
    """Dense GQA attention (textbook, double loop): q [h_q][d], keys/values [h_kv][T][d]."""
    hq_n, d = q.shape
    hk = keys.shape[0]
    g = hq_n // hk
    out = np.zeros((hq_n, d))
    for hq in range(hq_n):
        h = hq // g
        a = np.array([float(np.dot(q[hq], keys[h, t])) for t in range(keys.shape[1])]) / math.sqrt(d)
        p = np.exp(a - a.max())
        p /= p.sum()
        for t in range(keys.shape[1]):
            out[hq] += p[t] * values[h, t]
    return out


# ----------------------------------------------------------------------------
# value-chunk cache with temporal locality
# ----------------------------------------------------------------------------
class ValueChunkCache:
    """GPU-resident cache of selected value chunks for one (request, layer, KV head).

    P:105 "considering the temporal locality of the KV cache, a cache policy can be leveraged";
    P:156 "we conduct an index scan to detect the missed chunks and only rebuild the necessary KV
    pairs".  The paper names no policy (it cites PQCache); SPEC S:139-146, S:158 fix it as
    least-recently-SELECTED replacement at chunk granularity with capacity defaulting to the budget
    k (DESIGN reading R26).  ``fetch`` follows S:139-143 literally: the hit flags are true exactly for
    the ids resident before the call; every requested id becomes most recent; the misses are
    inserted in ascending id order, evicting least-recently-selected chunks while over capacity.
    Values themselves are bit copies of V rows ("round-trip fidelity"), so only the hit
    pattern is modelled here.
    """

    def __init__(self, capacity: int):
        self.capacity = int(capacity)
        self.last_use = {}            # chunk id -> call index of its last selection
        self.calls = 0
        self.hits = 0
        self.requested = 0

    def fetch(self, ids):
        ids = [int(i) for i in ids]
        assert len(set(ids)) == len(ids), "duplicate chunk id in one fetch"
        hit = np.array([i in self.last_use for i in ids], dtype=bool)
        t = self.calls
        self.calls += 1
        for i in sorted(ids):                        # every requested chunk is now most recent
            self.last_use[i] = t
        while len(self.last_use) > self.capacity:    # evict least recently selected (ties: lower id)
            victim = min(self.last_use, key=lambda j: (self.last_use[j], j))
            del self.last_use[victim]
        self.hits += int(hit.sum())
        self.requested += len(ids)
        return hit

    def hit_rate(self) -> float:
        return self.hits / self.requested if self.requested else 0.0


def replay_hits(trace, capacity: int):
    """Per-step hit counts of a selection trace [steps][k] through one ValueChunkCache."""
    cache = ValueChunkCache(capacity)
    return np.array([int(cache.fetch(ids).sum()) for ids in trace], dtype=np.int64)


def equivalent_bandwidth(S, C, K, O, alpha, B_gpu, B_pcie):
    """Sec 4.2: B_eq = 2 S B_GPU / (S/C + 2(K+O)C + (1-alpha) K C B_GPU / B_PCIe)."""
    return 2.0 * S * B_gpu / (S / C + 2.0 * (K + O) * C + (1.0 - alpha) * K * C * B_gpu / B_pcie)


def factorize(K_pre, r: int, svd=None):
    """Alg 1 "A in R^{b x s x r}, B in R^{b x h_kv x r x d} <- SVD(K)", per request.

    K_pre [b][h_kv][s][d] pre-RoPE keys.  Per request the keys of all KV heads are concatenated per
    token, X[t, h*d + j] = K[h][t][j] (R14), X = U Sigma V^T, and the rank-r truncation is
    split as A = U_r Sigma_r (shared across heads) and B_h = (V_r^T)[:, h*d:(h+1)*d].
    ``svd`` defaults to LAPACK (numpy) as the step; the pins also run it with ``jacobi_svd``.
    Returns (A [b][s][r], B [b][h_kv][r][d], sigma [b][min(s, h_kv*d)] descending).
    """
    K = np.asarray(K_pre, dtype=np.float64)
    nb, hk, s, d = K.shape
    A = np.zeros((nb, s, r)); B = np.zeros((nb, hk, r, d))
    sig_all = np.zeros((nb, min(s, hk * d)))
    for bi in range(nb):
        X = K[bi].transpose(1, 0, 2).reshape(s, hk * d)
        if svd is None:
            U, sig, Vt = np.linalg.svd(X, full_matrices=False)
        else:
            U, sig, Vt = svd(X)
        A[bi] = U[:, :r] * sig[:r]
        B[bi] = Vt[:r].reshape(r, hk, d).transpose(1, 0, 2)
        sig_all[bi] = sig[:min(s, hk * d)]
    return A, B, sig_all


def jacobi_svd(X, sweeps: int = 60, tol: float = 1e-15):
    """One-sided (Hestenes) Jacobi SVD: X = U diag(sig) Vt, sig descending.

    Used for Alg 1's "A, B <- SVD(K)" only in the rank pins; A = U Sigma, B = Vt.
    """
    X = np.array(X, dtype=np.float64, copy=True)
    m, n = X.shape
    W = X.copy()
    Vm = np.eye(n)
    for _ in range(sweeps):
        off = 0.0
        for p in range(n - 1):
            for q_ in range(p + 1, n):
                a = W[:, p] @ W[:, p]; b = W[:, q_] @ W[:, q_]; cpq = W[:, p] @ W[:, q_]
                if abs(cpq) <= tol * math.sqrt(a * b) or cpq == 0.0:
                    continue
                off = max(off, abs(cpq) / math.sqrt(a * b))
                zeta = (b - a) / (2.0 * cpq)
                t = math.copysign(1.0, zeta) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                cs = 1.0 / math.sqrt(1.0 + t * t); sn = cs * t
                wp = W[:, p].copy(); W[:, p] = cs * wp - sn * W[:, q_]; W[:, q_] = sn * wp + cs * W[:, q_]
                vp = Vm[:, p].copy(); Vm[:, p] = cs * vp - sn * Vm[:, q_]; Vm[:, q_] = sn * vp + cs * Vm[:, q_]
        if off < tol:
            break
    sig = np.sqrt((W * W).sum(axis=0))
    order = np.argsort(-sig, kind="stable")
    sig = sig[order]; W = W[:, order]; Vm = Vm[:, order]
    U = np.where(sig[None, :] > 0, W / np.where(sig > 0, sig, 1.0)[None, :], 0.0)
    return U, sig, Vm.T
