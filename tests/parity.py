"""Helpers for GPU-vs-oracle parity tests (tolerances are DESIGN.md §Parity; R1, R13, R23)."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import shadowkv_oracle as O

Z_TIE_TOL = 1e-5      # north_star: "bit-exact, except for score ties within 1e-5" (log-domain z, R1)
M_TIE_TOL = 1e-5      # same rule for the outlier ranking on min-cos m (R12)
OUT_TOL = 2e-2        # north_star: outputs within 2e-2 max-abs
KEY_REL_TOL = 1e-2    # north_star: rebuilt keys within 1e-2 relative (per-row L2, R23)


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def bf16_ulp(x: np.ndarray) -> np.ndarray:
    """Spacing of bf16 numbers at |x| (8 significant bits)."""
    ax = np.abs(x)
    e = np.floor(np.log2(np.where(ax > 0, ax, 1.0)))
    return np.where(ax > 0, 2.0 ** (e - 7), 2.0 ** -133)


def assert_bf16_close(got: np.ndarray, want: np.ndarray, abs_slack: float = 2e-6, what: str = ""):
    """<= 1 bf16 ulp (+ fp32-accumulation slack): GPU rounds an fp32 value, the oracle an fp64 one (R13)."""
    tol = bf16_ulp(np.maximum(np.abs(got), np.abs(want))) + abs_slack
    bad = np.abs(got - want) > tol
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} elements off by > 1 ulp; max diff " \
                          f"{np.abs(got - want).max():.3g}"


def selection_valid(gpu_ids: np.ndarray, z: np.ndarray, k: int, tol: float = Z_TIE_TOL) -> bool:
    """R1: GPU set G (|G| = k, distinct, ascending) is valid iff every member scores within tol of the
    oracle's k-th largest z (so any difference from the oracle set is a tie swap)."""
    g = np.asarray(gpu_ids)
    if len(g) != k or len(set(g.tolist())) != k or np.any(np.diff(g) <= 0):
        return False
    thr = np.sort(z)[::-1][k - 1]
    return bool(np.all(np.isfinite(z[g])) and np.all(z[g] >= thr - tol))


def outliers_valid(gpu_ids: np.ndarray, m: np.ndarray, o: int, tol: float = M_TIE_TOL) -> bool:
    g = np.asarray(gpu_ids)
    if o == 0:
        return True
    if len(set(g.tolist())) != o or np.any(np.diff(g) <= 0):
        return False
    thr = np.sort(m)[o - 1]
    return bool(np.all(m[g] <= thr + tol))


class Problem:
    """Seeded synthetic inputs for one layer (synth), the GPU state and the oracle state."""

    def __init__(self, cfg: synth.Config, seed: int, steps: int = 4, K_rope: bool = False, device="cuda",
                 value_cache: bool = False, q_len: int = 1, lowrank_gen: bool = False, vc_capacity: int = 0):
        from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace
        self.cfg, self.seed, self.steps = cfg, seed, steps
        self.inputs = synth.gen_layer(cfg, seed)
        self.inv, self.rot, self.il = synth.rope_table(cfg)
        self.q_len = q_len
        self.shape = Shape.from_config(cfg, steps=steps, q_len=q_len)
        self.st = LayerState(self.shape, device=device, value_cache=value_cache, lowrank_gen=lowrank_gen,
                             vc_capacity=vc_capacity)
        self.st.A.copy_(self.inputs["A"]); self.st.B.copy_(self.inputs["B"])
        self.st.V_host.copy_(self.inputs["V"])
        self.rope = RopeTable(self.inv, self.rot, self.il, device=device)
        self.ws = alloc_workspace(self.shape, device=device)
        self.K_rope = None
        if K_rope:   # given post-RoPE keys: independent random keys (not low rank)
            g = torch.Generator().manual_seed(synth.stream_seed(seed, 77))
            self.K_rope = torch.randn(cfg.batch, cfg.n_kv_heads, cfg.ctx_len, cfg.head_dim, generator=g).to(torch.bfloat16)
        self.A64, self.B64, self.V64 = f64(self.inputs["A"]), f64(self.inputs["B"]), f64(self.inputs["V"])

    def gpu_build(self):
        kr = self.K_rope.cuda() if self.K_rope is not None else None
        self.st.build(self.rope.struct, self.ws, K_rope=kr)
        torch.cuda.synchronize()

    def oracle_build(self, store=O.bf16_round):
        c = self.cfg
        return O.build(self.A64, self.B64, self.V64, self.inv, self.rot, self.il, c.chunk, c.n_outlier,
                       c.window_ctx, self.shape.window_cap,
                       K_rope=f64(self.K_rope) if self.K_rope is not None else None, store=store)

    def load_state_from_oracle(self, ost):
        """Feed the oracle's build output to the GPU as decode input (identical state bytes)."""
        bf = torch.bfloat16
        self.st.landmarks.copy_(torch.from_numpy(ost.landmarks).to(bf))
        if self.cfg.n_outlier:
            self.st.outlier_ids.copy_(torch.from_numpy(ost.outlier_ids).to(torch.int32))
            self.st.K_out.copy_(torch.from_numpy(ost.K_out).to(bf))
            self.st.V_out.copy_(torch.from_numpy(ost.V_out).to(bf))
        self.st.K_win.copy_(torch.from_numpy(ost.K_win).to(bf))
        self.st.V_win.copy_(torch.from_numpy(ost.V_win).to(bf))

    def step_inputs(self, step):
        """One decode call's inputs; with q_len > 1 the tokens of steps step..step+q_len-1 stacked as
        Alg 2's Q [b][h_q][s_q][d], K, V [b][h_kv][s_q][d]."""
        if self.q_len == 1:
            return synth.gen_step(self.cfg, self.seed, 0, step)
        toks = [synth.gen_step(self.cfg, self.seed, 0, step + i) for i in range(self.q_len)]
        return {n: torch.stack([t[n] for t in toks], dim=2) for n in ("q", "k_new", "v_new")}

    def gpu_decode(self, step, si, st=None):
        c, b = self.cfg, self.cfg.batch
        dev = "cuda"
        st = self.st if st is None else st
        out = torch.empty(si["q"].shape, dtype=torch.bfloat16, device=dev)
        sel = torch.empty(b, c.n_kv_heads, c.budget, dtype=torch.int32, device=dev)
        dbg = torch.empty(b, c.n_kv_heads, c.budget * c.chunk, c.head_dim, dtype=torch.bfloat16, device=dev)
        st.decode(self.rope.struct, si["q"].to(dev), si["k_new"].to(dev), si["v_new"].to(dev), step, out,
                  self.ws, sel_ids=sel, dbg_keys=dbg)
        torch.cuda.synchronize()
        return f64(out), sel.cpu().numpy(), f64(dbg)

    def oracle_decode(self, ost, step, si, store=O.bf16_round, sel=None):
        c = self.cfg
        return O.decode_step(ost, self.A64, self.B64, self.V64, f64(si["q"]), f64(si["k_new"]), f64(si["v_new"]),
                             step, c.budget, self.inv, self.rot, self.il, c.chunk, store=store, sel=sel)

    def check(self, ost, step, si, gpu):
        """GPU decode result `gpu` = (out, sel, keys) of this step vs the oracle from state `ost` (R1, R23);
        returns (exact head count, the oracle's next state)."""
        gout, gsel, gkeys = gpu
        oout, osel, oz, okeys, nst = self.oracle_decode(ost, step, si)
        exact = check_decode(self.cfg, gout, gsel, gkeys, oout, osel, oz, okeys,
                             rerun=lambda sel: self.oracle_decode(ost, step, si, sel=sel))
        return exact, nst


def check_decode(cfg, gout, gsel, gkeys, oout, osel, oz, okeys, rerun=None):
    """Every head: the GPU's selection is the oracle's or a valid tie swap of it (R1); the rebuilt keys
    (per-row relative L2 <= 1e-2) and the outputs (max-abs <= 2e-2) are compared on EVERY head (R23):
    against the oracle's own results where the sets are equal, else against the oracle evaluated on the
    GPU's set -- rerun(gsel) -> oracle.decode_step(..., sel=gsel)'s tuple, from the same prior state.
    Returns the number of heads whose selection equals the oracle's exactly."""
    b, hk, g = cfg.batch, cfg.n_kv_heads, cfg.n_q_heads // cfg.n_kv_heads
    exact = 0
    for bi in range(b):
        for h in range(hk):
            assert selection_valid(gsel[bi, h], oz[bi, h], cfg.budget), \
                f"invalid selection b={bi} h={h}: gpu {gsel[bi, h][:8]}.. oracle {osel[bi, h][:8]}.."
            exact += int(np.array_equal(gsel[bi, h], osel[bi, h]))
    if exact < b * hk:
        assert rerun is not None, f"{b * hk - exact} tie-swapped head(s): pass rerun= to compare them"
        r = rerun(gsel)
        oout_g, okeys_g = r[0], r[3]
    for bi in range(b):
        for h in range(hk):
            same = np.array_equal(gsel[bi, h], osel[bi, h])
            ko = okeys[bi, h] if same else okeys_g[bi, h]
            oo = oout if same else oout_g
            kg = gkeys[bi, h]
            rel = np.linalg.norm(kg - ko, axis=1) / np.maximum(np.linalg.norm(ko, axis=1), 1e-6)
            assert rel.max() <= KEY_REL_TOL, f"rebuilt keys rel err {rel.max():.3g} (b={bi} h={h}, same set {same})"
            err = np.abs(gout[bi, h * g:(h + 1) * g] - oo[bi, h * g:(h + 1) * g]).max()
            assert err <= OUT_TOL, f"output max-abs {err:.3g} > {OUT_TOL} (b={bi} h={h}, same set {same})"
    return exact
