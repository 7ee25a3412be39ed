#!/usr/bin/env python
"""ShadowKV decode-time sparse attention on B200: decode tokens/s at 128K (BASELINE.json configs[1]).

One "step" = one decode step of the whole hot path (score, select, key
rebuild + RoPE, host value gather, sparse attention) for every layer of the model, i.e. 32
calls of shadowkv_decode_step over 32 distinct layer states (Llama-3.1-8B shape, batch 1, 128K
context, rank 160, chunk 8, 48 outliers, k = 256 = 1.56 %).  tokens/s = batch * n_gpus /
step_time (attention path only; QKV/MLP/weights are outside the path -- DESIGN.md §Measurement).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Multi-GPU (torchrun, one process per GPU): every rank runs its own requests (weak scaling, no
data-path collective); NCCL is used only for the start barrier and the max-over-ranks time.
--impl reference times the CPU oracle (oracle/, fp64 numpy) on a bounded sample of the same
workload (one layer of one request per step), extrapolated to the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "decode tokens/s at 128K ctx, 1.56% budget, 1/2/4/8 B200; % of HBM/host roofline"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--breakdown", action="store_true", help="extra untimed pass timing every kernel")
    ap.add_argument("--graph", choices=["on", "off"], default="on",
                    help="time CUDA-graph replays of the 32-layer step (shadowkv_decode_step_dev, device-side step "
                         "counter) instead of per-call stream launches")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: every rank runs the config's batch; strong: the batch is split over ranks "
                         "(default: strong for c3, whose 64 requests SURVEY 8(d) splits 64/n, weak otherwise)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: gloo process group, shard plan and max-over-ranks timing of an empty step "
                         "(tests the multi-rank launch path on CPU)")
    ap.add_argument("--vc-rho", default="0.95",
                    help="value-cache leg (P:156, DESIGN R26/R27): comma list of query-drift correlations rho; "
                         "each runs the same step with a GPU value cache per layer and drifting queries and "
                         "reports the measured hit rate alpha ('' = skip)")
    ap.add_argument("--vc-capacity", default="1,4",
                    help="value-cache legs: comma list of capacities in units of the budget k (C = m * k chunks per "
                         "request and KV head; least-recently-selected replacement, DESIGN R26)")
    ap.add_argument("--q-len-leg", type=int, default=4,
                    help="multi-query leg (NEXT-3, Alg 2's s_q): the same 32-layer step with s_q query tokens per "
                         "call (speculative verification); 0 = skip")
    ap.add_argument("--lowrank-gen-leg", type=int, default=1,
                    help="low-rank generated keys leg (NEXT-4, P:196): the same step with skv_layer.A_gen; 0 = skip")
    ap.add_argument("--layer-states", type=int, default=0,
                    help="distinct layer states cycled per step (default: the model's layer count)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


MODEL_SHAPE = {"c1": "Llama-3.1-8B-shape (one layer)", "c2": "Llama-3.1-8B-shape", "c3": "Llama-3.1-8B-shape",
               "c4": "Llama-3-8B-1M-shape", "c5": "GLM-4-9B-1M-shape (32 q / 2 KV heads)"}


def workload_config(cfg: synth.Config, n_gpus: int) -> dict:
    shape = MODEL_SHAPE.get(cfg.name, f"{cfg.n_q_heads} q / {cfg.n_kv_heads} KV heads")
    return {"workload": f"{cfg.name}: {shape} decode attention, {cfg.n_layers} layers, batch "
                        f"{cfg.batch}/GPU, {cfg.ctx_len} ctx, rank {cfg.rank}, chunk {cfg.chunk}, "
                        f"{cfg.n_outlier} outlier chunks, k={cfg.budget} chunks (1.56%), window {cfg.window_ctx}",
            "n_q_heads": cfg.n_q_heads, "n_kv_heads": cfg.n_kv_heads, "head_dim": cfg.head_dim,
            "ctx_len": cfg.ctx_len, "layers": cfg.n_layers, "batch_per_gpu": cfg.batch,
            "global_batch": cfg.batch * n_gpus, "parallelism": f"requests sharded over {n_gpus} GPU(s), no collective",
            "l2": "inputs > L2: `layer_states` distinct layer states (c2: 32 = ~2.5 GB HBM + 8.6 GB pinned host) cycled every step",
            "values": "offloaded to pinned host DRAM, gathered zero-copy over PCIe each step"}


# ------------------------------------------------------------------------------------------------
# clocks (NVML) sampled during the timed region
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clocks_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "no samples")}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------
def bind_to_gpu_numa(local: int) -> str:
    """Restrict this process to the CPUs NVML reports as local to its GPU, so that the pinned value
    pool is first-touched (allocated) on that NUMA node and the host->GPU reads stay node-local."""
    try:
        import pynvml
        pynvml.nvmlInit()
        pr = torch.cuda.get_device_properties(local)        # NVML index != CUDA index under CUDA_VISIBLE_DEVICES
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus and cpus != set(range(os.cpu_count())):
            os.sched_setaffinity(0, cpus)
            return f"bound to {len(cpus)} GPU-local CPUs"
        return "all CPUs GPU-local"
    except Exception as e:                       # no NVML / no affinity info: leave it to the OS
        return f"unbound ({type(e).__name__})"


def pinned_pool(nbytes: int) -> torch.Tensor:
    """One page-locked, device-mapped host buffer (cudaHostRegister portable|mapped)."""
    buf = torch.empty(nbytes // 2, dtype=torch.bfloat16)
    err = torch.cuda.cudart().cudaHostRegister(buf.data_ptr(), buf.numel() * 2, 3)
    if int(err) != 0:
        raise RuntimeError(f"cudaHostRegister failed: {err}")
    return buf


def measure_dma_h2d(pool: torch.Tensor, world: int = 1):
    """Pinned host->device copy-engine bandwidth B_host(n), 1 GiB, best of 6 (GB/s).  With n ranks every
    rank copies at the same time (a barrier before each repetition), so the figure is the per-GPU
    bandwidth while all n GPUs pull from host DRAM concurrently; returns
    (this rank's GB/s, every rank's GB/s)."""
    n = min(pool.numel(), 1 << 29)
    src = pool[:n]
    dst = torch.empty(n, dtype=pool.dtype, device="cuda")
    best = 1e30
    for _ in range(6):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dst.copy_(src, non_blocking=True); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del dst
    own = n * 2 / best / 1e6
    if world > 1:
        t = torch.zeros(world, dtype=torch.float64, device="cuda")
        t[torch.distributed.get_rank()] = own
        torch.distributed.all_reduce(t)
        return own, [float(x) for x in t.cpu()]
    return own, [own]


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6553.3), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:  # noqa: BLE001
            return {}
    return {}


def cpu_baseline(cfg: synth.Config, seed: int, budget_s: float = 15.0):
    """The oracle as it stands, timed on the host cores: decode of ONE layer of ONE request of the
    workload, repeated for ~budget_s; extrapolated x n_layers x batch to decode tokens/s."""
    import numpy as np
    from oracle import shadowkv_oracle as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # noqa: BLE001
        cores = os.cpu_count()
    one = cfg.replace(batch=1)
    L = synth.gen_layer(one, seed, layer=0)
    inv, rot, il = synth.rope_table(one)
    f = lambda t: t.to(torch.float64).numpy()
    A, B, V = f(L["A"]), f(L["B"]), f(L["V"])
    n_c = (one.ctx_len - one.window_ctx) // one.chunk
    w_eff = one.ctx_len - n_c * one.chunk
    st = O.build(A, B, V, inv, rot, il, one.chunk, one.n_outlier, one.window_ctx, w_eff + 1100)
    times, step = [], 0
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s or len(times) < 2:
        si = synth.gen_step(one, seed, 0, step)
        t0 = time.perf_counter()
        O.decode_step(st, A, B, V, f(si["q"]), f(si["k_new"]), f(si["v_new"]), step, one.budget, inv, rot, il,
                      one.chunk)
        times.append(time.perf_counter() - t0)
        step += 1
        if step >= 1000:
            break
    t_layer = float(np.median(times))
    # the same oracle with its BLAS pinned to one thread (a short bounded sample)
    t1 = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            ts1 = []
            t_start = time.perf_counter()
            while (time.perf_counter() - t_start < budget_s / 3 or len(ts1) < 2) and len(ts1) < 50:
                si = synth.gen_step(one, seed, 0, step)
                t0 = time.perf_counter()
                O.decode_step(st, A, B, V, f(si["q"]), f(si["k_new"]), f(si["v_new"]), step, one.budget, inv, rot,
                              il, one.chunk)
                ts1.append(time.perf_counter() - t0)
                step += 1
            t1 = float(np.median(ts1))
    except Exception:  # noqa: BLE001
        pass
    return {"value": 1.0 / (cfg.n_layers * t_layer), "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1thread": (1.0 / (cfg.n_layers * t1)) if t1 else None,
            "t_layer_ms_1thread": t1 * 1e3 if t1 else None,
            "sample": f"fp64 numpy oracle decode_step of 1 layer x 1 request at {one.ctx_len} ctx, {len(times)} steps, "
                      f"median {t_layer * 1e3:.1f} ms/layer, extrapolated x{cfg.n_layers} layers (state built untimed)",
            "t_layer_ms": t_layer * 1e3}


# ------------------------------------------------------------------------------------------------
def run_reference(args, cfg):
    """The oracle as it stands (fp64 numpy, oracle/) on the box's host cores, on this arm's config,
    metric and unit.  One step = every layer of one request: for c2 (batch 1) that is the whole
    workload step, measured as is; for the batched configs one request's layers are the bounded
    sample and tokens/s counts that one request.  One layer state is built (untimed) and serves
    every layer's decode call with that layer's own fresh q / k_new / v_new (32 distinct states would
    only lengthen the untimed setup: the oracle's per-layer working set, ~0.3 GB, is far beyond the
    CPU caches either way)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    from oracle import shadowkv_oracle as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # noqa: BLE001
        cores = os.cpu_count()
    one = cfg.replace(batch=1)
    L = synth.gen_layer(one, args.seed, layer=0)
    inv, rot, il = synth.rope_table(one)
    f = lambda t: t.to(torch.float64).numpy()
    A, B, V = f(L["A"]), f(L["B"]), f(L["V"])
    n_steps = args.warmup + args.steps
    st = O.build(A, B, V, inv, rot, il, one.chunk, one.n_outlier, one.window_ctx,
                 (one.ctx_len - ((one.ctx_len - one.window_ctx) // one.chunk) * one.chunk) + n_steps + 2)
    Lm = cfg.n_layers

    def one_step(i):                       # all Lm layers of one request at decode step i
        for l in range(Lm):
            si = synth.gen_step(one, args.seed, l, i)
            O.decode_step(st, A, B, V, f(si["q"]), f(si["k_new"]), f(si["v_new"]), i, one.budget, inv, rot, il,
                          one.chunk)

    for i in range(args.warmup):
        one_step(i)
    t0 = time.perf_counter()
    for i in range(args.warmup, n_steps):
        one_step(i)
    ms_step = (time.perf_counter() - t0) / max(args.steps, 1) * 1e3
    value = 1.0 / (ms_step / 1e3)                   # one request's decode tokens per second
    whole = cfg.batch == 1
    sample = (f"each step = fp64 numpy oracle decode_step for all {Lm} layers of 1 request of {cfg.name} "
              f"({one.ctx_len} ctx, k={one.budget}); " +
              ("this is the whole workload step (batch 1)" if whole else
               f"a bounded sample of the {cfg.batch}-request step: tokens/s counts this one request") +
              "; one untimed layer state serves every layer's call")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth/)",
            "config": workload_config(cfg, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
def value_cache_leg(args, cfg, rho, capacity, states, rope, ws, out, stream, seed, host_bytes, host_peak, n_total, dev):
    """NEXT-1: the same 32-layer step with a GPU value-chunk cache per layer (skv_layer.vc_*,
    capacity k chunks per request and KV head, DESIGN R26) and temporally correlated queries (AR(1) drift
    over decode steps, synth.gen_q_drift, R27).  Hit rate alpha is read from the kernels' own counters.
    Timed like the main pass: one CUDA graph per step, W warm-up replays (which also fill the cache),
    K timed replays with CUDA events."""
    import copy
    from paper_2410_21465_b200 import binding as bd
    Lm, b = cfg.n_layers, cfg.batch
    n_states = len(states)
    steps, warm = args.steps, max(args.warmup, 3)
    try:
        layers = []
        for l in range(Lm):                    # each layer its own cache, even where layer states are shared
            st = copy.copy(states[l % n_states])
            C = capacity * cfg.budget
            st.vc_capacity = C
            st.vc_values = torch.empty(b, cfg.n_kv_heads, C, cfg.chunk, cfg.head_dim, dtype=torch.bfloat16, device=dev)
            st.vc_dir = torch.zeros(b, cfg.n_kv_heads, st.shape.n_c, dtype=torch.int64, device=dev)
            st.vc_stats = torch.zeros(b, cfg.n_kv_heads, 4, dtype=torch.int64, device=dev)
            st.vc_slots = torch.zeros(b, cfg.n_kv_heads, C + cfg.budget, dtype=torch.int64, device=dev)
            layers.append(st)
        qd = torch.stack([synth.gen_q_drift(cfg, seed + 104729, l, warm + steps, rho, device=dev)
                          for l in range(Lm)], dim=1)               # [step][layer][b][hq][d]
    except torch.OutOfMemoryError:
        return {"skipped": "out of HBM for per-layer caches", "q_drift_rho": rho}
    kv = [synth.gen_step(cfg, seed, l, 0, device=dev) for l in range(Lm)]
    k_g = torch.stack([x["k_new"] for x in kv]); v_g = torch.stack([x["v_new"] for x in kv])
    q_g = torch.empty_like(qd[0])
    step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
    cap = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        for l in range(Lm):
            layers[l].decode_dev(rope.struct, q_g[l], k_g[l], v_g[l], step_dev, n_total, out[l], ws, stream=cap)
        step_dev.add_(1)
    for st in layers:
        st.vc_dir.zero_(); st.vc_stats.zero_(); st.vc_slots.zero_()
    step_dev.fill_(0)
    torch.cuda.synchronize()
    for i in range(warm):
        q_g.copy_(qd[i], non_blocking=True)
        g.replay()
    torch.cuda.synchronize()
    h0 = sum(int(st.vc_stats[..., 3].sum()) for st in layers)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(warm, warm + steps):
        q_g.copy_(qd[i], non_blocking=True)
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    hits = sum(int(st.vc_stats[..., 3].sum()) for st in layers) - h0
    lookups = steps * Lm * b * cfg.n_kv_heads * cfg.budget
    alpha = hits / lookups
    miss_bytes = (1.0 - alpha) * host_bytes                          # host-link bytes per layer call
    t_roof = Lm * miss_bytes / (host_peak * 1e9)
    del g, layers, qd
    torch.cuda.empty_cache()
    from paper_2410_21465_b200 import shard
    value = shard.job_tokens_per_s(args.tok_rank, ms / 1e3, device=dev)  # all ranks: sum tokens / max time
    # P:200-206 equivalent bandwidth: the dense-attention KV bytes a layer would read (2 S M per KV head,
    # M = d * 2 B) over the measured layer time, and the paper's analytic B_eq at the measured alpha with
    # this box's bandwidths (HBM from MEASURED_PEAKS.json, host link measured live)
    hbm_gbs, _ = load_peaks()
    S, C, K, O = cfg.ctx_len, cfg.chunk, cfg.budget, cfg.n_outlier
    dense_bytes = 2.0 * S * cfg.head_dim * 2 * cfg.n_kv_heads * b
    beq_model = 2.0 * S * hbm_gbs / (S / C + 2.0 * (K + O) * C + (1.0 - alpha) * K * C * hbm_gbs / host_peak)
    beq_meas = dense_bytes / (ms * 1e-3 / Lm) / 1e9
    return {"q_drift_rho": rho, "capacity_chunks": capacity * cfg.budget, "capacity_over_k": capacity,
            "alpha": alpha, "value": value, "unit": UNIT, "ms_per_step": ms,
            "equivalent_bandwidth_GBps": {"measured": beq_meas, "paper_model_P204": beq_model, "hbm_peak": hbm_gbs,
                                          "host_peak": host_peak},
            "steps": steps, "warmup": warm, "host_bytes_per_layer": miss_bytes,
            "step_frac_of_host_roofline": t_roof / (ms * 1e-3),
            "note": "P:156 cache-aware decode: cached chunks come from HBM (least-recently-selected replacement, "
                    "capacity C chunks per request and KV head; C = k keeps exactly the previous selection); alpha "
                    "measured by the kernels' hit counters; queries drift as AR(1) over steps (synthetic: the "
                    "paper's ~60% is Fig 3c on real traces)"}


# ------------------------------------------------------------------------------------------------
def multi_query_leg(args, cfg, q_len, states, rope, seed, host_bytes, host_peak, dev):
    """NEXT-3 (Alg 2 with Q in R^{b x h_q x s_q x d}): every decode call carries s_q query
    tokens (e.g. draft tokens being verified) that share one selection and one value fetch.  Same
    layer states and graph-timed 32-layer step as the main line; tokens/s counts s_q tokens per request
    per step (all accepted: an upper bound for speculative decoding, the attention cost per call)."""
    from paper_2410_21465_b200 import LayerState, Shape, alloc_workspace, shard
    import copy
    if (cfg.n_q_heads // cfg.n_kv_heads) * q_len > 16:
        return {"skipped": f"GQA group x s_q = {(cfg.n_q_heads // cfg.n_kv_heads) * q_len} > 16 rows", "q_len": q_len}
    Lm, b = cfg.n_layers, cfg.batch
    n_states = len(states)
    steps, warm = args.steps, max(args.warmup, 3)
    shape = Shape.from_config(cfg, steps=steps + warm + 1, q_len=q_len)
    try:
        ws = alloc_workspace(shape, device=dev)
        layers = []
        for l in range(n_states):
            st = copy.copy(states[l])
            st.shape = shape
            # a window ring sized for this leg's s_q-token appends (context tail copied from the built state)
            st.K_win = torch.zeros(b, cfg.n_kv_heads, shape.window_cap, cfg.head_dim, dtype=torch.bfloat16, device=dev)
            st.V_win = torch.zeros_like(st.K_win)
            w_eff = shape.w_eff
            st.K_win[:, :, :w_eff].copy_(states[l].K_win[:, :, :w_eff]); st.V_win[:, :, :w_eff].copy_(states[l].V_win[:, :, :w_eff])
            layers.append(st)
    except torch.OutOfMemoryError:
        return {"skipped": "out of HBM", "q_len": q_len}
    gen = torch.Generator(device=dev).manual_seed(seed + 31337)
    q_g = (2.0 * torch.randn(Lm, b, cfg.n_q_heads, q_len, cfg.head_dim, device=dev, generator=gen)).to(torch.bfloat16)
    k_g = torch.randn(Lm, b, cfg.n_kv_heads, q_len, cfg.head_dim, device=dev, generator=gen).to(torch.bfloat16)
    v_g = torch.randn(k_g.shape, device=dev, generator=gen).to(torch.bfloat16)
    out = torch.empty(Lm, b, cfg.n_q_heads, q_len, cfg.head_dim, dtype=torch.bfloat16, device=dev)
    qs = [(2.0 * torch.randn(q_g.shape, device=dev, generator=gen)).to(torch.bfloat16) for _ in range(4)]
    step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
    max_step = (steps + warm) * q_len
    cap = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        for l in range(Lm):
            layers[l % n_states].decode_dev(rope.struct, q_g[l], k_g[l], v_g[l], step_dev, max_step, out[l], ws, stream=cap)
        step_dev.add_(q_len)
    step_dev.fill_(0)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    for i in range(warm):
        q_g.copy_(qs[i % 4], non_blocking=True)
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        q_g.copy_(qs[i % 4], non_blocking=True)                  # fresh queries: fresh selections
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    value = shard.job_tokens_per_s(args.tok_rank * q_len, ms / 1e3, device=dev)
    del g, layers, ws
    torch.cuda.empty_cache()
    return {"q_len": q_len, "value": value, "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warm,
            "step_frac_of_host_roofline": Lm * host_bytes / (host_peak * 1e9) / (ms * 1e-3),
            "note": "s_q query tokens per request per call share one selection (S1 = sum over s_q, P:171) and one "
                    "host value fetch; tokens/s counts all s_q tokens (every draft accepted)"}


# ------------------------------------------------------------------------------------------------
def lowrank_gen_leg(args, cfg, states, rope, ws, seed, dev):
    """NEXT-4 (P:196 footnote): the same graph-timed 32-layer step with skv_layer.A_gen, i.e. every
    generated token's key stored as one rank-r row (pre-RoPE k_new projected on the B rows) and rebuilt
    when attended, instead of h_kv*d post-RoPE values in the window."""
    import copy
    from paper_2410_21465_b200 import shard
    Lm, b = cfg.n_layers, cfg.batch
    n_states = len(states)
    steps, warm = args.steps, max(args.warmup, 3)
    try:
        layers = []
        for l in range(n_states):
            st = copy.copy(states[l])
            st.A_gen = torch.zeros(b, st.shape.window_cap, cfg.rank, dtype=torch.bfloat16, device=dev)
            layers.append(st)
    except torch.OutOfMemoryError:
        return {"skipped": "out of HBM"}
    gen = torch.Generator(device=dev).manual_seed(seed + 4242)
    q_g = (2.0 * torch.randn(Lm, b, cfg.n_q_heads, cfg.head_dim, device=dev, generator=gen)).to(torch.bfloat16)
    k_g = torch.randn(Lm, b, cfg.n_kv_heads, cfg.head_dim, device=dev, generator=gen).to(torch.bfloat16)
    v_g = torch.randn(Lm, b, cfg.n_kv_heads, cfg.head_dim, device=dev, generator=gen).to(torch.bfloat16)
    qs = [(2.0 * torch.randn(q_g.shape, device=dev, generator=gen)).to(torch.bfloat16) for _ in range(4)]
    out = torch.empty(Lm, b, cfg.n_q_heads, cfg.head_dim, dtype=torch.bfloat16, device=dev)
    step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
    max_step = steps + warm
    cap = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        for l in range(Lm):
            layers[l % n_states].decode_dev(rope.struct, q_g[l], k_g[l], v_g[l], step_dev, max_step, out[l], ws, stream=cap)
        step_dev.add_(1)
    step_dev.fill_(0)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    for i in range(warm):
        q_g.copy_(qs[i % 4], non_blocking=True)
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        q_g.copy_(qs[i % 4], non_blocking=True)
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    value = shard.job_tokens_per_s(args.tok_rank, ms / 1e3, device=dev)
    del g, layers
    torch.cuda.empty_cache()
    return {"value": value, "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warm,
            "key_bytes_per_generated_token": cfg.rank * 2, "plain_window_key_bytes": cfg.n_kv_heads * cfg.head_dim * 2,
            "note": "generated keys stored as rank-r rows (K' Psi, P:196) and rebuilt with RoPE when attended"}


# ------------------------------------------------------------------------------------------------
def run_ours(args, cfg):
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    numa_note = bind_to_gpu_numa(local)          # before the pinned pool is first touched
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace, binding as bd, shard

    dev = "cuda"
    tok_rank = None                              # this rank's decode tokens per step (sums to the job's)
    cfg0, strong_note = cfg, None
    if args.scaling == "strong":                 # by request, or by KV head when batch < n
        pl = shard.plan(cfg.batch, cfg.n_q_heads, cfg.n_kv_heads, rank, world)
        tok_rank = shard.tokens_this_rank(pl, cfg.n_kv_heads)
        cfg = cfg.replace(batch=pl.batch, n_kv_heads=pl.n_kv_heads, n_q_heads=pl.n_q_heads)
        strong_note = (f"strong scaling: {cfg0.batch} request(s) x {cfg0.n_kv_heads} KV heads split by {pl.mode} over "
                       f"{world} GPU(s); no collective on the data path")
    Lm, b = cfg.n_layers, cfg.batch
    if tok_rank is None:
        tok_rank = float(b)
    args.tok_rank = tok_rank
    n_total = args.warmup + 2 * args.steps + args.e2e_steps + 48
    shape = Shape.from_config(cfg, steps=n_total + 1)
    inv, rot, il = synth.rope_table(cfg)
    rope = RopeTable(inv, rot, il, device=dev)
    ws = alloc_workspace(shape, device=dev)
    seed = args.seed + 7919 * rank

    # --- states: L_m distinct layers (fewer if host RAM / HBM cannot hold them; every state is
    #     far larger than L2 either way), values in one pinned+mapped host pool -------------------
    per_layer = b * cfg.n_kv_heads * cfg.ctx_len * cfg.head_dim
    dev_layer = 2 * b * (cfg.ctx_len * cfg.rank + cfg.n_kv_heads * (shape.n_c * cfg.head_dim + cfg.rank * cfg.head_dim
                                                                     + 2 * (cfg.n_outlier * cfg.chunk + shape.window_cap) * cfg.head_dim))
    import psutil
    host_cap = int(0.6 * psutil.virtual_memory().available / world // (per_layer * 2))   # c5: pass --layer-states 8
    dev_cap = int(0.7 * torch.cuda.mem_get_info()[0] // dev_layer)
    n_states = args.layer_states or max(1, min(Lm, host_cap, dev_cap))
    if per_layer * 2 * n_states > 0.8 * psutil.virtual_memory().available / world:
        raise SystemExit(f"{per_layer * 2 * n_states / 1e9:.1f} GB of pinned values exceed host RAM; "
                         f"use a smaller --layer-states")
    t_setup = time.perf_counter()
    retried = False
    while True:                 # page-locking can fail below the RAM estimate: fewer states then
        try:
            pool = pinned_pool(per_layer * 2 * n_states)
            break
        except RuntimeError:
            torch.cuda.cudart().cudaGetLastError()
            if not retried:     # a previous process may still be releasing its pinned pages
                retried = True
                time.sleep(5)
                continue
            if args.layer_states or n_states == 1:
                raise
            n_states = max(1, n_states // 2)
    states = []
    for l in range(n_states):
        inp = synth.gen_layer(cfg, seed, layer=l, device=dev)
        vh = pool[l * per_layer:(l + 1) * per_layer].view(b, cfg.n_kv_heads, cfg.ctx_len, cfg.head_dim)
        st = LayerState(shape, device=dev, V_host=vh)
        st.A.copy_(inp["A"]); st.B.copy_(inp["B"]); vh.copy_(inp["V"])
        st.build(rope.struct, ws)
        states.append(st)
        del inp
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    # Alg 1 minus the SVD (a0, untimed setup): one layer's shadowkv_build_cache, CUDA events, median of 5
    bms = []
    for _ in range(5):
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(); states[0].build(rope.struct, ws); b1.record(); b1.synchronize()
        bms.append(b0.elapsed_time(b1))
    build_ms = statistics.median(bms)

    # --- per-step inputs (fresh q every step and layer => fresh selections, alpha ~ 0) --------
    def step_inputs(i, device):
        qs, ks, vs = [], [], []
        for l in range(Lm):
            si = synth.gen_step(cfg, seed, l, i, device=dev)
            qs.append(si["q"]); ks.append(si["k_new"]); vs.append(si["v_new"])
        return torch.stack(qs).to(device), torch.stack(ks).to(device), torch.stack(vs).to(device)

    dev_inputs = [step_inputs(i, dev) for i in range(args.warmup + args.steps)]
    out = torch.empty(Lm, b, cfg.n_q_heads, cfg.head_dim, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream()
    launches = [0]

    def step(i, q, kn, vn):
        for l in range(Lm):
            states[l % n_states].decode(rope.struct, q[l], kn[l], vn[l], i, out[l], ws, stream=stream)
            launches[0] += bd.shadowkv_last_launch_count()

    for i in range(args.warmup):
        step(i, *dev_inputs[i])
    torch.cuda.synchronize()

    # --- CUDA graph of one whole step: every layer through shadowkv_decode_step_dev (the step index
    #     lives in device memory) + the counter increment; replays advance the decode step ------------
    use_graph = args.graph == "on"
    if use_graph:
        q_g = torch.empty_like(dev_inputs[0][0]); k_g = torch.empty_like(dev_inputs[0][1])
        v_g = torch.empty_like(dev_inputs[0][2])
        step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        cap = torch.cuda.Stream()
        graph_launches = [0]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for l in range(Lm):
                states[l % n_states].decode_dev(rope.struct, q_g[l], k_g[l], v_g[l], step_dev, n_total, out[l], ws,
                                                stream=cap)
                graph_launches[0] += bd.shadowkv_last_launch_count()
            step_dev.add_(1)
        step_dev.fill_(args.warmup)
        torch.cuda.synchronize()

    def run_step(i, q, kn, vn):
        if use_graph:
            q_g.copy_(q, non_blocking=True); k_g.copy_(kn, non_blocking=True); v_g.copy_(vn, non_blocking=True)
            g.replay()
            launches[0] += graph_launches[0]
        else:
            step(i, q, kn, vn)

    if world > 1:
        torch.distributed.barrier()
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.warmup, args.warmup + args.steps):
            run_step(i, *dev_inputs[i])
        e1.record(stream)
        torch.cuda.synchronize()
    gpu_launches = launches[0]
    ms_local = e0.elapsed_time(e1) / args.steps
    value = shard.job_tokens_per_s(tok_rank, ms_local / 1e3, device=dev)  # sum tokens / max time
    ms = shard.max_over_ranks(ms_local, device=dev)

    # --- dominant-kernel timing: a second timed pass of K steps with CUDA events recorded on the
    #     launch stream around the fused sparse-attention kernel of every layer (kept out of the
    #     `value` pass because an event record between kernels disables their PDL overlap)
    i1 = args.warmup + args.steps
    bd.shadowkv_profile_begin(Lm * args.steps + 8, 1 << 2)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p0.record(stream)
    for i in range(args.steps):
        step(i1 + i, *dev_inputs[args.warmup + i])
    p1.record(stream)
    torch.cuda.synchronize()
    prof = bd.shadowkv_profile_end()
    prof_pass_ms = p0.elapsed_time(p1) / args.steps

    # --- e2e: host buffers through the public API, H2D inputs + D2H result inside the region --
    i0 = args.warmup + 2 * args.steps
    host_inputs = [tuple(t.cpu().pin_memory() for t in step_inputs(i, "cpu")) for i in range(i0, i0 + args.e2e_steps)]
    q_d = torch.empty_like(dev_inputs[0][0]); k_d = torch.empty_like(dev_inputs[0][1]); v_d = torch.empty_like(dev_inputs[0][2])
    out_h = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host_inputs[0]) if host_inputs else 0
    d2h = out_h.numel() * out_h.element_size()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for j, (qh, kh, vh) in enumerate(host_inputs):
        if use_graph:                                          # H2D straight into the graph's input buffers
            q_g.copy_(qh, non_blocking=True); k_g.copy_(kh, non_blocking=True); v_g.copy_(vh, non_blocking=True)
            g.replay()
        else:
            q_d.copy_(qh, non_blocking=True); k_d.copy_(kh, non_blocking=True); v_d.copy_(vh, non_blocking=True)
            step(i0 + j, q_d, k_d, v_d)
        out_h.copy_(out, non_blocking=True)
        stream.synchronize()                                   # host reads the step's result
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_local = f0.elapsed_time(f1) / max(1, args.e2e_steps)
    e2e_value = shard.job_tokens_per_s(tok_rank, e2e_local / 1e3, device=dev)
    e2e_ms = shard.max_over_ranks(e2e_local, device=dev)

    # --- roofline of the dominant kernel (fused rebuild+gather+attention: host-link bound) -----
    g_ms, g_cnt = prof["sparse_attn"]
    g_avg_ms = g_ms / max(g_cnt, 1)
    host_bytes = b * cfg.n_kv_heads * cfg.budget * cfg.chunk * cfg.head_dim * 2          # HOST_alg per launch
    host_peak, host_all = measure_dma_h2d(pool, world)
    achieved = host_bytes / (g_avg_ms * 1e-3) / 1e9
    nt = load_ncu_traffic()
    same = nt.get("config", "c2") == cfg.name and world == 1 and args.scaling == "weak"
    traffic = nt.get("sparse_attn_dram_bytes") if same else None       # one ncu --set full capture, per launch
    roofline = {"bound": "host_link", "kernel": "k_sparse_attn", "achieved": achieved, "peak": host_peak,
                "unit": "GB/s", "frac": achieved / host_peak, "traffic": traffic,
                "traffic_pcie": nt.get("sparse_attn_pcie_read_bytes") if same else None,
                "traffic_note": "traffic = dram__bytes_read+write of k_sparse_attn (A rows, B_h, outliers, window "
                                "from HBM; algorithmic 7.1 MB at c2); traffic_pcie = its host-link reads "
                                "(pcie__read_bytes, algorithmic 4.19 MB); source " + str(nt.get("source")),
                "algorithmic_bytes_per_launch": host_bytes, "avg_launch_ms": g_avg_ms, "launches": g_cnt,
                "share_of_step": g_ms / (prof_pass_ms * args.steps), "timing_pass_ms_per_step": prof_pass_ms,
                "step_frac_of_roofline": (Lm * host_bytes / (host_peak * 1e9)) / (ms * 1e-3),
                "peak_note": "pinned H2D copy-engine bandwidth measured live in this run (1 GiB, best of 6; with N "
                             "ranks all copy concurrently: B_host(n), this rank's share); zero-copy SM loads "
                             "saturate ~51 GB/s (profiles/r01_probe_hostlink.txt)",
                "host_link_concurrent_GBps": {"per_rank": host_all, "aggregate": sum(host_all), "n": world}}

    # --- selection adjacency: mean run length of consecutive selected chunk ids, so that
    #     contiguity is not silently helping the host link (2 KB pieces are fetched independently anyway)
    sel_ids = torch.empty(b, cfg.n_kv_heads, cfg.budget, dtype=torch.int32, device=dev)
    runs = []
    for l in range(min(4, n_states)):
        q0, k0, v0 = dev_inputs[l % len(dev_inputs)]
        states[l].decode(rope.struct, q0[l], k0[l], v0[l], n_total - 1, out[l], ws, sel_ids=sel_ids, stream=stream)
        ids = sel_ids.cpu().numpy().reshape(-1, cfg.budget)
        for row in ids:
            runs.append(cfg.budget / (1 + int(((row[1:] - row[:-1]) != 1).sum())))
    selection = {"mean_run_length_chunks": float(sum(runs) / len(runs)), "chunks_per_kv_head": cfg.budget,
                 "sample": f"{len(runs)} (layer, request, KV head) selections at the last step index"}

    def leg(fn, *a):
        """A widened-row leg never costs the headline line on one GPU: a failure is reported in its place.
        (With N > 1 the legs' collectives must stay in step across ranks, so errors propagate.)"""
        if world > 1:
            return fn(*a)
        try:
            return fn(*a)
        except Exception as e:  # noqa: BLE001
            torch.cuda.synchronize()
            return {"error": f"{type(e).__name__}: {e}"[:300]}

    value_cache = None
    if args.vc_rho:
        value_cache = [leg(value_cache_leg, args, cfg, float(r), int(c), states, rope, ws, out, stream, seed,
                           host_bytes, host_peak, n_total, dev)
                       for r in args.vc_rho.split(",") if r.strip() for c in args.vc_capacity.split(",") if c.strip()]

    multi_query = None
    if args.q_len_leg and args.q_len_leg > 1:
        multi_query = leg(multi_query_leg, args, cfg, args.q_len_leg, states, rope, seed, host_bytes, host_peak, dev)

    lowrank_gen = None
    if args.lowrank_gen_leg:
        lowrank_gen = leg(lowrank_gen_leg, args, cfg, states, rope, ws, seed, dev)

    breakdown = None
    if args.breakdown:
        bd.shadowkv_profile_begin(Lm * 5 * 20 + 8, 0x1F)
        for i in range(20):
            step(i0 + args.e2e_steps + i, *dev_inputs[i % len(dev_inputs)])
        torch.cuda.synchronize()
        breakdown = {k: {"avg_us": v[0] / max(v[1], 1) * 1e3, "launches": v[1]} for k, v in bd.shadowkv_profile_end().items()}

    if rank != 0:
        return
    hbm_peak, hbm_src = load_peaks()
    n_c = shape.n_c
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded, synth/; random rank-160 factors)",
            "config": dict(workload_config(cfg, world), layer_states=n_states, host_numa=numa_note,
                           launch="one CUDA graph per 32-layer step (shadowkv_decode_step_dev)" if use_graph
                           else "stream launches (shadowkv_decode_step)"),
            "roofline": roofline,
            "selection": selection,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
            "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src,
            "setup_s": setup_s,
            "build_ms_per_layer": build_ms}
    # P:200-206 equivalent bandwidth of the uncached step (alpha = 0): dense KV bytes / layer time, and the
    # paper's model with this box's bandwidths
    S_, C_, K_, O_ = cfg.ctx_len, cfg.chunk, cfg.budget, cfg.n_outlier
    dense_b = 2.0 * S_ * cfg.head_dim * 2 * cfg.n_kv_heads * b
    line["equivalent_bandwidth_GBps"] = {
        "measured": dense_b / (ms * 1e-3 / Lm) / 1e9,
        "paper_model_P204": 2.0 * S_ * hbm_peak / (S_ / C_ + 2.0 * (K_ + O_) * C_ + K_ * C_ * hbm_peak / host_peak),
        "note": "dense-attention KV bytes per layer over the measured layer time (P:200-206); alpha = 0 here"}
    if strong_note:                              # the job's batch, not the per-rank share
        line["config"].update(global_batch=cfg0.batch, parallelism=strong_note,
                              per_rank={"batch": cfg.batch, "n_kv_heads": cfg.n_kv_heads, "n_q_heads": cfg.n_q_heads})
    if value_cache:
        line["value_cache"] = value_cache[0] if len(value_cache) == 1 else value_cache
    if multi_query:
        line["multi_query"] = multi_query
    if lowrank_gen:
        line["lowrank_gen"] = lowrank_gen
    if breakdown:
        line["kernel_breakdown_us"] = breakdown
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.seed)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one process per GPU) on this node through
    torch.distributed.run with the same arguments, rendezvous on 127.0.0.1."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args, cfg):
    """--dry-run: the multi-rank path without a GPU -- gloo group, this rank's shard plan, an empty timed
    step bracketed by barriers, max over ranks; rank 0 prints the plan of every rank."""
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    from paper_2410_21465_b200 import shard
    pl = shard.plan(cfg.batch, cfg.n_q_heads, cfg.n_kv_heads, rank, world) if args.scaling == "strong" else \
        shard.Plan("request", (0, cfg.batch), (0, cfg.n_kv_heads), (0, cfg.n_q_heads))
    tok = shard.tokens_this_rank(pl, cfg.n_kv_heads)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    if world > 1:
        dist.barrier()
    ms = shard.max_over_ranks((time.perf_counter() - t0) * 1e3)
    plans = [None] * world
    if world > 1:
        dist.all_gather_object(plans, {"rank": rank, "mode": pl.mode, "requests": pl.requests,
                                       "kv_heads": pl.kv_heads, "q_heads": pl.q_heads, "tokens": tok})
    else:
        plans = [{"rank": 0, "mode": pl.mode, "requests": pl.requests, "kv_heads": pl.kv_heads,
                  "q_heads": pl.q_heads, "tokens": tok}]
    total = shard.sum_over_ranks(tok)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "world_size": world, "scaling": args.scaling,
                          "config": workload_config(cfg, world), "tokens_per_step": total, "ms_per_step": ms,
                          "ranks": plans}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    if args.scaling is None:
        args.scaling = "strong" if cfg.name == "c3" else "weak"
    rank, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.dry_run:
        run_dry(args, cfg)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
