"""Thin ctypes binding of libshadowkv.so (include/shadowkv.h).  Argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module only turns
torch tensors into pointers.  There is no CPU fallback: if the library is missing the
import-time ``load()`` raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libshadowkv.so")

SKV_OK, SKV_EINVAL, SKV_EUNSUPPORTED, SKV_ECUDA, SKV_ESTATE = range(5)
STATUS_NAMES = {0: "SKV_OK", 1: "SKV_EINVAL", 2: "SKV_EUNSUPPORTED", 3: "SKV_ECUDA", 4: "SKV_ESTATE"}
EXPORTED = ["shadowkv_init", "shadowkv_score_plan", "shadowkv_rope_sincos", "shadowkv_workspace_bytes", "shadowkv_build_cache", "shadowkv_decode_step", "shadowkv_decode_step_dev",
            "shadowkv_last_error", "shadowkv_abi_version", "shadowkv_last_launch_count",
            "shadowkv_profile_begin", "shadowkv_profile_end", "shadowkv_trace_buffer",
            "shadowkv_factorize_workspace_bytes", "shadowkv_factorize"]
KERNEL_NAMES = ["score", "select", "sparse_attn", "reserved", "combine"]


class SkvDims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("batch", "n_q_heads", "n_kv_heads", "head_dim", "ctx_len", "rank", "chunk",
                 "n_outlier", "budget", "window_ctx", "window_cap", "q_len")] + \
        [("ctx_lens", ctypes.c_void_p), ("ctx_lens_dev", ctypes.c_void_p)]


class SkvRope(ctypes.Structure):
    _fields_ = [("rotary_dim", ctypes.c_int32), ("interleaved", ctypes.c_int32), ("inv_freq", ctypes.c_void_p)]


class SkvLayer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("A", "B", "landmarks", "outlier_ids", "K_out", "V_out", "K_win", "V_win", "V_host",
                 "vc_values", "vc_dir", "vc_stats", "A_gen", "vc_slots")] + \
        [("vc_capacity", ctypes.c_int32), ("reserved0", ctypes.c_int32)]


class ShadowKVError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_LIB = None


def load(path: str = LIB_PATH):
    """Load the in-tree library (raises if it was not built -- no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.shadowkv_init.restype = ctypes.c_int
    lib.shadowkv_init.argtypes = [ctypes.c_int32]
    lib.shadowkv_score_plan.restype = ctypes.c_int
    lib.shadowkv_score_plan.argtypes = [P(SkvDims), ctypes.c_int32, P(ctypes.c_int32)]
    lib.shadowkv_rope_sincos.restype = ctypes.c_int
    lib.shadowkv_rope_sincos.argtypes = [P(SkvRope), ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    lib.shadowkv_workspace_bytes.restype = ctypes.c_size_t
    lib.shadowkv_workspace_bytes.argtypes = [P(SkvDims)]
    lib.shadowkv_build_cache.restype = ctypes.c_int
    lib.shadowkv_build_cache.argtypes = [P(SkvDims), P(SkvRope), P(SkvLayer), ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p]
    lib.shadowkv_decode_step.restype = ctypes.c_int
    lib.shadowkv_decode_step.argtypes = [P(SkvDims), P(SkvRope), P(SkvLayer), ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.shadowkv_decode_step_dev.restype = ctypes.c_int
    lib.shadowkv_decode_step_dev.argtypes = [P(SkvDims), P(SkvRope), P(SkvLayer), ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.shadowkv_factorize_workspace_bytes.restype = ctypes.c_size_t
    lib.shadowkv_factorize_workspace_bytes.argtypes = [P(SkvDims)]
    lib.shadowkv_factorize.restype = ctypes.c_int
    lib.shadowkv_factorize.argtypes = [P(SkvDims), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.shadowkv_last_error.restype = ctypes.c_char_p
    lib.shadowkv_last_error.argtypes = []
    lib.shadowkv_abi_version.restype = ctypes.c_int32
    lib.shadowkv_last_launch_count.restype = ctypes.c_int32
    lib.shadowkv_profile_begin.restype = ctypes.c_int
    lib.shadowkv_profile_begin.argtypes = [ctypes.c_int32, ctypes.c_int32]
    lib.shadowkv_profile_end.restype = ctypes.c_int
    lib.shadowkv_profile_end.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]
    lib.shadowkv_trace_buffer.restype = ctypes.c_int
    lib.shadowkv_trace_buffer.argtypes = [ctypes.c_void_p]
    _LIB = lib
    return lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _check(st: int):
    if st != SKV_OK:
        raise ShadowKVError(st, load().shadowkv_last_error().decode())


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def dims_struct(batch, n_q_heads, n_kv_heads, head_dim, ctx_len, rank, chunk, n_outlier, budget,
                window_ctx, window_cap, q_len=1, ctx_lens=None, ctx_lens_dev=None) -> SkvDims:
    """ctx_lens: host int32 tensor / array [batch] of per-request lengths (ragged batch) with its device
    mirror ctx_lens_dev; the caller keeps both alive while the struct is in use."""
    return SkvDims(batch, n_q_heads, n_kv_heads, head_dim, ctx_len, rank, chunk, n_outlier, budget,
                   window_ctx, window_cap, q_len, _ptr(ctx_lens), _ptr(ctx_lens_dev))


def rope_struct(rotary_dim: int, interleaved: bool, inv_freq) -> SkvRope:
    return SkvRope(rotary_dim, 1 if interleaved else 0, _ptr(inv_freq))


def layer_struct(A, B, landmarks, outlier_ids, K_out, V_out, K_win, V_win, V_host,
                 vc_values=None, vc_dir=None, vc_stats=None, A_gen=None, vc_slots=None,
                 vc_capacity: int = 0) -> SkvLayer:
    return SkvLayer(_ptr(A), _ptr(B), _ptr(landmarks), _ptr(outlier_ids), _ptr(K_out), _ptr(V_out),
                    _ptr(K_win), _ptr(V_win), _ptr(V_host), _ptr(vc_values), _ptr(vc_dir), _ptr(vc_stats),
                    _ptr(A_gen), _ptr(vc_slots), int(vc_capacity), 0)


_INIT_DEVICES: set = set()


def shadowkv_init(device: int | None = None):
    """One-time per-device setup (kernel attributes, internal streams, tensor-map encoder)."""
    if device is None:
        device = torch.cuda.current_device()
    device = int(device)
    if device not in _INIT_DEVICES:
        _check(load().shadowkv_init(device))
        _INIT_DEVICES.add(device)


def ensure_init(device) -> None:
    """shadowkv_init for a torch device ("cuda", "cuda:1", torch.device, index) if not done yet."""
    d = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    if d.type == "cuda":
        shadowkv_init(d.index if d.index is not None else torch.cuda.current_device())


def shadowkv_score_plan(dims: SkvDims, n_sm: int):
    """-> (grid, tiles_per_cta, heads_per_cta, ctas_per_head); raises ShadowKVError if unplannable."""
    plan = (ctypes.c_int32 * 4)()
    _check(load().shadowkv_score_plan(ctypes.byref(dims), int(n_sm), plan))
    return tuple(int(x) for x in plan)


def shadowkv_rope_sincos(rope: SkvRope, pos, n: int, sincos, stream=None):
    _check(load().shadowkv_rope_sincos(ctypes.byref(rope), _ptr(pos), int(n), _ptr(sincos), _stream_ptr(stream)))


def shadowkv_workspace_bytes(dims: SkvDims) -> int:
    n = load().shadowkv_workspace_bytes(ctypes.byref(dims))
    if n == 0:
        raise ShadowKVError(SKV_EINVAL, load().shadowkv_last_error().decode())
    return n


def shadowkv_build_cache(dims: SkvDims, rope: SkvRope, layer: SkvLayer, K_rope, workspace, stream=None):
    _check(load().shadowkv_build_cache(ctypes.byref(dims), ctypes.byref(rope), ctypes.byref(layer),
                                       _ptr(K_rope), _ptr(workspace), _stream_ptr(stream)))


def shadowkv_decode_step(dims: SkvDims, rope: SkvRope, layer: SkvLayer, q, k_new, v_new, step: int, out,
                         sel_ids=None, dbg_keys=None, workspace=None, stream=None):
    _check(load().shadowkv_decode_step(ctypes.byref(dims), ctypes.byref(rope), ctypes.byref(layer), _ptr(q),
                                       _ptr(k_new), _ptr(v_new), int(step), _ptr(out), _ptr(sel_ids),
                                       _ptr(dbg_keys), _ptr(workspace), _stream_ptr(stream)))


def shadowkv_decode_step_dev(dims: SkvDims, rope: SkvRope, layer: SkvLayer, q, k_new, v_new, step_dev,
                             max_step: int, out, sel_ids=None, dbg_keys=None, workspace=None, stream=None):
    _check(load().shadowkv_decode_step_dev(ctypes.byref(dims), ctypes.byref(rope), ctypes.byref(layer), _ptr(q),
                                           _ptr(k_new), _ptr(v_new), _ptr(step_dev), int(max_step), _ptr(out),
                                           _ptr(sel_ids), _ptr(dbg_keys), _ptr(workspace), _stream_ptr(stream)))


def shadowkv_last_launch_count() -> int:
    return int(load().shadowkv_last_launch_count())


def shadowkv_abi_version() -> int:
    return int(load().shadowkv_abi_version())


def shadowkv_profile_begin(capacity: int, kernel_mask: int):
    _check(load().shadowkv_profile_begin(int(capacity), int(kernel_mask)))


def shadowkv_profile_end():
    """-> {kernel_name: (total_ms, count)}"""
    ms = (ctypes.c_double * 5)()
    cnt = (ctypes.c_int32 * 5)()
    _check(load().shadowkv_profile_end(ms, cnt))
    return {n: (ms[i], cnt[i]) for i, n in enumerate(KERNEL_NAMES)}


def shadowkv_trace_buffer(buf):
    """Enable (device tensor of >= 4*4096*16 int64) or disable (None) the kernels' globaltimer stamps."""
    _check(load().shadowkv_trace_buffer(_ptr(buf)))


def shadowkv_factorize_workspace_bytes(dims: SkvDims) -> int:
    n = load().shadowkv_factorize_workspace_bytes(ctypes.byref(dims))
    if n == 0:
        raise ShadowKVError(SKV_EINVAL, load().shadowkv_last_error().decode())
    return n


def shadowkv_factorize(dims: SkvDims, K_pre, A, B, sigma=None, workspace=None, stream=None):
    _check(load().shadowkv_factorize(ctypes.byref(dims), _ptr(K_pre), _ptr(A), _ptr(B), _ptr(sigma),
                                     _ptr(workspace), _stream_ptr(stream)))
