"""C-ABI checks that need no GPU: the library loads, exports what include/shadowkv.h declares,
and rejects bad arguments synchronously (SKV_EINVAL / SKV_EUNSUPPORTED) before touching CUDA."""
import ctypes
import os
import re

import pytest

import synth
from paper_2410_21465_b200 import binding as bd
from paper_2410_21465_b200.state import Shape

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "shadowkv.h")


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(shadowkv_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    assert "shadowkv_build_cache" in syms and "shadowkv_decode_step" in syms
    assert set(syms) == set(bd.EXPORTED)


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert bd.shadowkv_abi_version() == 7


def _dims(**kw):
    base = dict(batch=1, n_q_heads=32, n_kv_heads=8, head_dim=128, ctx_len=4096, rank=160, chunk=8,
                n_outlier=4, budget=8, window_ctx=16, window_cap=32)
    base.update(kw)
    return bd.SkvDims(**base)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_workspace_bytes_for_every_config(lib, name):
    shp = Shape.from_config(synth.CONFIGS[name])
    n = bd.shadowkv_workspace_bytes(shp.dims())
    assert n > 0 and n % 256 == 0


@pytest.mark.parametrize("kw,status,needle", [
    (dict(budget=507), bd.SKV_EINVAL, "budget"),              # k > n_L
    (dict(budget=0), bd.SKV_EINVAL, "budget"),
    (dict(n_outlier=510), bd.SKV_EINVAL, "n_outlier"),        # o >= n_c
    (dict(rank=8), bd.SKV_EINVAL, "rank"),                    # r out of range
    (dict(rank=168), bd.SKV_EUNSUPPORTED, "rank"),
    (dict(head_dim=64), bd.SKV_EUNSUPPORTED, "head_dim"),
    (dict(chunk=16), bd.SKV_EUNSUPPORTED, "chunk"),
    (dict(n_q_heads=30), bd.SKV_EINVAL, "GQA"),
    (dict(n_q_heads=24), bd.SKV_EUNSUPPORTED, "group"),
    (dict(n_q_heads=96, n_kv_heads=3), bd.SKV_EUNSUPPORTED, "group"),
    (dict(window_cap=8), bd.SKV_EINVAL, "window_cap"),
    (dict(ctx_len=20), bd.SKV_EINVAL, "ctx_len"),
])
def test_invalid_dims_rejected(lib, kw, status, needle):
    assert lib.shadowkv_workspace_bytes(ctypes.byref(_dims(**kw))) == 0
    assert needle in lib.shadowkv_last_error().decode()
    rope = bd.SkvRope(128, 0, 16)
    layer = bd.SkvLayer(*([16] * 9 + [None] * 4))
    st = lib.shadowkv_decode_step(ctypes.byref(_dims(**kw)), ctypes.byref(rope), ctypes.byref(layer),
                                  16, 16, 16, 0, 16, None, None, 256, None)
    assert st == status


def test_decode_argument_errors_before_any_cuda_call(lib):
    d = _dims()
    rope = bd.SkvRope(128, 0, 16)
    layer = bd.SkvLayer(*([16] * 9 + [None] * 4))
    call = lambda **kw: lib.shadowkv_decode_step(
        ctypes.byref(d), ctypes.byref(kw.get("rope", rope)), ctypes.byref(kw.get("layer", layer)),
        kw.get("q", 16), 16, 16, kw.get("step", 0), kw.get("out", 16), None, None, kw.get("ws", 256), None)
    assert call(step=16) == bd.SKV_EINVAL                     # w_eff 16 + 16 + 1 > window_cap 32
    assert "window overflow" in lib.shadowkv_last_error().decode()
    assert call(step=-1) == bd.SKV_EINVAL
    assert call(q=0) == bd.SKV_EINVAL
    assert call(q=18) == bd.SKV_EINVAL                        # misaligned
    assert call(ws=0) == bd.SKV_EINVAL
    assert call(ws=272) == bd.SKV_EINVAL                      # workspace needs 256-B alignment
    assert call(rope=bd.SkvRope(127, 0, 16)) == bd.SKV_EINVAL  # odd rotary dim
    assert call(rope=bd.SkvRope(128, 0, 0)) == bd.SKV_EINVAL
    bad = bd.SkvLayer(*([16] * 8 + [0]))
    assert call(layer=bad) == bd.SKV_EINVAL and "V_host" in lib.shadowkv_last_error().decode()
    st = lib.shadowkv_build_cache(ctypes.byref(d), ctypes.byref(rope), ctypes.byref(bad), None, 256, None)
    assert st == bd.SKV_EINVAL
    assert lib.shadowkv_decode_step(None, None, None, 0, 0, 0, 0, 0, None, None, 0, None) == bd.SKV_EINVAL
    partial = bd.SkvLayer(*([16] * 9 + [16, None, 16]))     # value cache: all four pointers or none
    assert call(layer=partial) == bd.SKV_EINVAL and "vc_" in lib.shadowkv_last_error().decode()
    misal = bd.SkvLayer(*([16] * 9 + [16, 24, 16, None, 16]))
    assert call(layer=misal) == bd.SKV_EINVAL and "aligned" in lib.shadowkv_last_error().decode()
    small = bd.SkvLayer(*([16] * 9 + [16, 16, 16, None, 16, 1]))   # capacity below the budget
    assert call(layer=small) == bd.SKV_EINVAL and "vc_capacity" in lib.shadowkv_last_error().decode()
    gen_misal = bd.SkvLayer(*([16] * 9 + [None, None, None, 24]))  # low-rank generated keys (NEXT-4)
    assert call(layer=gen_misal) == bd.SKV_EINVAL and "A_gen" in lib.shadowkv_last_error().decode()


def test_ctypes_layer_struct_matches_header(tmp_path):
    """The binding's skv_layer / skv_dims / skv_rope mirror the header byte for byte (C compiler's view)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "shadowkv.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(skv_layer), offsetof(skv_layer, vc_values),'
                   ' offsetof(skv_layer, vc_stats), sizeof(skv_dims), sizeof(skv_rope), offsetof(skv_dims, ctx_lens_dev)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run([cc, "-I", os.path.dirname(HDR), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [ctypes.sizeof(bd.SkvLayer), bd.SkvLayer.vc_values.offset, bd.SkvLayer.vc_stats.offset,
                   ctypes.sizeof(bd.SkvDims), ctypes.sizeof(bd.SkvRope), bd.SkvDims.ctx_lens_dev.offset]


def test_python_binding_raises_on_error(lib):
    with pytest.raises(bd.ShadowKVError, match="SKV_EINVAL"):
        bd.shadowkv_workspace_bytes(_dims(budget=10_000))


def test_factorize_argument_errors(lib):
    """shadowkv_factorize validates before any CUDA call (S:46 rank range)."""
    ok = bd.dims_struct(1, 8, 8, 128, 4096, 160, 8, 0, 1, 0, 1)
    assert bd.shadowkv_factorize_workspace_bytes(ok) > 1024 * 1024 * 8 * 2   # G fp32 + fp64 at D = 1024
    for kw, status in [(dict(rank=8), bd.SKV_EINVAL), (dict(rank=170), bd.SKV_EINVAL),
                       (dict(n_kv_heads=64), bd.SKV_EUNSUPPORTED), (dict(ctx_len=100), bd.SKV_EINVAL),
                       (dict(head_dim=100), bd.SKV_EUNSUPPORTED)]:
        args = dict(batch=1, n_q_heads=8, n_kv_heads=8, head_dim=128, ctx_len=4096, rank=160, chunk=8,
                    n_outlier=0, budget=1, window_ctx=0, window_cap=1)
        args.update(kw)
        d = bd.SkvDims(**args)
        assert lib.shadowkv_factorize_workspace_bytes(ctypes.byref(d)) == 0
        assert lib.shadowkv_factorize(ctypes.byref(d), 16, 16, 16, None, 256, None) == status
    assert lib.shadowkv_factorize(ctypes.byref(ok), 0, 16, 16, None, 256, None) == bd.SKV_EINVAL
    assert lib.shadowkv_factorize(ctypes.byref(ok), 16, 16, 16, None, 272, None) == bd.SKV_EINVAL


def test_q_len_validation(lib):
    """s_q query tokens (NEXT-3): g * s_q must be a compiled row count; the window must hold s_q new tokens."""
    assert lib.shadowkv_workspace_bytes(ctypes.byref(_dims(q_len=4))) > 0           # g 4 x 4 = 16 rows
    assert lib.shadowkv_workspace_bytes(ctypes.byref(_dims(q_len=3))) == 0           # 12 rows
    assert "q_len" in lib.shadowkv_last_error().decode()
    assert lib.shadowkv_workspace_bytes(ctypes.byref(_dims(q_len=8))) == 0           # 32 rows
    # more rows -> more logits workspace
    assert lib.shadowkv_workspace_bytes(ctypes.byref(_dims(q_len=2))) > lib.shadowkv_workspace_bytes(ctypes.byref(_dims()))
    d = _dims(q_len=4, window_cap=16 + 4)
    rope = bd.SkvRope(128, 0, 16)
    layer = bd.SkvLayer(*([16] * 9 + [None] * 4))
    call = lambda step: lib.shadowkv_decode_step(ctypes.byref(d), ctypes.byref(rope), ctypes.byref(layer), 16, 16, 16,
                                                 step, 16, None, None, 256, None)
    assert call(1) == bd.SKV_EINVAL and "q_len" in lib.shadowkv_last_error().decode()   # 16 + 1 + 4 > 20


def test_ragged_lengths_validation(lib):
    """Ragged batch (NEXT-3): host and device length arrays together; every s_b in [w + c(o + k), ctx_len]."""
    import torch
    mk = lambda t, dev: bd.dims_struct(2, 32, 8, 128, 4096, 160, 8, 4, 8, 16, 40, 1, t, dev)
    lens = torch.tensor([4096, 3000], dtype=torch.int32)
    assert lib.shadowkv_workspace_bytes(ctypes.byref(mk(lens, 64))) > 0
    assert lib.shadowkv_workspace_bytes(ctypes.byref(mk(lens, None))) == 0
    for bad in ([4097, 3000], [4096, 16 + 8 * 12 - 1]):
        assert lib.shadowkv_workspace_bytes(ctypes.byref(mk(torch.tensor(bad, dtype=torch.int32), 64))) == 0
        assert "ctx_lens[" in lib.shadowkv_last_error().decode()
    shortest = torch.tensor([4096, 16 + 8 * 12], dtype=torch.int32)
    assert lib.shadowkv_workspace_bytes(ctypes.byref(mk(shortest, 64))) > 0


def test_shape_window_capacity_for_ragged_and_multi_query():
    """Shape.from_config sizes the window for the largest per-request tail (R8 per request, R29) plus
    steps x q_len generated tokens; dims() carries q_len and the length arrays."""
    cfg = synth.CONFIGS["c1"].replace(batch=3)
    lens = [4096, 3001, 2053]
    sh = Shape.from_config(cfg, steps=5, q_len=2, ctx_lens=lens)
    w_eff = [s - ((s - 16) // 8) * 8 for s in lens]
    assert sh.window_cap == max(w_eff) + 10 and sh.q_len == 2 and sh.ctx_lens == tuple(lens)
    import torch
    lh = torch.tensor(lens, dtype=torch.int32)
    d = sh.dims(lh, 64)
    assert d.q_len == 2 and d.ctx_lens == lh.data_ptr() and d.ctx_lens_dev == 64
    assert Shape.from_config(cfg, steps=5).window_cap == 16 + 5
    # the padded length's tail (4100: w_eff 20) also fits when every request has a shorter tail
    wide = Shape.from_config(cfg.replace(ctx_len=4100), steps=1, ctx_lens=[4096, 2064, 1040])
    assert wide.window_cap == 20 + 1
    assert bd.shadowkv_workspace_bytes(wide.dims()) > 0


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_score_plan_every_config(lib, name):
    """The tcgen05 scorer has a launch plan for every BASELINE config on a 148-SM B200, within its static
    limits (<= 64 tiles of 128 landmarks and <= 4 KV heads per CTA's contiguous tile range)."""
    shp = Shape.from_config(synth.CONFIGS[name])
    grid, tpc, heads, cph = bd.shadowkv_score_plan(shp.dims(), 148)
    tph = -(-shp.n_c // 128)
    assert 1 <= grid and tpc <= 64 and heads <= 4
    assert grid * tpc >= shp.batch * shp.n_kv_heads * tph          # every tile is covered


@pytest.mark.parametrize("ctx", [1 << 21, 1 << 22, (1 << 24) - 65536 - 8])
def test_score_plan_long_single_request(lib, ctx):
    """one request of 2M / 4M tokens (8 KV heads) used to overflow the scorer's 64-tile outlier
    bitmap once a partial-slot limit lowered the grid.  The softmax partials are now per tile (no slot
    limit), so the grid only grows: the tile bound holds at any length the ABI accepts."""
    d = _dims(ctx_len=ctx, budget=ctx // 512, n_outlier=48, window_cap=64)
    grid, tpc, heads, cph = bd.shadowkv_score_plan(d, 148)
    assert tpc <= 64 and heads <= 4
    assert grid * tpc >= 8 * -(-((ctx - 16) // 8) // 128)


def test_score_plan_argument_errors(lib):
    ok = _dims()
    assert lib.shadowkv_score_plan(ctypes.byref(ok), 0, (ctypes.c_int32 * 4)()) == bd.SKV_EINVAL
    assert lib.shadowkv_score_plan(ctypes.byref(_dims(budget=0)), 148, (ctypes.c_int32 * 4)()) == bd.SKV_EINVAL


def test_decode_needs_init_before_any_cuda(lib):
    """Valid arguments on a device shadowkv_init was not called for: SKV_ESTATE, nothing enqueued
    (here: no GPU at all, so no device is ever initialised)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    d = _dims(window_cap=64)
    rope = bd.SkvRope(128, 0, 16)
    layer = bd.SkvLayer(*([16] * 9 + [None] * 4))
    st = lib.shadowkv_decode_step(ctypes.byref(d), ctypes.byref(rope), ctypes.byref(layer), 16, 16, 16, 0, 16, None,
                                  None, 256, None)
    assert st == bd.SKV_ESTATE and "shadowkv_init" in lib.shadowkv_last_error().decode()
    assert lib.shadowkv_init(0) == bd.SKV_ECUDA
