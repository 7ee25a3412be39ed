"""ShadowKV (arXiv 2410.21465) decode-time sparse attention for B200 (sm_100a).

The hot path lives in ``lib/libshadowkv.so`` (CUDA C, C ABI in include/shadowkv.h);
``binding`` is a ctypes marshalling layer and ``state`` allocates the per-layer tensors.
"""
from . import binding  # noqa: F401
from .state import LayerState, RopeTable, Shape, alloc_workspace, factorize  # noqa: F401
