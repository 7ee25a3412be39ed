"""SASS instruction counts per kernel of the built libshadowkv.so (cuobjdump -sass; runs without a GPU).

    python tools/sass_counts.py [--lib PATH] [--out profiles/<tag>_sass_tensor_ops.txt]

UTCHMMA = tcgen05.mma kind::f16, LDTM = tcgen05.ld, UTCBAR = tcgen05.commit, UTMALDG = TMA tensor load,
UBLKCP = cp.async.bulk, HMMA = mma.sync, FFMA = CUDA-core fp32 FMA, STL/LDL = local-memory spill traffic.
"""
from __future__ import annotations

import argparse
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2410_21465_b200", "lib", "libshadowkv.so")
OPS = ("UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "HMMA", "FFMA", "SYNCS", "STL", "LDL")
_FUNC = re.compile(r"Function : (\S+)")
_INSN = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)")


def sass_counts(lib: str = LIB) -> dict[str, dict[str, int]]:
    """{mangled kernel name: {opcode family: count}} for every kernel in the library."""
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    counts: dict[str, dict[str, int]] = {}
    cur = None
    for line in out.splitlines():
        m = _FUNC.search(line)
        if m:
            cur = counts.setdefault(m.group(1), {op: 0 for op in OPS})
            continue
        if cur is None:
            continue
        m = _INSN.search(line)
        if m:
            op = m.group(1).split(".")[0]
            if op in cur:
                cur[op] += 1
    return counts


def kernels(counts: dict, stem: str) -> dict[str, dict[str, int]]:
    """The entries whose mangled name carries the kernel name `stem` (e.g. 'k_sparse_attn')."""
    tag = f"{len(stem)}{stem}"
    return {k: v for k, v in counts.items() if tag in k}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=LIB)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c = sass_counts(a.lib)
    lines = [__doc__.strip().splitlines()[0], ""]
    for k, v in c.items():
        nz = " ".join(f"{op}={n}" for op, n in v.items() if n)
        lines.append(f"{k[:90]:90s} {nz}")
    text = "\n".join(lines) + "\n"
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
