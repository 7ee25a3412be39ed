"""Per-CUDA-source-line stall samples from `ncu -i rep --page source --csv --print-source cuda,sass -k <kernel>`.

python tools/ncu_lines.py src.csv [N]   -> the N source lines with the most warp-stall samples"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg, text, fname, hdr = defaultdict(float), {}, None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].strip().isdigit():
        continue
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    agg[key] += s
    if r[1].strip():
        text[key] = r[1].strip()[:110]
tot = sum(agg.values())
print(f"total stall samples {tot:.0f}")
for key, s in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{s:7.0f} {100 * s / max(tot, 1):5.1f}%  {key[0]}:{key[1]}  {text.get(key, '')}")
