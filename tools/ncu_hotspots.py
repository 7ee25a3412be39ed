"""Top SASS hotspots from `ncu --page source --csv` output: python tools/ncu_hotspots.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
def num(x):
    try:
        return float(x)
    except ValueError:
        return None


data = [r for r in rows[2:] if len(r) > 4 and num(r[hdr.index("Warp Stall Sampling (All Samples)")]) is not None]
ia, isrc, ist, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot_s = sum(float(r[ist] or 0) for r in data)
tot_e = sum(float(r[iex] or 0) for r in data)
print(f"total stall samples {tot_s:.0f}, instructions executed {tot_e:.0f}")
for r in sorted(data, key=lambda r: -float(r[ist] or 0))[:n]:
    print(f"{r[ia]:>6s} {float(r[ist] or 0):7.0f} {float(r[iex] or 0):9.0f}  {r[isrc][:100]}")
