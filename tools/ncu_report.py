"""Summarise an ncu --set full report (raw page) into markdown + the traffic JSON bench.py reads.

python tools/ncu_report.py gpurun_out/<tag>_prof.ncu-rep profiles/<tag>_ncu_summary.md [config, default c2]"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("pcie__read_bytes.sum.per_second", "PCIe read (during kernel)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main(rep, out_md, config="c2"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(cold caches, serialised replays: compare shares, not absolutes).", ""]
    traffic = {}
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append(f"| top stall reasons (samples) | {', '.join(f'{n} {int(v)}' for v, n in stalls[:5])} |")
        lines.append("")

        def val(m):
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            u = units[i]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return v * scale
        key = "sparse_attn" if "sparse_attn" in name else ("score" if "score" in name else ("select" if "select" in name else name))
        try:
            traffic[f"{key}_dram_bytes"] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        except (ValueError, KeyError):
            pass
        try:   # host-link bytes of the kernel (PCIe read rate x duration)
            dur_s = val("gpu__time_duration.sum") * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(
                units[hdr.index("gpu__time_duration.sum")], 1e-9)
            i = hdr.index("pcie__read_bytes.sum.per_second")
            pre = units[i].split("byte")[0]
            rate = float(r[i].replace(",", "")) * {"": 1, "K": 1e3, "M": 1e6, "G": 1e9, "T": 1e12}.get(pre, 1)
            traffic[f"{key}_pcie_read_bytes"] = rate * dur_s
        except (ValueError, KeyError):
            pass
    open(out_md, "w").write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
    traffic["source"] = os.path.basename(rep)
    traffic["config"] = config
    json.dump(traffic, open(tj, "w"), indent=1)
    print(open(out_md).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "c2")
