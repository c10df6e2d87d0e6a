"""Summarise ncu reports (--set full) and launch lists into markdown for profiles/.

usage: python tools/ncu_summary.py OUT.md REPORT.ncu-rep[:label] ... [--launches LIST.csv[:label]]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem / block"),
]


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3}


def report_rows(path):
    """Rows of an .ncu-rep (via ncu -i) or of its `--page raw --csv` export."""
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                d[label] = f"{r[i]} {units[i]}".strip()
        try:  # achieved DRAM bandwidth of the launch: (read + write) / duration
            val = lambda k: float(r[h.index(k)].replace(",", "")) * SCALE[units[h.index(k)]]
            gbs = (val("dram__bytes_read.sum") + val("dram__bytes_write.sum")) / val("gpu__time_duration.sum") / 1e9
            d["DRAM GB/s (read + write / duration)"] = f"{gbs:.0f}"
        except (ValueError, KeyError):
            pass
        stalls = [(h[i], r[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h[i].endswith("_not_issued")]
        stalls = sorted(((float(v.replace(",", "") or 0), k.split("stalled_")[-1]) for k, v in stalls), reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        d["top stalls"] = ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in stalls[:4])
        out.append(d)
    return out


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0][:90]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    return lines


def main():
    out = sys.argv[1]
    args = sys.argv[2:]
    md = []
    mode = "rep"
    for a in args:
        if a == "--launches":
            mode = "launch"
            continue
        path, _, label = a.partition(":")
        if mode == "launch":
            md += [f"## Launch list: {label or path}", "", f"source: `{path}` "
                   "(ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised: compare shares)",
                   ""] + launches(path) + [""]
            continue
        md += [f"## {label or path}", "", f"source: `{path}` (ncu --set full --clock-control none --import-source on)", ""]
        for d in report_rows(path):
            md.append(f"### `{d.pop('kernel')[:110]}`")
            md.append("")
            md += ["| metric | value |", "|---|---|"] + [f"| {k} | {v} |" for k, v in d.items()] + [""]
    open(out, "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
