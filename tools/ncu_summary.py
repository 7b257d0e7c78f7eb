"""Summarise ncu artefacts into markdown for profiles/.

  python tools/ncu_summary.py launches <launches.csv>      per-kernel mean/min duration and share
  python tools/ncu_summary.py full <report.ncu-rep>        key --set full metrics per profiled kernel
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("nekb200::", "")
        agg.setdefault(name, []).append(float(r[vi]) / 1000.0)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | min us | share of listed time |")
    print("|---|---|---|---|---|")
    for k, v in agg.items():
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {min(v):.2f} | {100 * sum(v) / tot:.1f}% |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6,
             "ns": 1e-3, "us": 1.0, "ms": 1e3}
    print("| kernel | " + " | ".join(lbl for _, lbl in FULL_METRICS) + " | top stalls |")
    print("|---|" + "---|" * (len(FULL_METRICS) + 1))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = []
        for m, _ in FULL_METRICS:
            if m not in h:
                vals.append("-")
                continue
            k = h.index(m)
            v = r[k]
            if units[k] in scale and v not in ("", "n/a"):   # MB for bytes, us for times
                v = f"{float(v.replace(',', '')) * scale[units[k]]:.2f}"
            vals.append(v)
        st = [(h[k].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[k] or 0)) for k in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[k] and "not_issued" not in h[k]]
        tot = sum(v for _, v in st) or 1.0
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:3])
        print(f"| `{name}` | " + " | ".join(vals) + f" | {top} |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
