"""Top stall SASS lines of one kernel in an ncu report (source page, sass view).

  python tools/ncu_hot.py <report.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[2:]:
    if len(r) != len(h):
        continue
    try:
        s = float(r[si] or 0)
    except ValueError:
        continue
    st = {c: float(r[h.index(c)] or 0) for c in cols}
    data.append((s, r[0], r[1], st))
tot = sum(d[0] for d in data) or 1.0
print(f"total samples {tot:.0f}")
for s, addr, src, st in sorted(data, key=lambda d: -d[0])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{100 * s / tot:5.1f}% {addr} {src[:70]:70s} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in big))
