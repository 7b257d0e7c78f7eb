"""Kernel breakdown of one pMG V-cycle (CUPTI via torch.profiler), config 2 by default.

  python tools/pmg_profile.py [--ez 16] [--order 7] [--reps 3]

Prints one JSON line: total device time per V-cycle and per kernel name (summed over the launches
of one V-cycle), and the launch count."""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ez", type=int, default=16)
ap.add_argument("--order", type=int, default=7)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--precision", type=int, default=0)
a = ap.parse_args()
m = mg.box_mesh(16, 16, a.ez, a.order, deform="bubble", dirichlet="all")
ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask)
P = nek.PMG(ctx, m.xyz, 1.0, 0.0, **({"precision": a.precision} if a.precision else {}))
r = torch.from_numpy(mg.smooth_field(m, seed=1)).cuda()
z = torch.empty_like(r)
for _ in range(3):
    P.apply(r, z)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        P.apply(r, z)
    torch.cuda.synchronize()
path = "/tmp/pmg_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    name = e["name"].split("(")[0].replace("void ", "").replace("nekb200::", "")
    grid = e["args"].get("grid")
    key = f"{name} grid={grid}"
    agg[key][0] += 1
    agg[key][1] += e["dur"]
tot = sum(v[1] for v in agg.values()) / a.reps
rows = sorted(((k, v[0] // a.reps, round(v[1] / a.reps, 1)) for k, v in agg.items()), key=lambda t: -t[2])
print(json.dumps({"E": m.E, "N": m.N, "us_per_vcycle_kernels": round(tot, 1),
                  "launches_per_vcycle": sum(r_[1] for r_ in rows), "by_kernel": rows[:40]}))
P.free()
nek.free(ctx)
