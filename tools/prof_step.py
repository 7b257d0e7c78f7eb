"""Short workload for ncu: cfg2 (16^3, N=7) setup, then `--solves` PCG solves of
`--iters` iterations (eager launches, no graph) and `--ax` nek_ax calls."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2409_19119_b200 import nek
from workloads import meshgen as mg

ap = argparse.ArgumentParser()
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--ax", type=int, default=3)
ap.add_argument("--h2", type=float, default=0.0)
ap.add_argument("--ez", type=int, default=16)
ap.add_argument("--order", type=int, default=7)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--flush", action="store_true", help="write 256 MiB before every nek_ax (cold L2)")
a = ap.parse_args()
m = mg.box_mesh(16, 16, a.ez, a.order, deform="bubble", dirichlet="all")
ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask)
nek.set_variant(ctx, a.variant)
nek.set_timing(ctx, True)   # eager launches (one kernel per node in the profile)
b = torch.from_numpy(mg.smooth_field(m, 1)).cuda()
x = torch.zeros_like(b)
w = torch.empty_like(b)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.ax):
    if a.flush:
        flush.fill_(1)
    nek.ax(ctx, 1.0, a.h2, b, w)
for _ in range(a.solves):
    nek.pcg_solve(ctx, 1.0, a.h2, b, x, 0.0, a.iters)
torch.cuda.synchronize()
print(nek.get_stats(ctx))
nek.free(ctx)
