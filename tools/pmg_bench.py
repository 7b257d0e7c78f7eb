"""Time-to-solution: Jacobi-PCG vs pMG-PCG (NEXT #1) on one GPU.

  python tools/pmg_bench.py [--ez 16] [--order 7] [--tol 1e-8] [--h2 0] [--orders 7,5,3,1]
         [--degree 6] [--coarse-degree 20] [--reps 3]

Prints one JSON line per preconditioner: iterations, ms per solve (CUDA events, median of reps),
ms per iteration, and for pMG the ms per V-cycle (apply alone)."""
import argparse
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
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--h2", type=float, default=0.0)
ap.add_argument("--orders", default="")
ap.add_argument("--degree", type=int, default=0)
ap.add_argument("--coarse-degree", type=int, default=0)
ap.add_argument("--coarse-lo", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mesh", default="box")
ap.add_argument("--precision", type=int, default=0)
a = ap.parse_args()
if a.mesh == "rod":
    m = mg.rod_bundle(17, 17, 3, a.order, dirichlet="outlet" if a.h2 == 0 else "pins_walls")
else:
    m = mg.box_mesh(16, 16, a.ez, a.order, deform="bubble", dirichlet="all")
ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask)
b = torch.from_numpy(mg.smooth_field(m, seed=1)).cuda()
x = torch.zeros_like(b)
orders = [int(v) for v in a.orders.split(",")] if a.orders else None
t0 = torch.cuda.Event(True); t1 = torch.cuda.Event(True)
P = nek.PMG(ctx, m.xyz, 1.0, a.h2, orders=orders, degree=a.degree, coarse_degree=a.coarse_degree,
            coarse_lo=a.coarse_lo, precision=a.precision)


def timed(fn):
    out, ts = None, []
    for _ in range(a.reps):
        t0.record(); out = fn(); t1.record(); t1.synchronize()
        ts.append(t0.elapsed_time(t1))
    ts.sort()
    return out, ts[len(ts) // 2]


nek.pcg_solve(ctx, 1.0, a.h2, b, x, a.tol, 20000)
(st, it, rr, _), ms = timed(lambda: nek.pcg_solve(ctx, 1.0, a.h2, b, x, a.tol, 20000))
print(json.dumps({"pc": "jacobi", "E": m.E, "N": m.N, "n_dof": m.n_dof, "tol": a.tol, "iters": it, "relres": rr,
                  "ms": ms, "ms_per_iter": ms / max(it, 1)}), flush=True)
P.solve(b, x, a.tol, 2000)
(st, it, rr, _), ms = timed(lambda: P.solve(b, x, a.tol, 2000))
z = torch.empty_like(b)
P.apply(b, z)
_, mv = timed(lambda: P.apply(b, z))
info = P.info()
print(json.dumps({"pc": "pmg", "precision": info["precision"], "orders": info["orders"], "degree": info["degree"],
                  "coarse_degree": info["coarse_degree"], "lam_max": info["lam_max"], "lam_min": info["lam_min"],
                  "iters": it, "relres": rr, "ms": ms, "ms_per_iter": ms / max(it, 1), "ms_per_vcycle": mv}),
      flush=True)
P.free()
nek.free(ctx)
