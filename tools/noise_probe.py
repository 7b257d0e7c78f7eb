"""Rounding-sensitivity probe of the oracle's Jacobi-PCG (reading 17 yardsticks): how far the
||b||-normalised residual history moves when only the rounding of the inner products (Dot2 vs plain
recursive summation) or of the vector updates (fma vs separate multiply and add) changes."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle  # noqa: E402
from workloads import meshgen as mg  # noqa: E402

case = sys.argv[1]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
if case == "cfg2":
    m = mg.config_mesh(2)
elif case == "N12":
    m = mg.box_mesh(2, 2, 1, 12, deform="bubble", dirichlet="top")
else:
    m = mg.box_mesh(8, 8, 8, 7, deform="bubble", dirichlet="all")
O = oracle.Oracle.from_mesh(m)
uu, f = mg.manufactured(m)
b = oracle.mask(m.mask, O.gs_apply(O.wJ * f)) if case != "N12" else mg.smooth_field(m, seed=3)
L = oracle.lib()
L.or_set_upd_fma.argtypes = [ctypes.c_int]
runs = {}
for name, dm, uf in (("dot2_fma", 0, 1), ("dot2_plain", 0, 0), ("plain_fma", 2, 1), ("plain_plain", 2, 0)):
    L.or_set_upd_fma(uf)
    _, it, _, h = O.pcg(1.0, 0.0, b, tol, K, dot_mode=dm)
    runs[name] = h
L.or_set_upd_fma(0)
ref = runs["dot2_fma"]
for k, h in runs.items():
    n = min(len(h), len(ref))
    d = np.abs(h[:n] - ref[:n])
    print(f"{case} K={K}: {k:12s} vs dot2_fma: iters {len(h) - 1}, max |d hist| {d.max():.2e} at k={d.argmax()}")
