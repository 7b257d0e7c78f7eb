"""Loopback group workload for ncu: two virtual ranks on one GPU, each with the config-2 per-GPU problem
(16x16x16 elements, N = 7; z-slabs of a 16x16x32 box), a few eager PCG iterations (loopback launches
directly, no graph)."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402

P = int(os.environ.get("LB_P", "2"))
iters = int(os.environ.get("LB_ITERS", "6"))
m = mg.box_mesh(16, 16, 16 * P, 7, deform="bubble", dirichlet="all")
parts = mg.slab_partition(m, P)
subs = [mg.submesh(m, p) for p in parts]
b = mg.smooth_field(m, seed=1)
lb = nek.Loopback(P, 0)
P3 = m.Nq ** 3


def rank(r):
    s = subs[r]
    loc = (np.asarray(parts[r])[:, None] * P3 + np.arange(P3)).reshape(-1)
    ctx = nek.setup(s.E, s.N, s.xyz, s.gid, s.mask, comm=lb.comm(r), device=0)
    x = np.zeros(s.n_local)
    for _ in range(2):
        nek.pcg_solve(ctx, 1.0, 0.0, b[loc], x, 0.0, iters)
    nek.free(ctx)


th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
lb.free()
print("ok")
