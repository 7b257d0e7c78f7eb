"""Workload for compute-sanitizer: every kernel family of the hot path on small meshes.

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py [--loopback]

Config 1 (N=3, Ax v6), a 6x6x6 N=7 box (Ax v5 DMMA kernel, fused PCG, L2-keep path), N=5;
nek_ax / nek_gs / nek_pcg_solve (graph), pMG-PCG (FP64 and FP32), projection, makef.  With
--loopback the same on 2 virtual ranks on one GPU (halo pack/unpack and mailbox kernels).
Prints one line per case; exit status 0 when every call returned NEK_OK / NEK_MAXIT.
"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402


def run_case(name, m, comm=None, sub_of=None):
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, comm=comm, device=0)
    u = mg.random_evector(m, seed=1)
    w = np.zeros_like(u)
    nek.ax(ctx, 1.0, 0.3, u, w)
    v = u.copy()
    nek.gs(ctx, v)
    b = mg.smooth_field(m, seed=3)
    x = np.zeros_like(b)
    st, it, rr, _ = nek.pcg_solve(ctx, 1.0, 0.0, b, x, 0.0, 12, want_hist=True)
    if m.N <= 9:
        P = nek.PMG(ctx, m.xyz, 1.0, 0.0)
        xp = np.zeros_like(b)
        P.solve(b, xp, 1e-6, 3)
        P.free()
        P32 = nek.PMG(ctx, m.xyz, 1.0, 0.0, precision=1)
        P32.solve(b, xp, 1e-6, 2)
        P32.free()
    pr = nek.Projection(ctx, 4)
    for k in range(3):
        pr.solve(1.0, 0.0, b * (1 + 0.1 * k), x, 1e-8, 50)
    pr.free()
    if comm is None and m.N <= 9:
        mk = nek.Makef(ctx, m.xyz)
        f = [np.zeros_like(u) for _ in range(3)]
        mk.apply(u, u * 0.5, u * 0.25, *f)
        mk.free()
    nek.free(ctx)
    print(f"{name}: ok (pcg status {st}, {it} it)", flush=True)


def main():
    loop = "--loopback" in sys.argv
    meshes = [("cfg1_N3", mg.config_mesh(1)),
              ("box6_N7", mg.box_mesh(6, 6, 6, 7, deform="bubble")),
              ("box3_N5", mg.box_mesh(3, 3, 4, 5, deform="sin", eps=0.05, dirichlet="zends"))]
    if not loop:
        for name, m in meshes:
            run_case(name, m)
        return 0
    P = 2
    for name, m in meshes:
        parts = mg.slab_partition(m, P)
        g = nek.Loopback(P)
        errs = []

        def work(r):
            try:
                run_case(f"{name}_rank{r}", mg.submesh(m, parts[r]), comm=g.comm(r))
            except Exception as e:  # noqa: BLE001
                errs.append(f"rank {r}: {e}")
                g.abort()
        th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        g.free()
        if errs:
            print("\n".join(errs))
            return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
