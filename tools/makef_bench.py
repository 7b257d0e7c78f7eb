"""makef (NEXT #4) throughput on one GPU: CUDA-event time per apply (L2 flushed), algorithmic
bytes (u, v, w in; 9 M^3 lattice factors; 3 outputs) and flops of the sum-factorised algorithm,
against the measured copy peak and the measured FP64 FMA peak (nek_probe_dfma_tflops).

  python tools/makef_bench.py [--ez 16] [--order 7] [--reps 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402


def makef_cost(N):
    """(bytes, flops) per element of the implemented algorithm (reading M4)."""
    a = N + 1
    m = (3 * a + 1) // 2
    i_st, j_st, k_st = a * a * m * a, a * m * m * a, m ** 3 * a
    fma = 3 * (i_st + j_st + k_st) + 9 * m ** 3                      # U at the lattice, Ut
    fma += 3 * (2 * i_st + 3 * j_st + 3 * k_st + 3 * m ** 3 + (k_st + a * a * m * m + i_st))
    byts = 8 * (3 * a ** 3 + 9 * m ** 3 + 3 * a ** 3)
    return byts, 2 * fma


def run(ez, order, reps, peak_tf):
    m = mg.box_mesh(16, 16, ez, order, deform="bubble", dirichlet="all")
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask)
    K = nek.Makef(ctx, m.xyz)
    U = [torch.from_numpy(mg.smooth_field(m, seed=s)).cuda() for s in (1, 2, 3)]
    F = [torch.empty_like(U[0]) for _ in range(3)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        K.apply(*U, *F)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); K.apply(*U, *F); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    b, f = makef_cost(order)
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    gbs = b * m.E / (ms * 1e-3) / 1e9
    tfs = f * m.E / (ms * 1e-3) / 1e12
    out = {"E": m.E, "N": order, "M": K.M, "ms": ms, "gdof_per_s": m.n_dof / (ms * 1e-3) / 1e9,
           "algorithmic_GBps": gbs, "hbm_frac": gbs / hbm, "algorithmic_TFLOPs": tfs, "fp64_peak_TFLOPs": peak_tf,
           "fp64_frac": tfs / peak_tf, "flop_per_byte": f / b}
    K.free()
    nek.free(ctx)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ez", type=int, default=16)
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    peak = nek.probe_fp64_tflops(0)
    print(json.dumps(run(a.ez, a.order, a.reps, peak)))
