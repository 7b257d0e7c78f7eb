"""Config 5 (BASELINE configs[4]) on one GPU: N = 3..9 at ~20M DOF, nek_ax (Ax + gs) with the
per-kernel event timing of the library; prints one JSON line per N with GDOF/s and the Ax
kernel's algorithmic GB/s (u, 6 factors, w per local point) against the measured HBM peak."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402

# SURVEY 8(d) config 5 boxes (n ~ 20M DOF)
BOXES = {3: (88, 96, 88), 4: (66, 74, 64), 5: (53, 54, 56), 6: (44, 44, 48), 7: (38, 38, 40), 8: (32, 38, 32),
         9: (29, 30, 32)}
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
orders = [int(a) for a in sys.argv[1:]] or sorted(BOXES)
for N in orders:
    Ex, Ey, Ez = BOXES[N]
    m = mg.box_mesh(Ex, Ey, Ez, N, deform="bubble", dirichlet="all")
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask)
    variant = int(os.environ.get("NSWEEP_VARIANT", "0"))
    if variant:
        nek.set_variant(ctx, variant)
    u = torch.from_numpy(mg.smooth_field(m, 1)).cuda()
    w = torch.empty_like(u)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        nek.ax(ctx, 1.0, 0.0, u, w)
    nek.set_timing(ctx, True)
    nek.get_stats(ctx, reset=True)
    reps = 10
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        nek.ax(ctx, 1.0, 0.0, u, w)
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    st = nek.get_stats(ctx, reset=True)
    ax_ms = st["ax_ms"] / st["ax_launches"]
    gbs = st["ax_bytes"] / st["ax_launches"] / (ax_ms * 1e-3) / 1e9
    print(json.dumps({"N": N, "variant": variant, "box": [Ex, Ey, Ez], "n_dof": m.n_dof, "n_local": m.n_local,
                      "ax_gs_gdof_per_s": m.n_dof * reps / (tot * 1e-3) / 1e9, "ax_ms": ax_ms,
                      "gs_ms": st["gs_ms"] / max(1, st["gs_launches"]), "ax_GBps": gbs, "ax_frac_of_peak": gbs / peak}),
          flush=True)
    nek.free(ctx)
    del m, u, w
