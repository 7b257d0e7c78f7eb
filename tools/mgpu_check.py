"""Multi-GPU parity check (run under torchrun, one process per GPU).

Each rank owns a z-slab (or a block) of the elements of one mesh, sets up the
library with an NCCL communicator, and runs nek_ax, nek_gs and nek_pcg_solve.
Rank 0 gathers the per-rank results and compares them with the CPU oracle on
the whole mesh (single-rank oracle; gs also against the oracle's multi-rank
emulation, bit for bit).  Prints one JSON line on rank 0 and exits non-zero on
failure.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    results = {}
    ok = True
    cases = [("slab_N7", lambda: mg.box_mesh(4, 3, 2 * world, 7, deform="bubble"), "slab"),
             ("slab_N3", lambda: mg.box_mesh(3, 3, 2 * world, 3, deform="sin", eps=0.05, dirichlet="zends"), "slab"),
             ("block_N5", lambda: mg.box_mesh(4, 4, 4, 5, deform="bubble"), "block")]
    for name, mk, kind in cases:
        m = mk()
        if kind == "slab":
            parts = mg.slab_partition(m, world)
        else:
            if world == 2:
                parts = mg.block_partition(m, 2, 1, 1)
            elif world == 4:
                parts = mg.block_partition(m, 2, 2, 1)
            else:
                parts = mg.block_partition(m, 2, 2, 2)
        sub = mg.submesh(m, parts[rank])
        ctx = nek.setup(sub.E, sub.N, sub.xyz, sub.gid, sub.mask, comm=nek.comm_from_torch(dev), device=local)
        info = nek.get_info(ctx)
        P3 = m.Nq ** 3
        loc = (parts[rank][:, None] * P3 + np.arange(P3)).reshape(-1)
        u = mg.random_evector(m, seed=5)[loc]
        ud = torch.from_numpy(u).to(dev)
        wd = torch.empty_like(ud)
        nek.ax(ctx, 1.0, 0.3, ud, wd)
        vd = ud.clone()
        nek.gs(ctx, vd)
        b = mg.smooth_field(m, seed=3)[loc]
        xd = torch.zeros_like(ud)
        st, it, rr, hist = nek.pcg_solve(ctx, 1.0, 0.0, torch.from_numpy(b).to(dev), xd, 0.0, 40, want_hist=True)
        # p-multigrid (NEXT #1): one V-cycle of M QQ^T u and a converged pMG-PCG solve
        P = nek.PMG(ctx, sub.xyz, 1.0, 0.0)
        rd = vd.clone()
        rd[torch.from_numpy(sub.mask != 0).to(dev)] = 0.0
        zd = torch.empty_like(rd)
        P.apply(rd, zd)
        xpd = torch.zeros_like(ud)
        pst, pit, prr, _ = P.solve(torch.from_numpy(b).to(dev), xpd, 1e-10, 200)
        pinfo = P.info()
        P.free()
        P32 = nek.PMG(ctx, sub.xyz, 1.0, 0.0, precision=1)       # FP32 preconditioner (NEXT #3)
        x32d = torch.zeros_like(ud)
        pst32, pit32, _, _ = P32.solve(torch.from_numpy(b).to(dev), x32d, 1e-10, 200)
        P32.free()
        torch.cuda.synchronize()
        payload = {"w": wd.cpu().numpy(), "v": vd.cpu().numpy(), "x": xd.cpu().numpy(), "hist": hist, "it": it,
                   "info": info, "z": zd.cpu().numpy(), "xp": xpd.cpu().numpy(), "pit": pit, "pst": pst,
                   "lam": pinfo["lam_max"] + pinfo["lam_min"], "x32": x32d.cpu().numpy(), "pit32": pit32,
                   "pst32": pst32}
        gathered = [None] * world
        dist.all_gather_object(gathered, payload)
        if rank == 0:
            import oracle
            O = oracle.Oracle.from_mesh(m)
            uf = mg.random_evector(m, seed=5)
            wref = O.apply(1.0, 0.3, uf)
            wgot = np.zeros(m.n_local); vgot = np.zeros(m.n_local); xgot = np.zeros(m.n_local)
            for r_, pl in enumerate(gathered):
                lr = (parts[r_][:, None] * P3 + np.arange(P3)).reshape(-1)
                wgot[lr] = pl["w"]; vgot[lr] = pl["v"]; xgot[lr] = pl["x"]
            ax_err = float(np.abs(wgot - wref).max() / np.abs(wref).max())
            gs_ref_multi = oracle.gs_multi([mg.submesh(m, p).gid for p in parts],
                                           [uf[(p[:, None] * P3 + np.arange(P3)).reshape(-1)] for p in parts])
            gs_bit = all(np.array_equal(pl["v"], gr) for pl, gr in zip(gathered, gs_ref_multi))
            gs_err = float(np.abs(vgot - O.gs_apply(uf)).max() / np.abs(O.gs_apply(uf)).max())
            bf = mg.smooth_field(m, seed=3)
            xo, ito, sto, ho = O.pcg(1.0, 0.0, bf, 0.0, 40)
            tol = O.hist_tolerance(1.0, 0.0, bf, 40)
            h0 = gathered[0]["hist"]
            hist_ok = bool(np.all(np.abs(h0 - ho) <= tol)) and all(np.array_equal(pl["hist"], h0) for pl in gathered)
            x_err = float(np.abs(xgot - xo).max() / np.abs(xo).max())
            # copies of a node bit-identical across ranks
            allg = np.concatenate([mg.submesh(m, p).gid for p in parts])
            allw = np.concatenate([pl["w"] for pl in gathered])
            order = np.argsort(allg, kind="stable")
            sg, sw = allg[order], allw[order]
            same = np.all((sg[1:] != sg[:-1]) | (sw[1:] == sw[:-1]))
            # pMG against the single-rank oracle hierarchy on the whole mesh
            from oracle import pmg as opmg
            Po = opmg.PMG(O, m.xyz, 1.0, 0.0)
            lam_o = [L.lam_max for L in Po.levels] + [L.lam_min for L in Po.levels]
            lam_diff = max(abs(a - b_) / max(lam_o[:len(Po.levels)]) for pl in gathered for a, b_ in zip(pl["lam"], lam_o))
            rf = oracle.mask(m.mask, O.gs_apply(uf))
            zref = Po.apply(rf)
            zgot = np.zeros(m.n_local); xpgot = np.zeros(m.n_local); x32got = np.zeros(m.n_local)
            for r_, pl in enumerate(gathered):
                lr = (parts[r_][:, None] * P3 + np.arange(P3)).reshape(-1)
                zgot[lr] = pl["z"]; xpgot[lr] = pl["xp"]; x32got[lr] = pl["x32"]
            z_err = float(np.abs(zgot - zref).max() / np.abs(zref).max())
            xpo, pito, psto, _ = opmg.pcg(O, 1.0, 0.0, bf, 1e-10, 200, Po.apply)
            xp_err = float(np.abs(xpgot - xpo).max() / np.abs(xpo).max())
            x32_err = float(np.abs(x32got - xpo).max() / np.abs(xpo).max())
            pmg_ok = (lam_diff <= 1e-9 and z_err <= max(1e-11, 100 * lam_diff) and xp_err <= 1e-8
                      and all(abs(pl["pit"] - pito) <= 1 and pl["pst"] == 0 for pl in gathered)
                      and x32_err <= 1e-8 and all(pl["pit32"] <= pito + 2 and pl["pst32"] == 0 for pl in gathered))
            case_ok = (ax_err <= 1e-12 and gs_bit and gs_err <= 1e-14 and hist_ok and x_err <= 1e-10 and bool(same)
                       and pmg_ok)
            ok &= case_ok
            results[name] = {"ax_err": ax_err, "gs_bitexact_vs_multirank_oracle": gs_bit, "gs_err_vs_1rank": gs_err,
                             "hist_ok": hist_ok, "x_err": x_err, "copies_identical": bool(same), "iters": ito,
                             "halo_doubles": [pl["info"]["halo_doubles"] for pl in gathered],
                             "neighbors": [pl["info"]["n_neighbors"] for pl in gathered],
                             "transport": [pl["info"]["transport"] for pl in gathered],
                             "pmg": {"lam_diff": lam_diff, "vcycle_err": z_err, "x_err": xp_err, "iters_oracle": pito,
                                     "iters": [pl["pit"] for pl in gathered], "fp32_x_err": x32_err,
                                     "fp32_iters": [pl["pit32"] for pl in gathered], "ok": bool(pmg_ok)},
                             "ok": case_ok}
        nek.free(ctx)
    if rank == 0:
        print(json.dumps({"world": world, "ok": bool(ok), "cases": results}))
    okt = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(okt, 0)
    dist.destroy_process_group()
    return 0 if okt.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
