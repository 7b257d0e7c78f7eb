"""World-size-2 (and 3) multi-process test of the N>1 host path on CPU (gloo).

Each process plays one rank: it builds its element partition, runs the
library's host planner (nek_plan_*), exchanges surface gids with an
all_gather over gloo -- the setup collective nek_setup performs over NCCL --
then carries out the halo exchange the plan prescribes with gloo send/recv
and the rank-ordered sums; the result must equal the oracle's multi-rank
gather-scatter bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, split, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2409_19119_b200 import nek
        from workloads import meshgen as mg
        m = mg.box_mesh(4, 3, 6, 3, deform="bubble", dirichlet="zends")
        parts = mg.slab_partition(m, world) if split == "slab" else mg.block_partition(m, world, 1, 1)
        sub = mg.submesh(m, parts[rank])
        plan = nek.Plan(sub.E, sub.N, sub.gid, sub.mask, sub.xyz)
        mine = plan.surface_gids()
        lists = [None] * world
        dist.all_gather_object(lists, mine)
        plan.set_ranks(rank, world, lists)
        P3 = m.Nq ** 3
        v = mg.random_evector(m, seed=9)[(parts[rank][:, None] * P3 + np.arange(P3)).reshape(-1)]
        # local-only runs
        out = v.copy()
        pm, po = plan.get(nek.PLAN_PERM), plan.get(nek.PLAN_OFFS)
        for x in range(po.size - 1):
            c = pm[po[x]:po[x + 1]]
            s = v[c[0]]
            for t in c[1:]:
                s = s + v[t]
            out[c] = s
        # interface partials, packed per neighbour in the plan's slot order
        ip, io = plan.get(nek.PLAN_IFC_PERM), plan.get(nek.PLAN_IFC_OFFS)
        part = np.zeros(io.size - 1)
        for x in range(io.size - 1):
            c = ip[io[x]:io[x + 1]]
            s = v[c[0]]
            for t in c[1:]:
                s = s + v[t]
            part[x] = s
        nb, so, sr = plan.get(nek.PLAN_NEIGHBORS), plan.get(nek.PLAN_SEND_OFFS), plan.get(nek.PLAN_SEND_RUN)
        send = torch.from_numpy(part[sr].copy())
        recv = torch.zeros(so[-1] if so.size else 0, dtype=torch.float64)
        reqs = []
        for k, qr in enumerate(nb):
            reqs.append(dist.isend(send[so[k]:so[k + 1]].contiguous(), int(qr)))
        bufs = []
        for k, qr in enumerate(nb):
            b = torch.zeros(int(so[k + 1] - so[k]), dtype=torch.float64)
            reqs.append(dist.irecv(b, int(qr)))
            bufs.append((k, b))
        for rq in reqs:
            rq.wait()
        for k, b in bufs:
            recv[so[k]:so[k + 1]] = b
        recv = recv.numpy()
        co, cb = plan.get(nek.PLAN_CONTRIB_OFFS), plan.get(nek.PLAN_CONTRIB)
        for x in range(io.size - 1):
            terms = [part[x] if s_ < 0 else recv[s_] for s_ in cb[co[x]:co[x + 1]]]
            s = terms[0]
            for t in terms[1:]:
                s = s + t
            out[ip[io[x]:io[x + 1]]] = s
        allv = [None] * world
        dist.all_gather_object(allv, (out, v, sub.gid))
        if rank == 0:
            ref = oracle.gs_multi([a[2] for a in allv], [a[1] for a in allv])
            q.put(all(np.array_equal(a[0], b) for a, b in zip(allv, ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,split", [(2, "slab"), (3, "slab"), (2, "block")])
def test_gloo_halo_exchange(world, split):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, split, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
