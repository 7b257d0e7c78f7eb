"""CPU-only checks of the product library: it loads, exports every symbol that
include/nek.h declares, and its host planner (no GPU needed) builds gather-
scatter maps byte-equal to the oracle's, single- and multi-rank."""
import os
import re

import numpy as np
import pytest

import oracle
from workloads import meshgen as mg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nek():
    from paper_2409_19119_b200 import build
    build.build()
    from paper_2409_19119_b200 import nek as _nek
    return _nek


def test_header_symbols_exported(nek):
    hdr = open(os.path.join(ROOT, "include", "nek.h")).read()
    decl = set(re.findall(r"\b(nek_[a-z_]+)\s*\(", hdr))
    assert len(decl) >= 20
    import ctypes
    lib = ctypes.CDLL(nek.LIB_PATH)
    for name in decl:
        assert hasattr(lib, name), name
    assert set(nek.EXPORTED) <= decl
    assert nek.version() == 1


def test_no_oracle_in_product():
    """The product path never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2409_19119_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "liboracle" not in src, f


@pytest.mark.parametrize("mk", [lambda: mg.config_mesh(1), lambda: mg.box_mesh(3, 2, 4, 5, deform="sin"),
                                lambda: mg.box_mesh(2, 2, 2, 1, dirichlet="none")])
def test_plan_maps_equal_oracle(nek, mk):
    m = mk()
    P = nek.Plan(m.E, m.N, m.gid, m.mask, m.xyz)
    g = oracle.GsMap(m.gid)
    assert np.array_equal(P.get(nek.PLAN_PERM), g.perm)
    assert np.array_equal(P.get(nek.PLAN_OFFS), g.offs)
    assert np.array_equal(P.get(nek.PLAN_OWNER), oracle.owner_flags(m.gid))
    assert P.get(nek.PLAN_IFC_PERM).size == 0 and P.get(nek.PLAN_NEIGHBORS).size == 0


def test_plan_relabelled_gids_first_touch(nek):
    """Canonical order does not depend on how the caller numbered the ids (reading 7)."""
    m = mg.box_mesh(3, 3, 3, 3)
    rng = np.random.default_rng(0)
    u, inv = np.unique(m.gid, return_inverse=True)
    relab = rng.permutation(u.size)[inv].astype(np.int64) * 7 + 3
    P1 = nek.Plan(m.E, m.N, m.gid)
    P2 = nek.Plan(m.E, m.N, relab)
    assert np.array_equal(P1.get(nek.PLAN_PERM), P2.get(nek.PLAN_PERM))
    assert np.array_equal(P1.get(nek.PLAN_OFFS), P2.get(nek.PLAN_OFFS))
    assert np.array_equal(P2.get(nek.PLAN_PERM), oracle.GsMap(relab).perm)


def test_plan_errors(nek):
    m = mg.box_mesh(2, 1, 1, 2, deform="affine", dirichlet="none")
    with pytest.raises(nek.NekError) as e:
        nek.Plan(m.E, 16, np.zeros(17 ** 3 * 2, np.int64))
    assert e.value.code == nek.EORDER
    g = m.gid.copy(); g[5] = -1
    with pytest.raises(nek.NekError) as e:
        nek.Plan(m.E, m.N, g)
    assert e.value.code == nek.EINVAL
    mask = m.mask.copy(); mask[2] = 1
    with pytest.raises(nek.NekError) as e:
        nek.Plan(m.E, m.N, m.gid, mask)
    assert e.value.code == nek.ETOPO
    xyz = m.xyz.copy(); xyz[2, 2] += 1e-3
    with pytest.raises(nek.NekError) as e:
        nek.Plan(m.E, m.N, m.gid, None, xyz)
    assert e.value.code == nek.ETOPO


def emulate_halo_gs(nek, plans, vals):
    """Run the multi-rank gather-scatter using ONLY the plans' arrays and plain
    sums in the order the plan prescribes (what the kernels do), for checking
    the plan on CPU.  Returns per-rank results."""
    P = len(plans)
    partial, send = [], []
    for r in range(P):
        p = plans[r]
        ip, io = p.get(nek.PLAN_IFC_PERM), p.get(nek.PLAN_IFC_OFFS)
        part = np.array([sum_left(vals[r][ip[io[x]:io[x + 1]]]) for x in range(io.size - 1)])
        partial.append(part)
        send.append(part[p.get(nek.PLAN_SEND_RUN)] if part.size else np.zeros(0))
    outs = []
    for r in range(P):
        p = plans[r]
        v = vals[r].copy()
        pm, po = p.get(nek.PLAN_PERM), p.get(nek.PLAN_OFFS)
        for x in range(po.size - 1):
            v[pm[po[x]:po[x + 1]]] = sum_left(vals[r][pm[po[x]:po[x + 1]]])
        nb, so = p.get(nek.PLAN_NEIGHBORS), p.get(nek.PLAN_SEND_OFFS)
        recv = np.zeros(so[-1] if so.size else 0)
        for k, q in enumerate(nb):
            pq = plans[q]
            nbq, soq = pq.get(nek.PLAN_NEIGHBORS), pq.get(nek.PLAN_SEND_OFFS)
            kq = list(nbq).index(r)
            recv[so[k]:so[k + 1]] = send[q][soq[kq]:soq[kq + 1]]
        ip, io = p.get(nek.PLAN_IFC_PERM), p.get(nek.PLAN_IFC_OFFS)
        co, cb = p.get(nek.PLAN_CONTRIB_OFFS), p.get(nek.PLAN_CONTRIB)
        for x in range(io.size - 1):
            terms = [partial[r][x] if s < 0 else recv[s] for s in cb[co[x]:co[x + 1]]]
            v[ip[io[x]:io[x + 1]]] = sum_left(np.array(terms))
        outs.append(v)
    return outs


def sum_left(a):
    s = a[0]
    for t in a[1:]:
        s = s + t
    return s


@pytest.mark.parametrize("split", ["slab2", "slab4", "block222"])
def test_multirank_plans_reproduce_oracle(nek, split):
    m = mg.box_mesh(4, 4, 4, 2, deform="bubble", dirichlet="zends")
    parts = {"slab2": lambda: mg.slab_partition(m, 2), "slab4": lambda: mg.slab_partition(m, 4),
             "block222": lambda: mg.block_partition(m, 2, 2, 2)}[split]()
    subs = [mg.submesh(m, e) for e in parts]
    plans = [nek.Plan(s.E, s.N, s.gid, s.mask, s.xyz) for s in subs]
    lists = [p.surface_gids() for p in plans]
    for r, p in enumerate(plans):
        p.set_ranks(r, len(plans), lists)
    # neighbour symmetry and slot agreement (ascending gid on both sides)
    for r, p in enumerate(plans):
        nb, so, sr = p.get(nek.PLAN_NEIGHBORS), p.get(nek.PLAN_SEND_OFFS), p.get(nek.PLAN_SEND_RUN)
        gids = p.get(nek.PLAN_IFC_GID)
        for k, q in enumerate(nb):
            pq = plans[q]
            nbq = list(pq.get(nek.PLAN_NEIGHBORS))
            assert r in nbq
            kq = nbq.index(r)
            soq, srq, gq = pq.get(nek.PLAN_SEND_OFFS), pq.get(nek.PLAN_SEND_RUN), pq.get(nek.PLAN_IFC_GID)
            mine = gids[sr[so[k]:so[k + 1]]]
            theirs = gq[srq[soq[kq]:soq[kq + 1]]]
            assert np.array_equal(mine, theirs) and np.all(np.diff(mine) > 0)
    # owners: exactly one owner copy per gid over all ranks
    owners = np.concatenate([s.gid[p.get(nek.PLAN_OWNER) != 0] for s, p in zip(subs, plans)])
    assert owners.size == np.unique(m.gid).size and np.unique(owners).size == owners.size
    # boundary elements first
    for s, p in zip(subs, plans):
        assert sorted(p.get(nek.PLAN_ELEM_ORDER)) == list(range(s.E))
    # the emulated exchange equals the oracle's multi-rank gs bit for bit
    v = mg.random_evector(m, seed=3)
    P3 = m.Nq ** 3
    vals = [v[(e[:, None] * P3 + np.arange(P3)).reshape(-1)] for e in parts]
    got = emulate_halo_gs(nek, plans, vals)
    ref = oracle.gs_multi([s.gid for s in subs], vals)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_probe_argument_errors(nek):
    """The measurement probes validate their arguments before touching a device (include/nek.h)."""
    import ctypes
    d = ctypes.c_double(0.0)
    assert nek._lib.nek_probe_hbm_gbps(0, 1000, ctypes.byref(d), None, None) == nek.EINVAL
    assert nek._lib.nek_probe_smem_tbps(0, None) == nek.EINVAL
    assert nek._lib.nek_probe_dfma_tflops(0, None) == nek.EINVAL
