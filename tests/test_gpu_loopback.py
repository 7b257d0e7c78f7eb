"""Multi-rank parity on ONE GPU through the loopback group (SURVEY 4 "loopback comm backend",
SURVEY 8(a) a6; P:198-200 unit-depth exchange, P:391-398 overlap with interior work
rank-ordered reductions).

P virtual ranks, one host thread and one context each, run the same halo pack / unpack, mailbox
and split-wave kernels as one-process-per-GPU ranks (transport 0 = the NVLink peer-memory path;
1 = the NCCL-path pack/unpack kernels around staged copies).  Checked against the oracle:
  * gs: every rank's result bit-equal to the oracle's multi-rank emulation (reading 7), and the
    copies of a node bit-identical across ranks;
  * Ax (+ gs + halo): relative 1e-12 normwise against the single-rank oracle;
  * PCG over a fixed window: |d ||r_k||| <= 1e-12 max(||b||, ||r_k||) at every k against the
    single-rank oracle (reading 17: the rank-ordered partial sums only re-associate the inner
    products), every rank holding the same history bits; x within 1e-12 normwise;
  * both Ax orderings (boundary / interior on concurrent streams with the split wave, and in
    stream order), slab partitions P = 2, 3 and a 2x2x2 block partition (edges and corners).
"""
import os
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from workloads import meshgen as mg  # noqa: E402

WINDOW_TOL = oracle.WINDOW_TOL


@pytest.fixture(scope="module")
def nek():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_19119_b200 import nek as _nek
    return _nek


def rel(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b)).max()
    s = np.abs(np.asarray(b)).max()
    return d / (s if s > 0 else 1.0)


def run_ranks(nek, P, transport, fn, env=None):
    """fn(rank, comm) on P threads sharing one loopback group; returns the per-rank results."""
    lb = nek.Loopback(P, transport)
    out, errs = [None] * P, []
    saved = {}
    for k, v in (env or {}).items():
        saved[k] = os.environ.get(k)
        os.environ[k] = v

    def work(r):
        try:
            out[r] = fn(r, lb.comm(r))
        except BaseException as e:  # noqa: BLE001
            errs.append(f"rank {r}: {e!r}")
            lb.abort()
    try:
        th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        lb.free()
    assert not errs, errs
    return out


def parts_of(m, kind, P):
    if kind == "slab":
        return mg.slab_partition(m, P)
    px, py, pz = {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[P]
    return mg.block_partition(m, px, py, pz)


def local_index(m, elems):
    P3 = m.Nq ** 3
    return (np.asarray(elems)[:, None] * P3 + np.arange(P3)).reshape(-1)


def check_multirank(nek, m, parts, transport, env, window=40, h=(1.0, 0.0), pcg_device=False):
    P = len(parts)
    subs = [mg.submesh(m, p) for p in parts]
    locs = [local_index(m, p) for p in parts]
    u = mg.random_evector(m, seed=5)
    b = mg.smooth_field(m, seed=3)

    def fn(r, comm):
        s = subs[r]
        ctx = nek.setup(s.E, s.N, s.xyz, s.gid, s.mask, comm=comm, device=0)
        try:
            info = nek.get_info(ctx)
            w = np.empty(s.n_local)
            nek.ax(ctx, 1.0, 0.3, u[locs[r]], w)
            v = u[locs[r]].copy()
            nek.gs(ctx, v)
            if pcg_device:   # device pointers on torch's stream of this thread
                bd = torch.from_numpy(b[locs[r]]).cuda()
                xd = torch.zeros_like(bd)
                st, it, rr, hist = nek.pcg_solve(ctx, h[0], h[1], bd, xd, 0.0, window, want_hist=True)
                x = xd.cpu().numpy()
            else:
                x = np.zeros(s.n_local)
                st, it, rr, hist = nek.pcg_solve(ctx, h[0], h[1], b[locs[r]], x, 0.0, window, want_hist=True)
            return {"w": w, "v": v, "x": x, "hist": hist, "it": it, "st": st, "info": info}
        finally:
            nek.free(ctx)

    res = run_ranks(nek, P, transport, fn, env)
    O = oracle.Oracle.from_mesh(m)
    info0 = res[0]["info"]
    want_transport = 2 if transport == 0 else 1
    assert all(r_["info"]["transport"] == want_transport for r_ in res), [r_["info"]["transport"] for r_ in res]
    assert sum(r_["info"]["n_neighbors"] > 0 for r_ in res) == P
    # gs: bit-equal to the multi-rank emulation, and to the single-rank oracle to 1e-15 (reading 7)
    ref_multi = oracle.gs_multi([s_.gid for s_ in subs], [u[l_] for l_ in locs])
    for r_, rm in zip(res, ref_multi):
        assert np.array_equal(r_["v"], rm)
    vg, wg, xg = np.zeros(m.n_local), np.zeros(m.n_local), np.zeros(m.n_local)
    for r_, l_ in zip(res, locs):
        vg[l_] = r_["v"]; wg[l_] = r_["w"]; xg[l_] = r_["x"]
    assert rel(vg, O.gs_apply(u)) <= 1e-15
    # Ax + gs + halo
    assert rel(wg, O.apply(1.0, 0.3, u)) <= 1e-12
    # copies of every node bit-identical across ranks
    allg = np.concatenate([s_.gid for s_ in subs])
    allw = np.concatenate([r_["w"] for r_ in res])
    order = np.argsort(allg, kind="stable")
    sg, sw = allg[order], allw[order]
    assert np.all((sg[1:] != sg[:-1]) | (sw[1:] == sw[:-1]))
    # PCG window: WINDOW_TOL relative to max(||b||, ||r_k||) (reading 17), same bits on every rank
    xo, ito, _, ho = O.pcg(h[0], h[1], b, 0.0, window)
    h0 = res[0]["hist"]
    assert all(r_["it"] == window and r_["st"] == nek.MAXIT for r_ in res)
    assert all(np.array_equal(r_["hist"], h0) for r_ in res)
    dmax = oracle.window_error(h0, ho)
    print(f"P={P} transport={transport} env={env} N={m.N}: max |d h|/max(1,h) = {dmax:.2e}, "
          f"x err {rel(xg, xo):.2e}, halo doubles {[r_['info']['halo_doubles'] for r_ in res]}")
    assert dmax <= WINDOW_TOL
    assert rel(xg, xo) <= 1e-12
    return info0


MODES = {"concurrent": {"NEK_CONCURRENT_BND": "1"}, "stream_order": {"NEK_CONCURRENT_BND": "0"},
         "concurrent_nosplit": {"NEK_CONCURRENT_BND": "1", "NEK_BND_SPLIT": "0"}}


@pytest.mark.parametrize("N", [3, 5, 7])
@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("P", [2, 3])
def test_loopback_slab_p2p(nek, N, mode, P):
    m = mg.box_mesh(3, 4, 2 * P, N, deform="bubble", eps=0.05, dirichlet="all")
    check_multirank(nek, m, parts_of(m, "slab", P), 0, MODES[mode])


@pytest.mark.parametrize("N", [3, 5, 7])
@pytest.mark.parametrize("mode", ["concurrent", "stream_order"])
def test_loopback_block_2x2x2_p2p(nek, N, mode):
    """8 ranks, 2x2x2 blocks: every rank shares faces, edges and a corner (up to 7 neighbours)."""
    m = mg.box_mesh(4, 4, 4, N, deform="sin", eps=0.05, dirichlet="zends")
    check_multirank(nek, m, parts_of(m, "block", 8), 0, MODES[mode])


@pytest.mark.parametrize("N", [3, 7])
@pytest.mark.parametrize("kind,P", [("slab", 2), ("slab", 3), ("block", 8)])
def test_loopback_staged_transport(nek, N, kind, P):
    """The NCCL-path kernels (interface partial + pack, unpack after the exchange) on the staged
    loopback transport."""
    m = mg.box_mesh(4, 4, 4 if kind == "block" else 2 * P, N, deform="bubble", dirichlet="all")
    check_multirank(nek, m, parts_of(m, kind, P), 1, MODES["stream_order"])


def test_loopback_helmholtz_device_pointers(nek):
    """Helmholtz (h2 != 0) PCG with device-pointer b and x (torch, each thread's current stream)."""
    m = mg.box_mesh(4, 3, 4, 7, deform="bubble", dirichlet="all")
    check_multirank(nek, m, parts_of(m, "slab", 2), 0, MODES["concurrent"], window=30, h=(1.0, 5.0),
                    pcg_device=True)


def test_loopback_config2_slab_pair(nek):
    """Config 2 (16^3 elements, N = 7) split into two z-slabs: the launch configuration of the
    per-GPU bench at its full element count, 100-iteration PCG window."""
    m = mg.config_mesh(2)
    check_multirank(nek, m, parts_of(m, "slab", 2), 0, MODES["concurrent"], window=100)


def test_loopback_pmg_and_projection(nek):
    """p-multigrid V-cycle + converged pMG-PCG (each level exchanges its own halo) and a projection
    sequence across two virtual ranks, against the single-rank oracle hierarchy."""
    from oracle import pmg as opmg
    from oracle.projection import Projection as OProj
    m = mg.box_mesh(4, 3, 4, 7, deform="bubble", dirichlet="all")
    parts = parts_of(m, "slab", 2)
    subs = [mg.submesh(m, p) for p in parts]
    locs = [local_index(m, p) for p in parts]
    O = oracle.Oracle.from_mesh(m)
    u = mg.random_evector(m, seed=5)
    rf = oracle.mask(m.mask, O.gs_apply(u))
    b = mg.smooth_field(m, seed=3)
    b0, b1 = mg.smooth_field(m, seed=11), mg.smooth_field(m, seed=12)
    seq = [b0 + 0.02 * t * b1 for t in range(5)]

    def fn(r, comm):
        s = subs[r]
        ctx = nek.setup(s.E, s.N, s.xyz, s.gid, s.mask, comm=comm, device=0)
        try:
            Pm = nek.PMG(ctx, s.xyz, 1.0, 0.0)
            z = np.empty(s.n_local)
            Pm.apply(rf[locs[r]].copy(), z)
            x = np.zeros(s.n_local)
            st, it, _, _ = Pm.solve(b[locs[r]], x, 1e-10, 200)
            Pm.free()
            pr = nek.Projection(ctx, 4)
            its, xs = [], []
            for bb in seq:
                xp = np.zeros(s.n_local)
                pst, pit, _ = pr.solve(1.0, 0.0, bb[locs[r]], xp, 1e-9, 1000)
                its.append(pit); xs.append(xp)
            pr.free()
            return {"z": z, "x": x, "it": it, "st": st, "pits": its, "xs": xs}
        finally:
            nek.free(ctx)

    res = run_ranks(nek, 2, 0, fn, MODES["concurrent"])
    Po = opmg.PMG(O, m.xyz, 1.0, 0.0)
    zg, xg = np.zeros(m.n_local), np.zeros(m.n_local)
    for r_, l_ in zip(res, locs):
        zg[l_] = r_["z"]; xg[l_] = r_["x"]
    assert rel(zg, Po.apply(rf)) <= 1e-11
    xpo, pito, psto, _ = opmg.pcg(O, 1.0, 0.0, b, 1e-10, 200, Po.apply)
    assert all(r_["st"] == nek.OK and abs(r_["it"] - pito) <= 1 for r_ in res)
    assert rel(xg, xpo) <= 1e-9
    OP = OProj(O, 4)
    for t, bb in enumerate(seq):
        xo, ito, _ = OP.solve(1.0, 0.0, bb, 1e-9, 1000)
        xgt = np.zeros(m.n_local)
        for r_, l_ in zip(res, locs):
            xgt[l_] = r_["xs"][t]
        assert all(abs(r_["pits"][t] - ito) <= 1 for r_ in res), (t, [r_["pits"][t] for r_ in res], ito)
        assert rel(xgt, xo) <= 1e-8


def test_loopback_abort_is_an_error_not_a_hang(nek):
    """A rank that stops (its thread raises before a collective) aborts the group: the other rank's
    collective returns NEK_ENCCL instead of waiting forever."""
    m = mg.box_mesh(2, 2, 4, 3, deform="bubble")
    parts = parts_of(m, "slab", 2)
    subs = [mg.submesh(m, p) for p in parts]
    lb = nek.Loopback(2, 0)
    got = {}

    def rank0():
        s = subs[0]
        try:
            nek.setup(s.E, s.N, s.xyz, s.gid, s.mask, comm=lb.comm(0), device=0)
        except nek.NekError as e:
            got["code"] = e.code

    t = threading.Thread(target=rank0)
    t.start()
    lb.abort()          # rank 1 never joins
    t.join(timeout=120)
    assert not t.is_alive()
    lb.free()
    assert got.get("code") == nek.ENCCL


@pytest.mark.parametrize("mode", ["concurrent", "stream_order", "concurrent_nosplit"])
def test_loopback_deferred_bookkeeping_bitwise(nek, mode):
    """P2P deferred bookkeeping (N = 7: the next Ax pulls every rank's (rho', rr) from the mailbox, no
    separate bookkeeping kernel) against NEK_DEFER=0: the pulled sums are the same values in the same
    rank order, so statuses, iteration counts, histories and x are bit-identical -- for windows ending
    on an update (the finish kernel books it), mid-graph, and for a converged solve."""
    m = mg.box_mesh(4, 3, 6, 7, deform="bubble", dirichlet="all")
    parts = parts_of(m, "slab", 3)
    subs = [mg.submesh(m, p) for p in parts]
    locs = [local_index(m, p) for p in parts]
    b = mg.smooth_field(m, seed=8)

    def fn(r, comm):
        s = subs[r]
        ctx = nek.setup(s.E, s.N, s.xyz, s.gid, s.mask, comm=comm, device=0)
        try:
            out = []
            for tol, maxit in ((0.0, 20), (0.0, 7), (1e-9, 400), (0.0, 0)):
                x = np.zeros(s.n_local)
                st, it, rr, hist = nek.pcg_solve(ctx, 1.0, 0.0, b[locs[r]], x, tol, maxit, want_hist=True)
                out.append((st, it, rr, hist, x))
            return out
        finally:
            nek.free(ctx)

    res = {d: run_ranks(nek, 3, 0, fn, dict(MODES[mode], NEK_DEFER=d)) for d in ("0", "1")}
    for r in range(3):
        for (s0, i0, r0, h0, x0), (s1, i1, r1, h1, x1) in zip(res["0"][r], res["1"][r]):
            assert (s1, i1) == (s0, i0) and r1 == r0
            assert np.array_equal(h1, h0) and np.array_equal(x1, x0)
    conv = res["1"][0][2]
    assert conv[0] == nek.OK and 0 < conv[1] < 400
