"""Pins for the oracle's geometry, operator, gather-scatter and Jacobi diagonal.

Independent references: closed-form affine metrics, domain volumes, the
brute-force assembled matrix (oracle/assemble.py: Vandermonde derivatives,
analytic Jacobians, dense assembly), dense O(N^6) contractions, the Kronecker
form of the affine stiffness, invariants (symmetry, A.1 = 0, patch test) and
hand-countable gather-scatter facts.
"""
import os

import numpy as np
import pytest

import oracle
from oracle.assemble import assemble_box
from workloads import meshgen as mg


def test_geom_unit_cube_closed_form():
    """Unit-cube element: dx/dr = 1/2, J = 1/8, grad r = 2 -> G_rr = w_q/2."""
    for N in (1, 3, 5):
        m = mg.box_mesh(1, 1, 1, N, deform="affine")
        G, wJ = oracle.geom(1, N, m.xyz)
        x, w = oracle.gll(N)
        W = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
        np.testing.assert_allclose(wJ, W / 8, rtol=1e-14)
        for a, v in zip(range(6), (W / 2, 0, 0, W / 2, 0, W / 2)):
            np.testing.assert_allclose(G[0, a], v * np.ones_like(W), rtol=1e-14, atol=1e-15)
        assert abs(wJ.sum() - 1.0) < 1e-14


def test_geom_stretched_ratio():
    """2x1x1 element: metric diagonal ratio 1:4:4, cross terms 0."""
    m = mg.box_mesh(1, 1, 1, 4, deform="affine", extent=(2.0, 1.0, 1.0))
    G, wJ = oracle.geom(1, 4, m.xyz)
    np.testing.assert_allclose(G[0, 3] / G[0, 0], 4.0, rtol=1e-14)
    np.testing.assert_allclose(G[0, 5] / G[0, 0], 4.0, rtol=1e-14)
    assert np.abs(G[0, [1, 2, 4]]).max() < 1e-15
    assert abs(wJ.sum() - 2.0) < 1e-14


@pytest.mark.parametrize("N", [2, 3, 5, 7])
def test_geom_volume(N):
    """sum wJ = domain volume: bubble map keeps the unit volume (divergence of a
    field vanishing on the boundary); uniform scaling by 2 multiplies it by 8."""
    m = mg.box_mesh(2, 2, 2, N, deform="bubble", eps=0.05)
    _, wJ = oracle.geom(m.E, N, m.xyz)
    assert abs(wJ.sum() - 1.0) < 1e-13
    _, wJ2 = oracle.geom(m.E, N, 2.0 * m.xyz)
    assert abs(wJ2.sum() - 8.0) < 1e-12


def test_geom_rejects_inverted_element():
    m = mg.box_mesh(1, 1, 1, 2, deform="affine")
    xyz = m.xyz.copy()
    xyz[0] = -xyz[0]                          # mirror -> J < 0
    with pytest.raises(ValueError, match="element 0"):
        oracle.geom(1, 2, xyz)


def _dense_ax(N, G, wJ, h1, h2, u, D):
    """Dense O(N^6) contraction with Kronecker factors, one element."""
    Nq = N + 1
    I = np.eye(Nq)
    B = [np.kron(I, np.kron(I, D)), np.kron(I, np.kron(D, I)), np.kron(D, np.kron(I, I))]
    idx = [[0, 1, 2], [1, 3, 4], [2, 4, 5]]
    w = np.zeros(Nq ** 3)
    for a in range(3):
        for b in range(3):
            w += B[a].T @ (G[idx[a][b]] * (B[b] @ u))
    return h1 * w + h2 * wJ * u


@pytest.mark.parametrize("N", [1, 2, 3, 5])
def test_sum_factorization_equals_dense(N):
    """tensor apply == dense contraction (random symmetric G)."""
    rng = np.random.default_rng(N)
    P3 = (N + 1) ** 3
    G = rng.standard_normal((1, 6, P3)); wJ = rng.uniform(0.5, 1, P3); u = rng.standard_normal(P3)
    D = oracle.deriv(N)
    w = oracle.ax_local(1, N, G, wJ, 0.7, 0.2, u, D=D)
    ref = _dense_ax(N, G[0], wJ, 0.7, 0.2, u, D)
    assert np.abs(w - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("N,deform", [(2, "bubble"), (3, "bubble"), (4, "bubble"), (3, "affine"),
                                      (1, "affine"), (3, "shear")])
@pytest.mark.parametrize("h", [(1.0, 0.0), (1.0, 0.3), (0.0, 1.0)])
def test_operator_equals_brute_force_assembly(N, deform, h):
    """Matrix-free M QQ^T A_L M u == Q A u_g with A assembled by an independent route."""
    h1, h2 = h
    eps = 0.05 if deform != "shear" else 0.02
    m = mg.box_mesh(2, 2, 2, N, deform=deform, eps=eps, dirichlet="none")
    O = oracle.Oracle.from_mesh(m)
    x, w = oracle.gll(N)
    A, l2g = assemble_box(m.shape, N, h1, h2, x, w, deform=deform, eps=eps)
    assert np.array_equal(l2g, m.gid)
    ug = np.random.default_rng(7).standard_normal(A.shape[0])
    ref = (A @ ug)[m.gid]
    got = O.apply(h1, h2, ug[m.gid])
    tol = 1e-13 if deform != "shear" else None
    if tol is None:   # shear map is not polynomial: isoparametric geometry is inexact
        assert np.abs(got - ref).max() <= 0.05 * np.abs(ref).max()
    else:
        assert np.abs(got - ref).max() <= tol * np.abs(ref).max()
    # diagonal of the assembled matrix (reading 10)
    if deform != "shear":
        d = O.diag(h1, h2)
        np.testing.assert_allclose(d, np.diag(A)[m.gid], rtol=1e-13, atol=1e-15)


def test_operator_symmetric_and_annihilates_constants():
    m = mg.box_mesh(2, 2, 2, 3, deform="bubble", eps=0.05, dirichlet="none")
    O = oracle.Oracle.from_mesh(m)
    rng = np.random.default_rng(3)
    x = mg.smooth_field(m, seed=1, masked=False); y = mg.smooth_field(m, seed=2, masked=False)
    Ax, Ay = O.apply(1.0, 0.0, x), O.apply(1.0, 0.0, y)
    assert abs(O.dot(y, Ax) - O.dot(x, Ay)) <= 1e-13 * abs(O.dot(x, Ax))
    one = np.ones(m.n_local)
    assert np.abs(O.apply(1.0, 0.0, one)).max() <= 1e-14 * np.abs(Ax).max()
    # SPD on the masked subspace
    m2 = mg.config_mesh(1)
    O2 = oracle.Oracle.from_mesh(m2)
    for s in range(3):
        v = mg.smooth_field(m2, seed=10 + s)
        assert O2.dot(v, O2.apply(1.0, 0.0, v)) > 0


@pytest.mark.parametrize("N", [2, 3])
def test_affine_kronecker_form(N):
    """Affine hx x hy x hz element: K_e = (hy hz/2hx) W(x)W(x)K + (hx hz/2hy) W(x)K(x)W
    + (hx hy/2hz) K(x)W(x)W in (k,j,i) ordering, K = D^T W D."""
    hx, hy, hz = 0.7, 1.3, 0.4
    m = mg.box_mesh(1, 1, 1, N, deform="affine", extent=(hx, hy, hz))
    G, wJ = oracle.geom(1, N, m.xyz)
    x, w = oracle.gll(N)
    D = oracle.deriv(N, x)
    W = np.diag(w); K = D.T @ W @ D
    ref = (hy * hz / (2 * hx)) * np.kron(W, np.kron(W, K)) + (hx * hz / (2 * hy)) * np.kron(W, np.kron(K, W)) \
        + (hx * hy / (2 * hz)) * np.kron(K, np.kron(W, W))
    P3 = (N + 1) ** 3
    cols = np.stack([oracle.ax_local(1, N, G, wJ, 1.0, 0.0, e) for e in np.eye(P3)], 1)
    assert np.abs(cols - ref).max() <= 1e-14 * np.abs(ref).max() * P3


@pytest.mark.parametrize("N", [2, 3, 5])
@pytest.mark.parametrize("kind", ["jitter", "bubble"])
def test_patch_test_linear(N, kind):
    """QQ^T K_L (a.x + c) = 0 at rows not on the domain boundary (exercises the
    cross-term factors G_rs, G_rt, G_st)."""
    if kind == "jitter":
        m = mg.box_mesh(3, 3, 3, N, deform="affine", jitter=0.2, seed=5, dirichlet="all")
    else:
        m = mg.box_mesh(3, 3, 3, N, deform="bubble", eps=0.05, dirichlet="all")
    O = oracle.Oracle(m.E, m.N, m.xyz, m.gid, None)
    u = 0.3 * m.xyz[0] - 1.1 * m.xyz[1] + 0.7 * m.xyz[2] + 2.0
    w = O.gs_apply(O.ax_local(1.0, 0.0, u))
    interior = m.mask == 0
    scale = np.abs(O.ax_local(1.0, 0.0, mg.smooth_field(m, 3, masked=False))).max()
    assert np.abs(w[interior]).max() <= 1e-13 * scale


def test_patch_test_fails_at_N1():
    """At N=1 the discrete metric identities fail on perturbed trilinear meshes
    (2.3e-3) -- guards against a vacuous patch test."""
    m = mg.box_mesh(3, 3, 3, 1, deform="affine", jitter=0.2, seed=5, dirichlet="all")
    O = oracle.Oracle(m.E, m.N, m.xyz, m.gid, None)
    u = 0.3 * m.xyz[0] - 1.1 * m.xyz[1] + 0.7 * m.xyz[2]
    w = O.gs_apply(O.ax_local(1.0, 0.0, u))
    assert np.abs(w[m.mask == 0]).max() > 1e-6


# ----------------------------------------------------------- gather-scatter --
def _golden_rows(golden_dir, name):
    out = []
    for line in open(os.path.join(golden_dir, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append([c.strip() for c in line.split("|")])
    return out


def test_box_dof_counts(golden_dir):
    for dims, nu, n2 in _golden_rows(golden_dir, "box_dof_counts.txt"):
        Ex, Ey, Ez, N = map(int, dims.split())
        m = mg.box_mesh(Ex, Ey, Ez, N, deform="affine", dirichlet="none")
        assert m.n_unique() == int(nu)
        O = oracle.Oracle.from_mesh(m)
        mult = O.gs_apply(np.ones(m.n_local))             # field = 1 -> multiplicity
        np.testing.assert_array_equal(mult, oracle.multiplicity(m.gid))
        if int(n2) >= 0:
            _, first = np.unique(m.gid, return_index=True)
            assert int((mult[first] == 2).sum()) == int(n2)


def test_gs_map_canonical_structure():
    m = mg.box_mesh(3, 2, 2, 3, deform="bubble", dirichlet="none")
    g = oracle.GsMap(m.gid)
    firsts = g.perm[g.offs[:-1]]
    assert np.all(np.diff(firsts) > 0)                           # runs ordered by first touch
    for r in range(g.nruns):
        c = g.perm[g.offs[r]:g.offs[r + 1]]
        assert c.size >= 2 and np.all(np.diff(c) > 0)            # ascending within a run
        assert np.all(m.gid[c] == g.rgid[r])
    mult = oracle.multiplicity(m.gid)
    assert np.array_equal(np.sort(g.perm), np.nonzero(mult >= 2)[0])   # every shared copy once
    # cfg1 counts: 127 shared runs, 296 copies
    g1 = oracle.GsMap(mg.config_mesh(1).gid)
    assert g1.nruns == 127 and g1.perm.size == 296


def test_gs_algebra():
    m = mg.box_mesh(3, 2, 2, 3, deform="bubble", dirichlet="none")
    O = oracle.Oracle.from_mesh(m)
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(m.n_local), rng.standard_normal(m.n_local)
    mult = oracle.multiplicity(m.gid).astype(float)
    gu, gv = O.gs_apply(u), O.gs_apply(v)
    assert abs(np.dot(gu, v) - np.dot(u, gv)) <= 1e-12 * np.abs(gu).sum()        # symmetric
    np.testing.assert_allclose(O.gs_apply(gu), gu * mult, rtol=1e-14)             # gs^2 = gs*mult
    f = m.gid.astype(float)
    np.testing.assert_array_equal(O.gs_apply(f) / mult, f)                        # idempotence
    # copies of an id hold identical bits
    _, inv = np.unique(m.gid, return_inverse=True)
    first = np.zeros(inv.max() + 1); first[inv] = gu
    assert np.array_equal(first[inv], gu)


@pytest.mark.parametrize("parts", ["slab2", "slab3", "block222"])
def test_gs_multi_rank_equals_single(parts):
    m = mg.box_mesh(4, 4, 4, 3, deform="bubble", dirichlet="none")
    if parts == "slab2":
        P = mg.slab_partition(m, 2)
    elif parts == "slab3":
        P = mg.slab_partition(m, 3)
    else:
        P = mg.block_partition(m, 2, 2, 2)
    v = np.random.default_rng(2).standard_normal(m.n_local)
    ref = oracle.Oracle.from_mesh(m).gs_apply(v)
    subs = [mg.submesh(m, e) for e in P]
    vr = [v[(e[:, None] * 64 + np.arange(64)).reshape(-1)] for e in P]
    out = oracle.gs_multi([s.gid for s in subs], vr)
    full = np.zeros(m.n_local)
    for e, o in zip(P, out):
        full[(e[:, None] * 64 + np.arange(64)).reshape(-1)] = o
    assert np.abs(full - ref).max() <= 1e-15 * np.abs(ref).max() * 4
    # all copies of an id bit-identical across ranks
    _, inv = np.unique(m.gid, return_inverse=True)
    first = np.zeros(inv.max() + 1); first[inv] = full
    assert np.array_equal(first[inv], full)
    # integer-valued data: exact
    iv = np.floor(10 * v)
    outi = oracle.gs_multi([s.gid for s in subs], [iv[(e[:, None] * 64 + np.arange(64)).reshape(-1)] for e in P])
    fulli = np.zeros(m.n_local)
    for e, o in zip(P, outi):
        fulli[(e[:, None] * 64 + np.arange(64)).reshape(-1)] = o
    assert np.array_equal(fulli, oracle.Oracle.from_mesh(m).gs_apply(iv))


def test_rod_bundle_mesh_and_operator():
    """Config-4-like curved rod-bundle mesh (reading 13): conforming (copies share coordinates),
    positive Jacobians, volume = cell squares minus pins up to the isoparametric circle error,
    multiplicities up to 16, A.1 = 0 and symmetry on curved elements."""
    m = mg.rod_bundle(2, 2, 2, 4)
    O = oracle.Oracle.from_mesh(m)
    mult = np.bincount(oracle.multiplicity(m.gid))
    assert mult.size == 17 and mult[16] > 0
    exact = 4 * 1.26 ** 2 * 2 * 1.26 - 4 * np.pi * 0.475 ** 2 * 2 * 1.26
    assert abs(O.wJ.sum() - exact) < 1e-5 * exact and O.wJ.min() > 0
    one = np.ones(m.n_local)
    scale = np.abs(O.ax_local(1.0, 0.0, mg.smooth_field(m, 3, masked=False))).max()
    assert np.abs(O.gs_apply(O.ax_local(1.0, 0.0, one))).max() <= 1e-13 * scale
    x, y = mg.smooth_field(m, 1), mg.smooth_field(m, 2)
    assert abs(O.dot(y, O.apply(1.0, 2.0, x)) - O.dot(x, O.apply(1.0, 2.0, y))) <= 1e-12 * abs(O.dot(x, O.apply(1.0, 2.0, x)))
    # slabs of layers generate the same ids as the whole column
    top = mg.rod_bundle(2, 2, 1, 4, z0_layer=1, nlayers_total=2)
    assert np.isin(top.gid, m.gid).all()
