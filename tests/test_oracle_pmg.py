"""Pins for the oracle's p-multigrid preconditioner (NEXT #1).

Each pin ties a step to something other than the oracle itself:
  * interpolation: exact on polynomials of the coarse degree, exact endpoint rows (GLL end nodes);
  * coarse node ids: the equivalence classes equal those of the coarse node COORDINATES (an
    independent geometric route), also after a random relabelling of the fine ids; the coarse
    mask equals "node on the Dirichlet boundary";
  * coarse operator: equals the operator of a mesh generated directly at the coarse order
    (bubble map, degree 2, reproduced exactly by the interpolated coordinates for N_c >= 2);
  * Chebyshev: the closed-form error polynomial T_k((theta - lam)/delta) / T_k(theta/delta) on a
    diagonal operator; degree 1 is damped Jacobi with weight 2/(lo + hi);
  * Lanczos: Ritz values interlace the dense spectrum of Dinv A and reach its ends;
  * V-cycle: symmetric and positive definite (explicit matrix on a tiny mesh), R = P^T in the
    owner inner product, linear;
  * pMG-PCG: the dense solution, fewer iterations than Jacobi-PCG, near E-independence."""
import numpy as np
import pytest

import oracle
from oracle import pmg
from oracle.assemble import assemble_box
from workloads import meshgen as mg


def test_schedule_defaults():
    assert pmg.default_schedule(7) == [7, 5, 3, 1]
    assert pmg.default_schedule(9) == [9, 5, 3, 1]
    assert pmg.default_schedule(5) == [5, 3, 1]
    assert pmg.default_schedule(3) == [3, 1]
    assert pmg.default_schedule(1) == [1]


@pytest.mark.parametrize("Nf,Nc", [(7, 5), (5, 3), (3, 1), (7, 1), (9, 4)])
def test_interpolation_exact_on_polynomials(Nf, Nc):
    xf, _ = oracle.gll(Nf)
    xc, _ = oracle.gll(Nc)
    J = pmg.lagrange_interp(xf, xc)
    for deg in range(Nc + 1):
        assert np.abs(J @ xc ** deg - xf ** deg).max() <= 1e-13
    assert J[0, 0] == 1.0 and np.all(J[0, 1:] == 0.0)
    assert J[-1, -1] == 1.0 and np.all(J[-1, :-1] == 0.0)
    assert np.abs(J.sum(axis=1) - 1.0).max() <= 1e-14


def _classes(keys):
    _, inv = np.unique(keys, axis=0, return_inverse=True)
    first = {}
    return np.array([first.setdefault(int(c), i) for i, c in enumerate(inv.ravel())])


@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("Nc", [5, 3, 1])
def test_coarse_ids_match_coordinates(Nc, relabel):
    m = mg.box_mesh(3, 2, 2, 7, deform="affine", jitter=0.12, seed=5, dirichlet="zends")
    gid = m.gid
    if relabel:
        u = np.unique(gid)
        perm = np.random.default_rng(1).permutation(u.size)
        gid = perm[np.searchsorted(u, gid)].astype(np.int64) * 7 + 3
    gc, mc = pmg.coarse_ids(m.E, 7, gid, m.mask, Nc)
    x7, _ = oracle.gll(7)
    xc, _ = oracle.gll(Nc)
    J = pmg.lagrange_interp(xc, x7)
    xyz = np.stack([pmg.interp_elements(J, m.xyz[d], 7, Nc) for d in range(3)])
    keys = np.round(xyz.T / 1e-9).astype(np.int64)
    assert np.array_equal(_classes(gc), _classes(keys))
    # Dirichlet on the z = 0 and z = extent planes (dirichlet="zends")
    z = xyz[2]
    want = (np.abs(z - z.min()) < 1e-12) | (np.abs(z - z.max()) < 1e-12)
    assert np.array_equal(mc.astype(bool), want)


@pytest.mark.parametrize("Nc", [5, 3, 2])
def test_coarse_operator_equals_direct_mesh(Nc):
    m7 = mg.box_mesh(2, 3, 2, 7, deform="bubble", dirichlet="all")
    O7 = oracle.Oracle.from_mesh(m7)
    P = pmg.PMG(O7, m7.xyz, 1.0, 0.3, schedule=[7, Nc, 1])
    Oc = P.levels[1].O
    md = mg.box_mesh(2, 3, 2, Nc, deform="bubble", dirichlet="all")
    Od = oracle.Oracle.from_mesh(md)
    assert np.abs(Oc.wJ - Od.wJ).max() <= 1e-13 * np.abs(Od.wJ).max()
    assert np.abs(Oc.G - Od.G).max() <= 1e-12 * np.abs(Od.G).max()
    x, y, z = md.xyz
    u = oracle.mask(md.mask, np.sin(2 * x + 0.3) * np.cos(y - z) + x * y)
    assert np.abs(Oc.apply(1.0, 0.3, u) - Od.apply(1.0, 0.3, u)).max() <= 1e-12 * np.abs(Od.apply(1.0, 0.3, u)).max()


@pytest.mark.parametrize("k", [1, 2, 3, 6, 9])
def test_chebyshev_closed_form_on_diagonal_operator(k):
    lam = np.linspace(0.05, 2.0, 40)
    lo, hi = 0.2, 2.2
    xs = np.cos(np.arange(40.0))
    f = lam * xs
    x = pmg.chebyshev(lambda v: lam * v, np.ones(40), f, None, k, lo, hi)
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    Tk = np.polynomial.chebyshev.Chebyshev.basis(k)
    want = Tk((theta - lam) / delta) / Tk(theta / delta) * xs
    assert np.abs((xs - x) - want).max() <= 1e-13
    if k == 1:
        assert np.abs(x - f * 2.0 / (lo + hi)).max() <= 1e-15


def test_chebyshev_fixed_point_and_initial_guess():
    lam = np.linspace(0.1, 1.0, 12)
    xs = np.sin(np.arange(12.0)) + 2.0
    f = lam * xs
    x = pmg.chebyshev(lambda v: lam * v, 1.0 / lam, f, xs, 6, 0.1, 1.1)
    assert np.abs(x - xs).max() <= 1e-13


@pytest.fixture(scope="module")
def tiny():
    m = mg.config_mesh(1)               # 2x2x2, N = 3, bubble, Dirichlet all faces
    O = oracle.Oracle.from_mesh(m)
    return m, O, pmg.PMG(O, m.xyz, 1.0, 0.0)


def _owner_basis(O):
    """Columns: continuous masked unit vectors of the unmasked unique ids."""
    o = np.nonzero((O.owner != 0) & (O.mask == 0))[0]
    B = np.zeros((O.n, o.size))
    for c, l in enumerate(o):
        B[O.gid == O.gid[l], c] = 1.0
    return B, o


def test_lanczos_ritz_values_interlace(tiny):
    m, O, P = tiny
    B, o = _owner_basis(O)
    A = np.stack([O.apply(1.0, 0.0, B[:, c])[o] for c in range(B.shape[1])], axis=1)
    d = np.diag(A)
    ev = np.sort(np.linalg.eigvals(A / d[:, None]).real)
    lo, hi = pmg.lanczos_bounds(P.levels[0], 20)
    assert ev[0] - 1e-12 <= lo <= hi <= ev[-1] + 1e-12
    assert hi >= 0.995 * ev[-1]
    lo, hi = pmg.lanczos_bounds(P.levels[0], B.shape[1] + 5)     # full Krylov space: exact ends
    assert abs(hi - ev[-1]) <= 1e-8 * ev[-1] and abs(lo - ev[0]) <= 1e-6 * ev[-1]


def test_vcycle_spd_linear_and_zero(tiny):
    m, O, P = tiny
    assert np.all(P.apply(np.zeros(O.n)) == 0.0)
    B, o = _owner_basis(O)
    Mm = np.stack([P.apply(B[:, c])[o] for c in range(B.shape[1])], axis=1)
    assert np.abs(Mm - Mm.T).max() <= 1e-12 * np.abs(Mm).max()
    assert np.linalg.eigvalsh(0.5 * (Mm + Mm.T)).min() > 0.0
    r1, r2 = B @ np.cos(np.arange(B.shape[1])), B @ np.sin(np.arange(B.shape[1]))
    assert np.abs(P.apply(2.0 * r1 - r2) - (2.0 * P.apply(r1) - P.apply(r2))).max() <= 1e-12 * np.abs(P.apply(r1)).max()


def test_restriction_is_prolongation_transpose():
    m = mg.box_mesh(3, 2, 2, 7, deform="sin", eps=0.05, dirichlet="top")
    O = oracle.Oracle.from_mesh(m)
    P = pmg.PMG(O, m.xyz, 1.0, 0.0)
    rng = np.random.default_rng(3)
    for l in range(len(P.levels) - 1):
        Of, Oc = P.levels[l].O, P.levels[l + 1].O
        r = oracle.mask(Of.mask, Of.gs_apply(rng.standard_normal(Of.n)) / oracle.multiplicity(Of.gid))
        e = oracle.mask(Oc.mask, Oc.gs_apply(rng.standard_normal(Oc.n)) / oracle.multiplicity(Oc.gid))
        lhs = Oc.dot(P.restrict(l, r), e)
        rhs = Of.dot(r, P.prolong(l, e))
        assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1e-300) * 10


def test_pmg_pcg_solves_the_system_with_fewer_iterations():
    m = mg.box_mesh(3, 3, 3, 5, deform="bubble", dirichlet="all")
    O = oracle.Oracle.from_mesh(m)
    P = pmg.PMG(O, m.xyz, 1.0, 0.0)
    b = mg.smooth_field(m, seed=4)
    x, it, st, h = pmg.pcg(O, 1.0, 0.0, b, 1e-10, 100, P.apply)
    xj, itj, stj, _ = O.pcg(1.0, 0.0, b, 1e-10, 2000)
    assert st == 0 and stj == 0 and it < itj / 5
    xg, wg = oracle.gll(m.N)
    A, _ = assemble_box(m.shape, m.N, 1.0, 0.0, xg, wg, deform=m.deform, eps=m.eps)
    keep = np.ones(A.shape[0], bool); keep[m.gid[m.mask != 0]] = False
    bg = np.zeros(A.shape[0]); bg[m.gid[O.owner != 0]] = oracle.mask(m.mask, b)[O.owner != 0]
    xs = np.zeros(A.shape[0]); xs[keep] = np.linalg.solve(A[np.ix_(keep, keep)], bg[keep])
    assert np.abs(x - xs[m.gid]).max() <= 1e-8 * np.abs(xs).max()
    x0, it0, st0, _ = pmg.pcg(O, 1.0, 0.0, np.zeros(O.n), 1e-10, 100, P.apply)
    assert it0 == 0 and np.all(x0 == 0.0)


@pytest.mark.slow
def test_pmg_iterations_nearly_E_independent():
    its = []
    for ne in (2, 4):
        m = mg.box_mesh(ne, ne, ne, 5, deform="bubble", dirichlet="all")
        O = oracle.Oracle.from_mesh(m)
        P = pmg.PMG(O, m.xyz, 1.0, 0.0)
        _, it, st, _ = pmg.pcg(O, 1.0, 0.0, mg.smooth_field(m, seed=1), 1e-8, 100, P.apply)
        assert st == 0
        its.append(it)
    assert its[1] <= 1.3 * its[0] + 1, its
