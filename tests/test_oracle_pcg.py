"""Pins for the oracle's Jacobi-PCG and the whole path (CPU only).

References: CG facts (b = 0 -> 0 iterations; a diagonal operator with exact
Jacobi converges in one step), a dense direct solve of the assembled masked
system, A-norm monotonicity of the CG error, and the paper's spectral
convergence claim C = O(h^N) / "more efficient to increase N"
checked on the manufactured solution u = sin(pi x) sin(pi y) sin(pi z).
"""
import numpy as np
import pytest

import oracle
from oracle.assemble import assemble_box
from workloads import meshgen as mg


def _rhs(O, m):
    """b = M QQ^T (wJ * f) for the manufactured f = 3 pi^2 u* (lumped GLL mass)."""
    u, f = mg.manufactured(m)
    return oracle.mask(m.mask, O.gs_apply(O.wJ * f)), u


def test_pcg_zero_rhs():
    m = mg.config_mesh(1)
    O = oracle.Oracle.from_mesh(m)
    x, it, st, hist = O.pcg(1.0, 0.0, np.zeros(m.n_local), 1e-10, 50)
    assert it == 0 and st == 0 and np.all(x == 0)


def test_pcg_pure_mass_one_iteration():
    """(h1,h2) = (0,1): the operator is diagonal, Jacobi is exact -> 1 iteration."""
    m = mg.config_mesh(1)
    O = oracle.Oracle.from_mesh(m)
    b = mg.smooth_field(m, seed=4)
    x, it, st, hist = O.pcg(0.0, 1.0, b, 1e-12, 20)
    assert st == 0 and it == 1
    np.testing.assert_allclose(O.apply(0.0, 1.0, x), oracle.mask(m.mask, b), rtol=0, atol=1e-14 * np.abs(b).max())


def _dense_system(m, h1, h2):
    x, w = oracle.gll(m.N)
    A, _ = assemble_box(m.shape, m.N, h1, h2, x, w, deform=m.deform, eps=m.eps)
    ng = A.shape[0]
    bmask = np.zeros(ng, bool)
    bmask[m.gid[m.mask != 0]] = True
    keep = ~bmask
    return A, keep


@pytest.mark.parametrize("h", [(1.0, 0.0), (1.0, 10.0)])
def test_pcg_matches_dense_solve_and_error_monotone(h):
    h1, h2 = h
    m = mg.config_mesh(1)
    O = oracle.Oracle.from_mesh(m)
    b = mg.smooth_field(m, seed=9)
    A, keep = _dense_system(m, h1, h2)
    ng = A.shape[0]
    bg = np.zeros(ng); bg[m.gid] = b                      # b is continuous
    Ak = A[np.ix_(keep, keep)]
    xs = np.zeros(ng); xs[keep] = np.linalg.solve(Ak, bg[keep])
    kappa = np.linalg.cond(Ak)
    tol = 1e-10
    x, it, st, hist = O.pcg(h1, h2, b, tol, 500)
    assert st == 0 and it > 1
    err = np.abs(x - xs[m.gid]).max() / np.abs(xs).max()
    assert err <= kappa * tol
    # A-norm of the error decreases monotonically (the CG optimality property)
    prev = np.inf
    for k in range(1, it + 1):
        xk, _, _, _ = O.pcg(h1, h2, b, 0.0, k)
        e = xs.copy(); e[m.gid] -= xk
        an = e[keep] @ Ak @ e[keep]
        assert an <= prev * (1 + 1e-12)
        prev = an


def test_manufactured_config1():
    """Config 1 (BASELINE configs[0]): deformed 2^3 box, N=3, tol 1e-10."""
    m = mg.config_mesh(1)
    O = oracle.Oracle.from_mesh(m)
    b, u = _rhs(O, m)
    x, it, st, hist = O.pcg(1.0, 0.0, b, 1e-10, 500)
    assert st == 0
    err = np.abs(x - u).max()
    # SURVEY 8(c) "Whole path" pin: 24 iterations, max error 1.54e-3 (the oracle is deterministic)
    assert it == 24
    assert abs(err - 1.54e-3) <= 0.01 * 1.54e-3
    assert hist[0] == 1.0 and hist[-1] <= 1e-10


def test_manufactured_8cubed_N7():
    """8^3 elements, N = 7, bubble map, tol 1e-10 -> 336 iterations, max error 6.0e-12."""
    m = mg.box_mesh(8, 8, 8, 7, deform="bubble", eps=0.05, dirichlet="all")
    O = oracle.Oracle.from_mesh(m)
    b, u = _rhs(O, m)
    x, it, st, hist = O.pcg(1.0, 0.0, b, 1e-10, 2000)
    assert st == 0 and it == 336
    assert abs(np.abs(x - u).max() - 6.0e-12) <= 0.05 * 6.0e-12


@pytest.mark.slow
def test_manufactured_config2():
    """config 2 (16^3, N = 7), tol 1e-10 -> 665 iterations, max error 6.4e-12,
    ||r_100|| / ||b|| = 0.12."""
    m = mg.config_mesh(2)
    O = oracle.Oracle.from_mesh(m)
    b, u = _rhs(O, m)
    x, it, st, hist = O.pcg(1.0, 0.0, b, 1e-10, 2000)
    assert st == 0 and it == 665
    assert abs(np.abs(x - u).max() - 6.4e-12) <= 0.05 * 6.4e-12
    assert abs(hist[100] - 0.12) <= 0.005


@pytest.mark.slow
def test_spectral_convergence():
    """err(N=8) <= 1e-4 err(N=4) on the deformed 2^3 box."""
    errs = {}
    for N in (4, 8):
        m = mg.box_mesh(2, 2, 2, N, deform="bubble", eps=0.05, dirichlet="all")
        O = oracle.Oracle.from_mesh(m)
        b, u = _rhs(O, m)
        x, it, st, _ = O.pcg(1.0, 0.0, b, 1e-12, 2000)
        assert st == 0
        errs[N] = np.abs(x - u).max()
    assert errs[8] <= 1e-4 * errs[4]


def test_pcg_reports_indefinite():
    """<p, A p> <= 0 -> error status -5: negative h1 makes A negative definite."""
    m = mg.config_mesh(1)
    O = oracle.Oracle.from_mesh(m)
    b = mg.smooth_field(m, seed=1)
    dinv = O.dinv(1.0, 0.0)
    _, it, st, _ = O.pcg(-1.0, 0.0, b, 1e-10, 10, dinv=dinv)
    assert st == -5 and it == 0
