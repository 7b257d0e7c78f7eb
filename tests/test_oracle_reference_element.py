"""Pins for the oracle's GLL rule and derivative matrix (CPU only).

Each check ties oracle/nek_oracle.c to something other than itself: textbook
closed forms (tests/golden/*.txt, cited there), quadrature exactness, numpy's
independent Legendre root finder, and analytic derivatives.
"""
import math
import os

import numpy as np
import pytest
from numpy.polynomial import legendre as L

import oracle


def _read_golden(path):
    rows = []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append([c.strip() for c in line.split("|")])
    return rows


def _ev(expr):
    return float(eval(expr, {"sqrt": math.sqrt}))


def test_gll_closed_forms(golden_dir):
    for N, nodes, weights in _read_golden(os.path.join(golden_dir, "gll_closed_forms.txt")):
        N = int(N)
        x, w = oracle.gll(N)
        xe = np.array([_ev(s) for s in nodes.split(";")])
        we = np.array([_ev(s) for s in weights.split(";")])
        np.testing.assert_allclose(x, xe, rtol=0, atol=2e-16)
        np.testing.assert_allclose(w, we, rtol=0, atol=4e-16)


@pytest.mark.parametrize("N", range(1, 16))
def test_gll_invariants(N):
    x, w = oracle.gll(N)
    assert x[0] == -1.0 and x[-1] == 1.0
    assert np.all(np.diff(x) > 0)
    assert np.all(x == -x[::-1])                       # symmetric about 0
    assert np.all(w > 0)
    assert abs(w.sum() - 2.0) <= 1e-13                 # |[-1,1]|
    # exact for degree <= 2N-1 ...
    for k in range(2 * N):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.dot(w, x ** k) - exact) <= 1e-13, k
    # ... and not for degree 2N (threshold 1e-12, reading 19)
    assert abs(np.dot(w, x ** (2 * N)) - 2.0 / (2 * N + 1)) > 1e-12


@pytest.mark.parametrize("N", range(2, 16))
def test_gll_interior_nodes_are_roots_of_dPN(N):
    """Independent library route: numpy's companion-matrix roots of P_N'."""
    c = np.zeros(N + 1); c[N] = 1.0
    r = np.sort(np.real(L.legroots(L.legder(c))))
    x, _ = oracle.gll(N)
    np.testing.assert_allclose(x[1:-1], r, rtol=0, atol=1e-12)


def test_gll_rejects_bad_order():
    for N in (0, 16, -3):
        with pytest.raises(ValueError):
            oracle.gll(N)


@pytest.mark.parametrize("N", range(1, 16))
def test_deriv_rows_and_exactness(N):
    x, _ = oracle.gll(N)
    D = oracle.deriv(N, x)
    assert np.abs(D.sum(axis=1)).max() <= 1e-13 * max(1, N * N)      # d/dx 1 = 0
    np.testing.assert_allclose(D @ x, np.ones(N + 1), rtol=0, atol=1e-12 * N * N)
    for p in range(2, N + 1):                                          # exact on degree <= N
        np.testing.assert_allclose(D @ x ** p, p * x ** (p - 1), rtol=0, atol=1e-11 * N * N)
    assert abs(D[0, 0] + N * (N + 1) / 4.0) <= 1e-14 * N * N
    assert abs(D[N, N] - N * (N + 1) / 4.0) <= 1e-14 * N * N


def test_deriv_x6_N6():
    """SPEC S:53 worked example: N=6, d/dx x^6 = 6x^5 at every node within 1e-11."""
    x, _ = oracle.gll(6)
    D = oracle.deriv(6, x)
    assert np.abs(D @ x ** 6 - 6 * x ** 5).max() <= 1e-11


def test_stiffness_1d_closed_forms(golden_dir):
    for N, ent in _read_golden(os.path.join(golden_dir, "stiffness_1d.txt")):
        N = int(N)
        K = np.array([_ev(s) for s in ent.split(";")]).reshape(N + 1, N + 1)
        x, w = oracle.gll(N)
        D = oracle.deriv(N, x)
        np.testing.assert_allclose(D.T @ np.diag(w) @ D, K, rtol=0, atol=1e-14)


@pytest.mark.parametrize("N", [3, 5, 7, 9, 12, 15])
def test_deriv_matches_vandermonde_route(N):
    """D (closed form) vs V_r V^{-1} (Legendre-Vandermonde), an independent route."""
    from oracle.assemble import vandermonde_deriv
    x, _ = oracle.gll(N)
    np.testing.assert_allclose(oracle.deriv(N, x), vandermonde_deriv(x), rtol=0, atol=1e-10 * N)
