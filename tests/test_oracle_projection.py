"""Pins for the oracle's projection initial guess (NEXT #2).

References: CG on the projected residual must reproduce the plain solve when the space is
empty; a repeated right-hand side lies in the space (0 iterations); the stored basis is
A-orthonormal; the projected guess never has a larger A-norm error than the zero guess
(dense solve of the assembled system as the exact solution); and over a slowly drifting
sequence of right-hand sides the space lowers the mean iteration count."""
import numpy as np
import pytest

import oracle
from oracle.assemble import assemble_box
from oracle.projection import Projection
from workloads import meshgen as mg


@pytest.fixture(scope="module")
def setup():
    m = mg.box_mesh(3, 3, 3, 4, deform="bubble", dirichlet="all")
    return m, oracle.Oracle.from_mesh(m)


def test_empty_space_equals_plain_pcg(setup):
    m, O = setup
    b = mg.smooth_field(m, seed=1)
    P = Projection(O, 8)
    x, it, st = P.solve(1.0, 0.0, b, 1e-10, 500)
    x0, it0, st0, _ = O.pcg(1.0, 0.0, b, 1e-10, 500)
    assert it == it0 and np.array_equal(x, x0)


def test_repeated_rhs_needs_no_iterations(setup):
    m, O = setup
    b = mg.smooth_field(m, seed=2)
    P = Projection(O, 8)
    x1, it1, _ = P.solve(1.0, 0.0, b, 1e-10, 500)
    x2, it2, _ = P.solve(1.0, 0.0, b, 1e-10, 500)
    assert it1 > 5 and it2 == 0
    assert np.abs(x2 - x1).max() <= 1e-8 * np.abs(x1).max()


def test_basis_A_orthonormal_and_guess_no_worse(setup):
    m, O = setup
    P = Projection(O, 6)
    rng = np.random.default_rng(0)
    b0, b1 = mg.smooth_field(m, seed=3), mg.smooth_field(m, seed=4)
    for t in range(6):
        P.solve(1.0, 0.0, b0 + 0.3 * t * b1, 1e-10, 500)
    l = len(P.X)
    assert l == 6
    Gm = np.array([[P._dot(xi, O.apply(1.0, 0.0, xj)) for xj in P.X] for xi in P.X])
    assert np.abs(Gm - np.eye(l)).max() <= 1e-9
    # exact solution of a new right-hand side by a dense solve
    x, w = oracle.gll(m.N)
    A, _ = assemble_box(m.shape, m.N, 1.0, 0.0, x, w, deform=m.deform, eps=m.eps)
    keep = np.ones(A.shape[0], bool); keep[m.gid[m.mask != 0]] = False
    bn = b0 + 2.0 * b1 + 0.1 * mg.smooth_field(m, seed=9)
    bg = np.zeros(A.shape[0]); bg[m.gid] = bn
    xs = np.zeros(A.shape[0]); xs[keep] = np.linalg.solve(A[np.ix_(keep, keep)], bg[keep])
    xbar = sum(P._dot(xi, oracle.mask(m.mask, bn)) * xi for xi in P.X)
    e_proj = xs.copy(); e_proj[m.gid] -= xbar
    enorm = lambda e: e[keep] @ A[np.ix_(keep, keep)] @ e[keep]
    assert enorm(e_proj) <= enorm(xs) + 1e-12


def test_drifting_sequence_fewer_iterations(setup):
    m, O = setup
    b0, b1 = mg.smooth_field(m, seed=5), mg.smooth_field(m, seed=6)
    means = {}
    for L in (0, 8):
        P = Projection(O, L)
        its = []
        for t in range(16):
            _, it, st = P.solve(1.0, 0.0, b0 + 0.01 * t * b1, 1e-8, 500)
            assert st == 0
            its.append(it)
        means[L] = np.mean(its[4:])
    assert means[8] < means[0]
