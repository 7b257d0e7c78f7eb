"""Pins for the oracle's dealiased advection (NEXT #4).

  * u = 0 gives 0;
  * a linear velocity u(x) = c + B x on a general affine mesh: (u . grad) u = B c + B^2 x is linear,
    phi_l times it has degree N + 1 <= 2N - 1, so the element integral is exactly the GLL sum:
    F(l) = - w_l J (B c + B^2 x_l) (closed form through the GLL weights, an independent route);
  * dealiasing (reading M2): for velocities that are polynomials of degree <= N per reference
    direction on affine elements the integrand has degree <= 3N <= 2M - 1, so the 3/2-rule lattice
    equals a much finer one (M = 20) to rounding, while M = N + 1 shows the aliasing gap;
  * spectral accuracy: for a smooth analytic velocity on a curved (bubble) mesh, F approaches the
    fine-lattice projection of the exact (u . grad) u as N grows."""
import numpy as np
import pytest

import oracle
from oracle.makef import Makef, default_m
from workloads import meshgen as mg


def affine_mesh(N, A=None, t=(0.3, -0.2, 0.1)):
    m = mg.box_mesh(3, 2, 2, N, deform="affine")
    A = np.array([[1.2, 0.3, -0.1], [0.1, 0.9, 0.2], [-0.2, 0.15, 1.1]]) if A is None else A
    m.xyz = (A @ m.xyz) + np.asarray(t)[:, None]
    return m


def test_default_lattice():
    assert default_m(7) == 12 and default_m(3) == 6 and default_m(1) == 3
    with pytest.raises(ValueError):
        m = mg.box_mesh(1, 1, 1, 5)
        Makef(m.E, m.N, m.xyz, M=5)


def test_zero_velocity():
    m = mg.box_mesh(2, 2, 1, 4, deform="bubble")
    F = Makef(m.E, m.N, m.xyz).apply(*(np.zeros(m.n_local),) * 3)
    assert all(np.all(f == 0.0) for f in F)


@pytest.mark.parametrize("N", [2, 3, 5, 7])
def test_linear_velocity_closed_form(N):
    m = affine_mesh(N)
    c = np.array([0.4, -0.7, 0.25])
    B = np.array([[0.3, -0.5, 0.2], [0.6, 0.1, -0.4], [-0.2, 0.35, 0.15]])
    X = m.xyz
    U = c[:, None] + B @ X
    F = Makef(m.E, m.N, m.xyz).apply(*U)
    adv = (B @ c)[:, None] + B @ (B @ X)           # (u . grad) u at the nodes
    O = oracle.Oracle.from_mesh(m)                 # wJ = w_i w_j w_k J at the GLL nodes
    for d in range(3):
        want = -O.wJ * adv[d]
        assert np.abs(F[d] - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("N", [3, 5, 7])
def test_dealiasing_exact_for_degree_N_velocity(N):
    m = affine_mesh(N)
    x, y, z = m.xyz
    # a polynomial velocity of degree N in the physical (= affine reference) coordinates
    p = N
    U = [x ** p - 0.5 * y + z * y, y ** p + 0.3 * x * z, -z ** p + x * y]
    F12 = Makef(m.E, m.N, m.xyz).apply(*U)
    F20 = Makef(m.E, m.N, m.xyz, M=20).apply(*U)
    Fal = Makef(m.E, m.N, m.xyz, M=N + 1).apply(*U)
    for a, b, c in zip(F12, F20, Fal):
        s = np.abs(b).max()
        assert np.abs(a - b).max() <= 1e-12 * s
        assert np.abs(c - b).max() > 1e-9 * s          # the aliasing gap, far above rounding


def test_spectral_accuracy_on_curved_mesh():
    errs = []
    for N in (3, 5, 7):
        m = mg.box_mesh(2, 2, 2, N, deform="bubble", eps=0.05)
        mk = Makef(m.E, m.N, m.xyz)
        x, y, z = m.xyz
        U = [np.sin(x) * np.cos(y), -np.cos(x) * np.sin(y) * np.cos(z), 0.3 * np.sin(z) * x]
        F = mk.apply(*U)
        # exact (u . grad) u_x at the fine points, projected with the same quadrature
        a = N + 1
        J = mk.J
        X = np.asarray(m.xyz).reshape(3, m.E, a, a, a)
        xq = [np.einsum("Ii,Jj,Kk,ekji->eKJI", J, J, J, X[d]) for d in range(3)]
        ux, uy, uz = np.sin(xq[0]) * np.cos(xq[1]), -np.cos(xq[0]) * np.sin(xq[1]) * np.cos(xq[2]), 0.3 * np.sin(xq[2]) * xq[0]
        adv_x = ux * np.cos(xq[0]) * np.cos(xq[1]) + uy * (-np.sin(xq[0]) * np.sin(xq[1]))
        rhoJ = np.linalg.det(np.moveaxis(np.stack([
            np.stack([np.einsum("Ii,Jj,Kk,ekji->eKJI", mk.Dq, J, J, X[d]),
                      np.einsum("Ii,Jj,Kk,ekji->eKJI", J, mk.Dq, J, X[d]),
                      np.einsum("Ii,Jj,Kk,ekji->eKJI", J, J, mk.Dq, X[d])]) for d in range(3)]), (0, 1), (-2, -1)))
        _, wq = np.polynomial.legendre.leggauss(mk.M)
        rhoJ = rhoJ * np.einsum("K,J,I->KJI", wq, wq, wq)
        ref = -np.einsum("Ii,Jj,Kk,eKJI->ekji", J, J, J, rhoJ * adv_x).reshape(-1)
        errs.append(np.abs(F[0] - ref).max() / np.abs(ref).max())
    assert errs[-1] <= 1e-5 and errs[2] < errs[1] < errs[0], errs
