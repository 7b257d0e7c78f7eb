"""Dealiased advection `makef` -- TEST INFRASTRUCTURE.

P:417-420 "the nonlinear advection operator (makef), which is dealiased using N_q=11 quadrature
points in each direction"; "advection is dealiased with the 3/2's rule, the working data
set per element is 12^3, rather than 8^3"; Table 1 P:333 (makef 14.6%).
Readings M1-M4:

  M1  per element e, component c and local GLL test node l:
        F_c(l) = - sum_q  rho_q J_q  phi_l(xi_q)  ( u(xi_q) . grad u_c(xi_q) )
      u(xi_q) = sum_j u_j phi_j(xi_q) (the velocity interpolated to the fine points), grad from the
      derivative of the same interpolant, J_q and d r / d x from the isoparametric map
      x(xi) = sum_j x_j phi_j(xi); rho_q the tensor Gauss-Legendre weights.  Local (unassembled)
      output: the caller applies QQ^T (and any mask) as for every E-vector.
  M2  fine lattice: M Gauss-Legendre points per direction, M = ceil(3 (N+1) / 2) (the 3/2 rule;
      N = 7 -> M = 12, the paper's order N_q = 11); M >= N + 1 accepted.
  M3  with G_ab(q) = rho_q J_q (d r_a / d x_b)(xi_q):  (u . grad u_c) rho J = sum_a Ut_a d_a u_c,
      Ut_a = sum_b G_ab u_b  (contravariant velocity), d_a = d / d r_a of the interpolant.

Steps, plain numpy (numpy's leggauss and einsum are the library primitives used):
  J = Lagrange interpolation GLL(N) -> GL(M), Dq = J D (derivative at the fine points),
  geometry from the interpolated map, then M3 and the transpose interpolation back.
"""
from __future__ import annotations

import math

import numpy as np

import oracle as _or
from oracle.pmg import lagrange_interp


def default_m(N: int) -> int:
    """Reading M2: the 3/2 rule."""
    return int(math.ceil(1.5 * (N + 1)))


class Makef:
    def __init__(self, E, N, xyz, M=None):
        self.E, self.N = int(E), int(N)
        self.M = int(M) if M is not None else default_m(N)
        if self.M < self.N + 1:
            raise ValueError("N_q < N (S:468)")
        a, m = self.N + 1, self.M
        xg, _ = _or.gll(self.N)
        D = _or.deriv(self.N, xg)
        xq, wq = np.polynomial.legendre.leggauss(m)
        self.J = lagrange_interp(xq, xg)                   # [m][a]
        self.Dq = self.J @ D                               # [m][a]: d/dr of the interpolant at xi_q
        X = np.asarray(xyz, dtype=np.float64).reshape(3, self.E, a, a, a)   # [d][e][k][j][i]
        # dx_d / dr_a at the fine points, a = r (i), s (j), t (k)
        J_, Dq = self.J, self.Dq
        dr = np.einsum("Ii,Jj,Kk,dekji->deKJI", Dq, J_, J_, X)
        ds = np.einsum("Ii,Jj,Kk,dekji->deKJI", J_, Dq, J_, X)
        dt = np.einsum("Ii,Jj,Kk,dekji->deKJI", J_, J_, Dq, X)
        Jac = np.stack([dr, ds, dt], axis=1)               # [d][a][e][K][J][I] = dx_d / dr_a
        Jm = np.moveaxis(Jac, (0, 1), (-2, -1))            # [e][K][J][I][d][a]
        det = np.linalg.det(Jm)
        if np.any(det <= 0):
            raise ValueError("non-positive Jacobian at a fine point")
        inv = np.linalg.inv(Jm)                            # [..][a][b] = d r_a / d x_b
        rho = np.einsum("K,J,I->KJI", wq, wq, wq)
        # G_ab = rho J dr_a/dx_b  -> [e][a][b][K][J][I]
        self.G = np.moveaxis(inv * (rho[None, :, :, :, None, None] * det[..., None, None]), (-2, -1), (1, 2))

    def apply(self, u, v, w):
        """(F_x, F_y, F_z) of reading M1 for the velocity E-vectors (u, v, w)."""
        a = self.N + 1
        J_, Dq = self.J, self.Dq
        comps = [np.asarray(c, dtype=np.float64).reshape(self.E, a, a, a) for c in (u, v, w)]
        # velocity at the fine points and contravariant velocity Ut_a = sum_b G_ab u_b
        U = np.stack([np.einsum("Ii,Jj,Kk,ekji->eKJI", J_, J_, J_, c) for c in comps], axis=1)   # [e][b][..]
        Ut = np.einsum("eabKJI,ebKJI->eaKJI", self.G, U)
        out = []
        for c in comps:
            d0 = np.einsum("Ii,Jj,Kk,ekji->eKJI", Dq, J_, J_, c)
            d1 = np.einsum("Ii,Jj,Kk,ekji->eKJI", J_, Dq, J_, c)
            d2 = np.einsum("Ii,Jj,Kk,ekji->eKJI", J_, J_, Dq, c)
            f = Ut[:, 0] * d0 + Ut[:, 1] * d1 + Ut[:, 2] * d2
            out.append(-np.einsum("Ii,Jj,Kk,eKJI->ekji", J_, J_, J_, f).reshape(-1))
        return tuple(out)
