"""Tiny brute-force assembler -- TEST INFRASTRUCTURE (pins the oracle).

Builds the assembled global matrix A = sum_e Q_e^T A_e Q_e of the SEM
Helmholtz operator on a structured box (the plain definition of what the
matrix-free apply computes, P:188-192 / SURVEY 8(c)), by a route independent
of oracle/nek_oracle.c:

  * derivatives of the Lagrange basis through a Legendre-Vandermonde matrix,
    D_alt = V_r V^{-1} (V_ij = P_j(x_i), V_r,ij = P_j'(x_i)), not the closed form;
  * the Jacobian of the element map from the ANALYTIC derivative of the mesh
    map (affine box composed with the bubble / sin / shear deformation), not by
    differentiating nodal coordinates;
  * dense element matrices A_e[p,q] = sum_quad w_q J (h1 grad phi_p . grad phi_q)
    + h2 w_q J delta_pq with GLL quadrature at the nodes, scattered into a
    dense n_g x n_g matrix.

Only the GLL nodes/weights are shared with the oracle (they are pinned
separately against closed forms).
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as L


def vandermonde_deriv(x):
    N = x.size - 1
    V = np.zeros((N + 1, N + 1)); Vr = np.zeros((N + 1, N + 1))
    for j in range(N + 1):
        c = np.zeros(N + 1); c[j] = 1.0
        V[:, j] = L.legval(x, c)
        Vr[:, j] = L.legval(x, L.legder(c))
    return Vr @ np.linalg.inv(V)


def _map_and_jac(x0, extent, deform, eps):
    """phi(x0) and d phi / d x0 (3x3 per point) of the deformation, analytically."""
    Lv = np.asarray(extent, dtype=float)
    xh = x0 / Lv[:, None]
    npt = x0.shape[1]
    Jd = np.zeros((npt, 3, 3))
    for d in range(3):
        Jd[:, d, d] = 1.0
    if deform in ("none", "affine"):
        return x0.copy(), Jd
    if deform in ("bubble", "sin"):
        if deform == "bubble":
            f = [xh[c] * (1 - xh[c]) for c in range(3)]
            df = [1 - 2 * xh[c] for c in range(3)]
            scale = 64.0
        else:
            f = [np.sin(np.pi * xh[c]) for c in range(3)]
            df = [np.pi * np.cos(np.pi * xh[c]) for c in range(3)]
            scale = 1.0
        b = scale * f[0] * f[1] * f[2]
        grad = [scale * df[0] * f[1] * f[2], scale * f[0] * df[1] * f[2], scale * f[0] * f[1] * df[2]]
        x = x0 + eps * Lv[:, None] * b[None, :]
        for d in range(3):
            for c in range(3):
                Jd[:, d, c] += eps * Lv[d] * grad[c] / Lv[c]
        return x, Jd
    if deform == "shear":
        x = x0.copy()
        x[0] += eps * Lv[0] * np.sin(np.pi * xh[1])
        Jd[:, 0, 1] += eps * Lv[0] * np.pi * np.cos(np.pi * xh[1]) / Lv[1]
        return x, Jd
    raise ValueError(deform)


def assemble_box(shape, N, h1, h2, xi, wq, deform="bubble", eps=0.05, extent=(1.0, 1.0, 1.0)):
    """Dense assembled matrix (n_g x n_g) in lattice numbering
    g = I + NX (J + NY K), plus the local->global map of every element."""
    Ex, Ey, Ez = shape
    Nq = N + 1
    NX, NY, NZ = Ex * N + 1, Ey * N + 1, Ez * N + 1
    ng = NX * NY * NZ
    Dr = vandermonde_deriv(np.asarray(xi))
    I1 = np.eye(Nq)
    Br = np.kron(I1, np.kron(I1, Dr))      # index i + Nq j + Nq^2 k: i fastest
    Bs = np.kron(I1, np.kron(Dr, I1))
    Bt = np.kron(Dr, np.kron(I1, I1))
    W = np.einsum("k,j,i->kji", wq, wq, wq).reshape(-1)
    r = np.asarray(xi)
    R = np.broadcast_to(r[None, None, :], (Nq, Nq, Nq)).reshape(-1)
    S = np.broadcast_to(r[None, :, None], (Nq, Nq, Nq)).reshape(-1)
    T = np.broadcast_to(r[:, None, None], (Nq, Nq, Nq)).reshape(-1)
    A = np.zeros((ng, ng))
    h = np.array([extent[0] / Ex, extent[1] / Ey, extent[2] / Ez])
    l2g = []
    for ez in range(Ez):
        for ey in range(Ey):
            for ex in range(Ex):
                x0 = np.stack([h[0] * (ex + (R + 1) / 2), h[1] * (ey + (S + 1) / 2), h[2] * (ez + (T + 1) / 2)])
                _, Jd = _map_and_jac(x0, extent, deform, eps)
                Jm = Jd * (h / 2)[None, None, :]          # dx/dr = dphi/dx0 * diag(h/2)
                det = np.linalg.det(Jm)
                Jinv = np.linalg.inv(Jm)                  # rows: grad r, grad s, grad t
                Bx = [sum(Jinv[:, a, d][:, None] * Bmat for a, Bmat in enumerate((Br, Bs, Bt)))
                      for d in range(3)]
                wJ = W * det
                Ae = h1 * sum(Bx[d].T @ (wJ[:, None] * Bx[d]) for d in range(3)) + h2 * np.diag(wJ)
                i = np.arange(Nq)
                Ig = (ex * N + i)[None, None, :]
                Jg = (ey * N + i)[None, :, None]
                Kg = (ez * N + i)[:, None, None]
                g = (Ig + NX * (Jg + NY * Kg)).reshape(-1)
                A[np.ix_(g, g)] += Ae
                l2g.append(g)
    return A, np.concatenate(l2g)
