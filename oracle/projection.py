"""Projection initial guess -- TEST INFRASTRUCTURE.

P:513-519: "generate an initial guess for the pressure (and velocity) by
projecting onto the space of prior solutions [fisc98]" and "increasing the
number of prior solutions from 8 to 30".  Fischer's
method, step by step (plain numpy around the C oracle's operator and PCG):

  space: x_1..x_l A-orthonormal (x_i^T A x_j = delta_ij), with b_i = A x_i kept
  solve(b):
    alpha_i = <x_i, b>                      (owner-copy inner products, reading 8)
    xbar = sum_i alpha_i x_i,  bbar = sum_i alpha_i b_i
    db = M b - bbar                         (the projected residual)
    solve A dx = db with Jacobi-PCG (x0 = 0) to ||r|| <= tol ||M b||
    x = xbar + dx
  update(dx) -- classical Gram-Schmidt applied twice in the A inner product:
    if l < L:  repeat twice { c_i = <b_i, dx>; dx -= sum c_i x_i; adx -= sum c_i b_i }   (adx = A dx)
               nrm = sqrt(<dx, adx>); if nrm > 0: x_{l+1} = dx / nrm, b_{l+1} = adx / nrm
    else:      restart with the current solution: x_1 = x / sqrt(<x, A x>), b_1 = A x_1
"""
from __future__ import annotations

import numpy as np


class Projection:
    def __init__(self, O, max_vectors: int):
        self.O = O
        self.L = int(max_vectors)
        self.X, self.B = [], []
        self.hkey = None

    def reset(self):
        self.X, self.B = [], []

    def _dot(self, a, b):
        o = self.O.owner != 0
        return float(np.dot(a[o], b[o]))   # numpy pairwise sum: a different order from the GPU's (tolerance-compared)

    def solve(self, h1, h2, b, tol, maxit):
        O = self.O
        if self.hkey != (h1, h2):
            self.reset()
            self.hkey = (h1, h2)
        mb = O.mask.astype(bool)
        bm = np.array(b, dtype=np.float64, copy=True)
        bm[mb] = 0.0
        xbar = np.zeros(O.n)
        bbar = np.zeros(O.n)
        for xi, bi in zip(self.X, self.B):
            a = self._dot(xi, bm)
            xbar += a * xi
            bbar += a * bi
        db = bm - bbar
        bnorm = np.sqrt(self._dot(bm, bm))
        dnorm = np.sqrt(self._dot(db, db))
        if bnorm == 0.0:
            return np.zeros(O.n), 0, 0
        rel = tol * bnorm / dnorm if dnorm > 0 else 1.0
        dx, it, st, _ = O.pcg(h1, h2, db, min(rel, 1.0) if rel < 1.0 else 1.0, maxit)
        x = xbar + dx
        self._update(h1, h2, x, dx, bm)
        return x, it, st

    def _update(self, h1, h2, x, dx, bm):
        O = self.O
        if self.L == 0:
            return
        if len(self.X) < self.L:
            v = dx.copy()
            av = O.apply(h1, h2, v)
            for _ in range(2):
                c = [self._dot(bi, v) for bi in self.B]
                for ci, xi, bi in zip(c, self.X, self.B):
                    v -= ci * xi
                    av -= ci * bi
            nrm2 = self._dot(v, av)
            if nrm2 > 0.0:
                nrm = np.sqrt(nrm2)
                self.X.append(v / nrm)
                self.B.append(av / nrm)
        else:
            ax = O.apply(h1, h2, x)
            nrm = np.sqrt(self._dot(x, ax))
            self.X, self.B = [x / nrm], [ax / nrm]
