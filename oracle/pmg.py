"""p-multigrid preconditioner with Chebyshev smoothing -- TEST INFRASTRUCTURE.

P:195-198 "fast (exact or inexact) block solvers for local Poisson problems, which serve as local
smoothers for p-multigrid (pMG) [lottes05]"; "aggressive p-multigrid schedules of
p=7, 5, 3, and 1 with 6th-order Chebyshev smoothing"; Table 1 (pMG smoother, coarse
grid); SPEC S:337-343, S:362-379 for the V-cycle / Chebyshev interfaces.  Plain numpy around
the C oracle's operator, step by step in the order DESIGN.md "pMG readings" states:

  levels      l = 0..L with orders schedule[l] (default [N,5,3,1] for N >= 7, [N,3,1] for 4 <= N < 7,
              [N,1] for 2 <= N < 4; reading P1).  Level l is the same E elements rediscretised at
              order N_l: GLL-node coordinates interpolated from the finest level (P2), node ids from
              mesh entities (P3), the SEM operator A_l = M_l QQ^T_l (h1 K_l + h2 B_l) M_l, and its
              exact Jacobi diagonal.
  transfers   prolongation e_f = (J x J x J) e_c per element, J[I, i] = h^{N_c}_i(xi^{N_f}_I);
              restriction  f_c = M_c QQ^T_c (J^T x J^T x J^T)(O_f * r_f), O_f the owner-copy
              indicator, so R = P^T in the owner inner product (P4).
  smoother    Chebyshev iteration (Saad, Alg. 12.1) of degree k for A_l x = f with Jacobi
              preconditioning on [0.1 lam, 1.1 lam] (P5); lam from a 20-step Lanczos estimate (P6).
  coarse      degree-k_c Chebyshev on [c_lo lam_min, 1.1 lam_max] of the order-1 level (P7).
  V-cycle     x = S(f); r = f - A x; e = V(R r); x += P e; x = x + S(f - A x)   (symmetric, linear).
  PCG         Hestenes-Stiefel CG with z = V(r) in place of Dinv r.
"""
from __future__ import annotations

import numpy as np

import oracle as _or

MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------- helpers --
def default_schedule(N: int):
    """Reading P1 (P:522-523 for N = 7; SPEC S:417 for the other orders)."""
    if N >= 7:
        return [N, 5, 3, 1]
    if N >= 4:
        return [N, 3, 1]
    if N >= 2:
        return [N, 1]
    return [1]


def lagrange_interp(xf, xc):
    """J[I, i] = h_i(xf[I]) for the Lagrange basis h_i on the nodes xc (Eq. 3 interpolants),
    by the product formula; exactly 1 / 0 where xf[I] coincides with a node."""
    J = np.zeros((len(xf), len(xc)))
    for I, x in enumerate(xf):
        for i, xi in enumerate(xc):
            v = 1.0
            for m, xm in enumerate(xc):
                if m != i:
                    v *= (x - xm) / (xi - xm)
            J[I, i] = v
        hit = np.nonzero(xc == x)[0]
        if hit.size:
            J[I, :] = 0.0
            J[I, hit[0]] = 1.0
    return J


def splitmix64(z: int) -> int:
    """Counter-based generator shared by definition with the GPU path (reading P6)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def hash_field(gid):
    """v[l] = 2 * (splitmix64(gid[l]) >> 11) * 2^-53 - 1: continuous (a function of the id)."""
    return np.array([2.0 * ((splitmix64(int(g)) >> 11) * 2.0 ** -53) - 1.0 for g in np.asarray(gid)])


def interp_elements(J, U, Nin, Nout):
    """Per element U (E*(Nin+1)^3, i fastest) -> (J x J x J) U on (Nout+1)^3 points."""
    a, b = Nin + 1, Nout + 1
    Ue = np.asarray(U, dtype=np.float64).reshape(-1, a, a, a)          # [e, k, j, i]
    return np.einsum("Ii,Jj,Kk,ekji->eKJI", J, J, J, Ue).reshape(-1)


def interp_elements_T(J, V, Nbig, Nsmall):
    """Transpose: (J^T x J^T x J^T) V from (Nbig+1)^3 to (Nsmall+1)^3 points per element."""
    a = Nbig + 1
    Ve = np.asarray(V, dtype=np.float64).reshape(-1, a, a, a)          # [e, K, J, I]
    return np.einsum("Ii,Jj,Kk,eKJI->ekji", J, J, J, Ve).reshape(-1)


# ------------------------------------------------------- coarse node ids --
def coarse_ids(E, Nf, gid_f, mask_f, Nc):
    """Node ids and Dirichlet mask of the order-Nc level from the order-Nf ids (reading P3).

    Entity keys are fine node ids, so they are global without communication:
      vertex  fine id of the vertex node, slot 0
      edge    fine id of the edge node next to the end vertex with the smaller id; slot = distance
              (in coarse nodes) from that vertex
      face    fine id of the face node diagonally next to the corner with the smallest id;
              axis u toward the smaller-id neighbour corner of that origin, slot = u * (Nc+1) + v
      inside  fine id of the element's fine node (1,1,1); slot = i + (Nc+1)(j + (Nc+1) k)
    id = key * (Nc+1)^3 + slot.  The mask of a coarse node is the mask of its key node."""
    if Nf < 2:
        raise ValueError("coarsening needs a fine order >= 2")
    a, c = Nf + 1, Nc + 1
    S = c ** 3
    g = np.asarray(gid_f, dtype=np.int64).reshape(E, a, a, a)          # [e, K, J, I]
    mk = np.asarray(mask_f, dtype=np.uint8).reshape(E, a, a, a)
    gc = np.zeros((E, c, c, c), np.int64)
    mc = np.zeros((E, c, c, c), np.uint8)

    def fidx(ci):   # coarse end index -> fine end index
        return 0 if ci == 0 else Nf

    for e in range(E):
        G = lambda I, J_, K: int(g[e, K, J_, I])        # noqa: E731
        Mf = lambda I, J_, K: int(mk[e, K, J_, I])      # noqa: E731
        for k in range(c):
            for j in range(c):
                for i in range(c):
                    idx = [i, j, k]
                    ends = [q in (0, Nc) for q in idx]
                    ne = sum(ends)
                    if ne == 3:
                        F = [fidx(q) for q in idx]
                        key, slot = G(*F), 0
                    elif ne == 2:
                        d = ends.index(False)
                        F = [fidx(q) if ends[t] else 0 for t, q in enumerate(idx)]
                        A_ = list(F); A_[d] = 0
                        B_ = list(F); B_[d] = Nf
                        if G(*A_) < G(*B_):
                            kn = list(F); kn[d] = 1
                            slot = idx[d]
                        else:
                            kn = list(F); kn[d] = Nf - 1
                            slot = Nc - idx[d]
                        key = G(*kn)
                    elif ne == 1:
                        fixed = ends.index(True)
                        d1, d2 = [t for t in range(3) if t != fixed]
                        base = [0, 0, 0]; base[fixed] = fidx(idx[fixed])

                        def corner(o1, o2):
                            p = list(base); p[d1] = o1; p[d2] = o2
                            return p
                        cs = [(o1, o2) for o2 in (0, Nf) for o1 in (0, Nf)]
                        o1, o2 = min(cs, key=lambda o: G(*corner(*o)))
                        n1 = G(*corner(Nf - o1, o2))     # neighbour along d1
                        n2 = G(*corner(o1, Nf - o2))     # neighbour along d2
                        t1 = abs(idx[d1] - (0 if o1 == 0 else Nc))
                        t2 = abs(idx[d2] - (0 if o2 == 0 else Nc))
                        pu, pv = (t1, t2) if n1 < n2 else (t2, t1)
                        kn = corner(1 if o1 == 0 else Nf - 1, 1 if o2 == 0 else Nf - 1)
                        key, slot = G(*kn), pu * c + pv
                    else:
                        kn = [1, 1, 1]
                        key, slot = G(*kn), i + c * (j + c * k)
                    if ne == 3:
                        kn = F
                    gc[e, k, j, i] = key * S + slot
                    mc[e, k, j, i] = Mf(*kn)
    return gc.reshape(-1), mc.reshape(-1)


# ---------------------------------------------------------------- levels --
class Level:
    def __init__(self, O, h1, h2):
        self.O = O
        self.N = O.N
        self.h1, self.h2 = h1, h2
        self.dinv = O.dinv(h1, h2)
        self.lam_max = None
        self.lam_min = None

    def A(self, v):
        return self.O.apply(self.h1, self.h2, v)


def lanczos_bounds(L: Level, m: int = 20):
    """Extreme Ritz values of Dinv A after m Jacobi-PCG steps from v = M hash(gid) (reading P6):
    T[j,j] = 1/alpha_j + beta_{j-1}/alpha_{j-1}, T[j,j+1] = sqrt(beta_j)/alpha_j (Saad 6.7.3)."""
    O = L.O
    b = _or.mask(O.mask, hash_field(O.gid))
    r = b.copy()
    z = L.dinv * r
    p = z.copy()
    rho = O.dot(r, z)
    al, be = [], []
    for _ in range(m):
        w = L.A(p)
        sig = O.dot(p, w)
        if not sig > 0.0:
            break
        a = rho / sig
        r = r - a * w
        z = L.dinv * r
        rho1 = O.dot(r, z)
        bt = rho1 / rho
        al.append(a); be.append(bt)
        rho = rho1
        p = z + bt * p
    k = len(al)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / al[j] + (be[j - 1] / al[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(be[j]) / al[j]
    ev = np.linalg.eigvalsh(T)
    return float(ev[0]), float(ev[-1])


def chebyshev(A, dinv, f, x0, k, lo, hi):
    """Chebyshev iteration of degree k for A x = f, Jacobi-preconditioned, on [lo, hi]
    (Saad, Iterative Methods, Alg. 12.1; reading P5).  x0 None means x0 = 0."""
    theta = 0.5 * (hi + lo)
    delta = 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    if x0 is None:
        x = np.zeros_like(f)
        r = f.copy()
    else:
        x = x0.copy()
        r = f - A(x0)
    d = dinv * r / theta
    for i in range(1, k + 1):
        x = x + d
        if i == k:
            break
        r = r - A(d)
        rho1 = 1.0 / (2.0 * sigma - rho)
        d = rho1 * rho * d + (2.0 * rho1 / delta) * (dinv * r)
        rho = rho1
    return x


class PMG:
    """V-cycle preconditioner for the fine-level operator of oracle `O0` (readings P1-P7)."""

    def __init__(self, O0, xyz, h1, h2, schedule=None, degree=6, coarse_degree=20, lmin_frac=0.1,
                 lmax_factor=1.1, coarse_lo=1.0, lanczos_steps=20):
        self.schedule = list(schedule) if schedule is not None else default_schedule(O0.N)
        if self.schedule[0] != O0.N or self.schedule[-1] != 1 or any(
                a <= b for a, b in zip(self.schedule, self.schedule[1:])):
            raise ValueError("schedule must start at N, decrease strictly and end at 1 (S:367)")
        if degree < 1 or coarse_degree < 1:
            raise ValueError("Chebyshev degree < 1 (S:375)")
        self.degree, self.coarse_degree = degree, coarse_degree
        self.lmin_frac, self.lmax_factor, self.coarse_lo = lmin_frac, lmax_factor, coarse_lo
        N0, E = O0.N, O0.E
        x0, _ = _or.gll(N0)
        self.levels = [Level(O0, h1, h2)]
        self.J = []
        xyz = np.asarray(xyz, dtype=np.float64).reshape(3, -1)
        for Nc in self.schedule[1:]:
            xc, _ = _or.gll(Nc)
            Jg = lagrange_interp(xc, x0)                        # finest -> order Nc (coordinates)
            xyz_c = np.stack([interp_elements(Jg, xyz[d], N0, Nc) for d in range(3)])
            gid_c, mask_c = coarse_ids(E, N0, O0.gid, O0.mask, Nc)
            Oc = _or.Oracle(E, Nc, xyz_c, gid_c, mask_c)
            Nf = self.levels[-1].N
            xf, _ = _or.gll(Nf)
            self.J.append(lagrange_interp(xf, xc))              # order Nc -> order Nf (prolongation)
            self.levels.append(Level(Oc, h1, h2))
        for L in self.levels:
            L.lam_min, L.lam_max = lanczos_bounds(L, lanczos_steps)

    def smooth(self, l, f, x0):
        L = self.levels[l]
        return chebyshev(L.A, L.dinv, f, x0, self.degree, self.lmin_frac * L.lam_max, self.lmax_factor * L.lam_max)

    def coarse(self, f):
        L = self.levels[-1]
        return chebyshev(L.A, L.dinv, f, None, self.coarse_degree, self.coarse_lo * L.lam_min,
                         self.lmax_factor * L.lam_max)

    def prolong(self, l, ec):
        """Level l+1 -> level l."""
        return interp_elements(self.J[l], ec, self.levels[l + 1].N, self.levels[l].N)

    def restrict(self, l, r):
        """Level l -> level l+1: M_c QQ^T_c (J^T)^3 (O_l * r)."""
        Of, Oc = self.levels[l].O, self.levels[l + 1].O
        v = interp_elements_T(self.J[l], r * Of.owner, self.levels[l].N, self.levels[l + 1].N)
        return _or.mask(Oc.mask, Oc.gs_apply(v))

    def vcycle(self, f, l=0):
        if l == len(self.levels) - 1:
            return self.coarse(f)
        L = self.levels[l]
        x = self.smooth(l, f, None)
        r = f - L.A(x)
        e = self.vcycle(self.restrict(l, r), l + 1)
        x = x + self.prolong(l, e)
        return self.smooth(l, f, x)

    def apply(self, r):
        return self.vcycle(np.asarray(r, dtype=np.float64))


def pcg(O, h1, h2, b, tol, maxit, M):
    """Hestenes-Stiefel PCG with preconditioner z = M(r); owner-copy dots (reading 8).
    Returns (x, iters, status, hist)."""
    r = _or.mask(O.mask, b)
    x = np.zeros_like(r)
    z = M(r)
    p = z.copy()
    rho = O.dot(r, z)
    bb = np.sqrt(O.dot(r, r))
    hist = []
    k = 0
    status = 1
    while True:
        rn = np.sqrt(O.dot(r, r))
        hist.append(rn / bb if bb > 0 else 0.0)
        if rn <= tol * bb:
            status = 0
            break
        if k >= maxit:
            break
        w = O.apply(h1, h2, p)
        sig = O.dot(p, w)
        if not sig > 0.0:
            status = -5
            break
        a = rho / sig
        x = x + a * p
        r = r - a * w
        z = M(r)
        rho1 = O.dot(r, z)
        beta = rho1 / rho
        rho = rho1
        p = z + beta * p
        k += 1
    return x, k, status, np.array(hist)
