"""CPU oracle for the NekRS hot path (arXiv 2409.19119) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2409_19119_b200) never imports it and shares no code with it.

The arithmetic lives in plain C (oracle/nek_oracle.c, compiled with gcc -O2, no
-ffast-math, no FMA contraction); this module loads it with ctypes and adds the
plain-numpy glue: owner flags, the Jacobi inverse diagonal, and the multi-rank
gather-scatter emulation (reading 7: per-rank left folds, then totals summed in
ascending rank order).

Every function cites the passage it follows; the pins that tie it to something
other than itself are listed in DESIGN.md "Oracle pins" and live in
tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nek_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc -O2; checker build, not a product), and the same source with
    -fopenmp for the all-cores timing of bench.py's cpu_baseline (element / run / point loops split
    over threads, inner products sequential: bitwise the same results)."""
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            tmp = out + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
                                   "-ffp-contract=off", *extra, "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, out)
    return _LIB


_lib = None
_libs = {}
_use_omp = False


def use_openmp(on: bool):
    """Route every oracle call through the OpenMP build (True) or the serial one (False)."""
    global _use_omp, _lib
    _use_omp = bool(on)
    _lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        path = _LIB_OMP if _use_omp else _LIB
        if path in _libs:
            _lib = _libs[path]
            return _lib
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_gll.argtypes = [i32, P, P]; L.or_gll.restype = i32
        L.or_deriv.argtypes = [i32, P, P]; L.or_deriv.restype = None
        L.or_geom.argtypes = [i64, i32, P, P, P, P, P, P]; L.or_geom.restype = i32
        L.or_ax_local.argtypes = [i64, i32, P, P, P, dbl, dbl, P, P]; L.or_ax_local.restype = None
        L.or_gs_map.argtypes = [i64, P, i64, P, P, P]; L.or_gs_map.restype = i64
        L.or_gs_apply.argtypes = [i64, P, P, P]; L.or_gs_apply.restype = None
        L.or_gs_partial.argtypes = [i64, P, P, P, P]; L.or_gs_partial.restype = None
        L.or_mask.argtypes = [i64, P, P]; L.or_mask.restype = None
        L.or_diag_local.argtypes = [i64, i32, P, P, P, dbl, dbl, P]; L.or_diag_local.restype = None
        L.or_pcg.argtypes = [i64, i32, P, P, P, P, i64, P, P, P, P, dbl, dbl, P, P, dbl, i32,
                             ctypes.POINTER(ctypes.c_int), P]
        L.or_pcg.restype = i32
        L.or_op_apply.argtypes = [i64, i32, P, P, P, P, i64, P, P, dbl, dbl, P, P]
        L.or_op_apply.restype = None
        L.or_set_dot_mode.argtypes = [i32]; L.or_set_dot_mode.restype = None
        L.or_set_upd_fma.argtypes = [i32]; L.or_set_upd_fma.restype = None
        L.or_triad_gbps.argtypes = [i64, i32]; L.or_triad_gbps.restype = dbl
        L.or_threads.argtypes = []; L.or_threads.restype = i32
        _libs[path] = L
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ------------------------------------------------------------------ basics --
def gll(N: int):
    """GLL nodes (ascending) and weights, order N (Eq. 3)."""
    x = np.zeros(N + 1); w = np.zeros(N + 1)
    if lib().or_gll(N, _p(x), _p(w)) != 0:
        raise ValueError(f"order N={N} outside [1,15] (S:38)")
    return x, w


def deriv(N: int, x=None):
    """D[i,j] = h_j'(x_i) on the GLL nodes (Eq. 3 interpolants)."""
    if x is None:
        x, _ = gll(N)
    D = np.zeros((N + 1, N + 1))
    lib().or_deriv(N, _p(_c(x, np.float64)), _p(D))
    return D


def geom(E: int, N: int, xyz):
    """Geometric factors G[E,6,Nq^3] (rr,rs,rt,ss,st,tt) and wJ[E*Nq^3]
    (reading 4).  Raises on J <= 0."""
    x, w = gll(N)
    D = deriv(N, x)
    P3 = (N + 1) ** 3
    xyz = _c(xyz, np.float64)
    G = np.zeros((E, 6, P3)); wJ = np.zeros(E * P3)
    bad = ctypes.c_int64(-1)
    st = lib().or_geom(E, N, _p(D), _p(w), _p(xyz), _p(G), _p(wJ), ctypes.addressof(bad))
    if st != 0:
        l = bad.value
        raise ValueError(f"non-positive Jacobian at element {l // P3}, node {l % P3}")
    return G, wJ


def ax_local(E, N, G, wJ, h1, h2, u, D=None):
    """w = h1 K_L u + h2 B_L u, element by element."""
    if D is None:
        D = deriv(N)
    u = _c(u, np.float64); w = np.zeros_like(u)
    lib().or_ax_local(E, N, _p(_c(D, np.float64)), _p(_c(G, np.float64)), _p(_c(wJ, np.float64)),
                      float(h1), float(h2), _p(u), _p(w))
    return w


class GsMap:
    """Canonical gather-scatter map (reading 7)."""

    def __init__(self, gid, min_len: int = 2):
        gid = _c(gid, np.int64)
        n = gid.size
        perm = np.zeros(max(n, 1), np.int32); offs = np.zeros(n + 1, np.int64); rgid = np.zeros(max(n, 1), np.int64)
        nr = lib().or_gs_map(n, _p(gid), int(min_len), _p(perm), _p(offs), _p(rgid))
        self.nruns = int(nr)
        self.offs = offs[: nr + 1].copy()
        self.perm = perm[: self.offs[-1]].copy()
        self.rgid = rgid[:nr].copy()
        self.n = n

    def apply(self, v):
        """v <- QQ^T v (left fold in canonical order, then broadcast)."""
        v = np.array(v, dtype=np.float64, copy=True)
        lib().or_gs_apply(self.nruns, _p(self.perm), _p(self.offs), _p(v))
        return v

    def partial(self, v):
        v = _c(v, np.float64)
        out = np.zeros(max(self.nruns, 1))
        lib().or_gs_partial(self.nruns, _p(self.perm), _p(self.offs), _p(v), _p(out))
        return out[: self.nruns]


def mask(m, v):
    v = np.array(v, dtype=np.float64, copy=True)
    v[np.asarray(m) != 0] = 0.0
    return v


def owner_flags(gid):
    """1 on the smallest local index of every gid (reading 8)."""
    gid = np.asarray(gid)
    _, first = np.unique(gid, return_index=True)
    o = np.zeros(gid.size, np.uint8)
    o[first] = 1
    return o


def multiplicity(gid):
    gid = np.asarray(gid)
    _, inv, cnt = np.unique(gid, return_inverse=True, return_counts=True)
    return cnt[inv]


# ------------------------------------------------------------ the operator --
class Oracle:
    """Single-rank oracle for one mesh: geometry, maps, operator, Jacobi, PCG."""

    def __init__(self, E, N, xyz, gid, dirichlet=None):
        self.E, self.N = int(E), int(N)
        self.Nq = self.N + 1
        self.n = self.E * self.Nq ** 3
        self.x, self.w = gll(self.N)
        self.D = deriv(self.N, self.x)
        self.G, self.wJ = geom(self.E, self.N, xyz)
        self.gid = _c(gid, np.int64)
        self.mask = np.zeros(self.n, np.uint8) if dirichlet is None else _c(dirichlet, np.uint8)
        self.gs = GsMap(self.gid)
        self.owner = owner_flags(self.gid)

    @classmethod
    def from_mesh(cls, mesh):
        return cls(mesh.E, mesh.N, mesh.xyz, mesh.gid, mesh.mask)

    def ax_local(self, h1, h2, u):
        return ax_local(self.E, self.N, self.G, self.wJ, h1, h2, u, D=self.D)

    def apply(self, h1, h2, u):
        """w = M QQ^T (h1 K_L + h2 B_L) M u (reading 6)."""
        u = _c(u, np.float64); w = np.zeros_like(u)
        lib().or_op_apply(self.E, self.N, _p(self.D), _p(self.G), _p(self.wJ), _p(self.mask),
                          self.gs.nruns, _p(self.gs.perm), _p(self.gs.offs), float(h1), float(h2),
                          _p(u), _p(w))
        return w

    def gs_apply(self, v):
        return self.gs.apply(v)

    def diag(self, h1, h2):
        """Assembled diagonal QQ^T diag(h1 K_L + h2 B_L)."""
        d = np.zeros(self.n)
        lib().or_diag_local(self.E, self.N, _p(self.D), _p(self.G), _p(self.wJ), float(h1), float(h2), _p(d))
        return self.gs.apply(d)

    def dinv(self, h1, h2):
        """Jacobi inverse diagonal M / d (0 on Dirichlet nodes)."""
        d = self.diag(h1, h2)
        out = np.zeros(self.n)
        keep = self.mask == 0
        out[keep] = 1.0 / d[keep]
        return out

    def dot(self, x, y):
        """Owner-copy inner product (reading 8)."""
        o = self.owner != 0
        s = 0.0
        for a, b in zip(np.asarray(x)[o], np.asarray(y)[o]):
            s += a * b
        return s

    def pcg(self, h1, h2, b, tol, maxit, dinv=None, dot_mode=0):
        """Jacobi-PCG; returns (x, iters, status, hist).
        Inner products are Dot2 sums (nek_oracle.c).  dot_mode (reading 17 yardsticks only): 1 = the
        same in descending index order, 2 = plain recursive summation."""
        if dinv is None:
            dinv = self.dinv(h1, h2)
        lib().or_set_dot_mode(int(dot_mode))
        b = _c(b, np.float64); x = np.zeros(self.n); hist = np.zeros(maxit + 1)
        it = ctypes.c_int(0)
        st = lib().or_pcg(self.E, self.N, _p(self.D), _p(self.G), _p(self.wJ), _p(self.mask),
                          self.gs.nruns, _p(self.gs.perm), _p(self.gs.offs), _p(self.owner),
                          _p(_c(dinv, np.float64)), float(h1), float(h2), _p(b), _p(x),
                          float(tol), int(maxit), ctypes.byref(it), _p(hist))
        lib().or_set_dot_mode(0)
        return x, it.value, st, hist[: it.value + 1]

    def reproducible_window(self, h1, h2, b, maxit, dinv=None):
        """Largest k <= maxit up to which this oracle reproduces its own residual history to a tenth
        of WINDOW_TOL (window_error) when only the rounding of its inner products changes (Dot2 vs
        plain recursive sums).  Beyond it CG's loss of orthogonality amplifies rounding differences
        exponentially (SURVEY 8(c) reading 17), so no two FP64 codes can be held to the bar there."""
        _, _, _, h = self.pcg(h1, h2, b, 0.0, maxit, dinv=dinv)
        _, _, _, hp = self.pcg(h1, h2, b, 0.0, maxit, dinv=dinv, dot_mode=2)
        k = min(h.size, hp.size)
        e = np.abs(h[:k] - hp[:k]) / np.maximum(1.0, np.abs(h[:k]))
        bad = np.nonzero(e > 0.1 * WINDOW_TOL)[0]
        return int(k - 1 if bad.size == 0 else max(bad[0] - 1, 0))

    def hist_tolerance(self, h1, h2, b, maxit, dinv=None):
        """Per-iteration tolerance on ||r_k||/||b|| for a CONVERGED solve of another FP64
        implementation (SURVEY 8(c) reading 17): max(1e-12, 10 * self-noise_k), the noise being
        this oracle against itself with its inner products summed the plain recursive way instead
        of by Dot2 (the rounding drift between two correct FP64 CG codes).  Fixed windows of
        <= 100 iterations use the flat WINDOW_TOL instead."""
        _, _, _, h = self.pcg(h1, h2, b, 0.0, maxit, dinv=dinv)
        _, _, _, hr = self.pcg(h1, h2, b, 0.0, maxit, dinv=dinv, dot_mode=2)
        k = min(h.size, hr.size)
        # the envelope (running maximum) of the drift: the divergence of two CG runs grows on average,
        # and a pointwise noise sample can dip where another realisation does not
        return np.maximum(WINDOW_TOL, 10.0 * np.maximum.accumulate(np.abs(h[:k] - hr[:k])))


# Fixed-window PCG parity bar (BASELINE north_star "CG residuals must agree to relative 1e-12";
# SURVEY 8(c) reading 17; reading 17): on windows of <= 100 iterations
#   |d ||r_k||| <= 1e-12 * max(||b||, ||r_k||)   at every k,
# i.e. 1e-12 relative to the residual itself, measured against ||b|| once the residual has dropped
# below it (so tiny late residuals do not blow the relative measure up).  No self-noise term.
WINDOW_TOL = 1e-12


def window_error(h_got, h_ref):
    """max_k |d h_k| / max(1, h_k) for ||b||-normalised histories h (the WINDOW_TOL measure)."""
    h_got, h_ref = np.asarray(h_got), np.asarray(h_ref)
    return float((np.abs(h_got - h_ref) / np.maximum(1.0, np.abs(h_ref))).max())


# ------------------------------------------------ multi-rank gather-scatter --
def gs_multi(gids, vals):
    """QQ^T across ranks (reading 7): each rank left-folds its copies of a gid
    in ascending l; the total is ((p_r0 + p_r1) + ...) over the ranks holding
    the gid in ascending rank order; every copy on every rank gets the total."""
    P = len(gids)
    maps = [GsMap(g, min_len=1) for g in gids]
    parts = [m.partial(v) for m, v in zip(maps, vals)]
    allg = np.unique(np.concatenate([m.rgid for m in maps]))
    total = np.zeros(allg.size)
    seen = np.zeros(allg.size, bool)
    for r in range(P):
        pos = np.searchsorted(allg, maps[r].rgid)
        t = total[pos]
        total[pos] = np.where(seen[pos], t + parts[r], parts[r])
        seen[pos] = True
    outs = []
    for r in range(P):
        v = np.array(vals[r], dtype=np.float64, copy=True)
        pos = np.searchsorted(allg, maps[r].rgid)
        m = maps[r]
        for ri in range(m.nruns):
            v[m.perm[m.offs[ri]:m.offs[ri + 1]]] = total[pos[ri]]
        outs.append(v)
    return outs
