"""Thin ctypes binding of the C ABI in include/nek.h (argument marshalling only).

Every numerical step runs inside libnek.so (CUDA kernels for sm_100a + NCCL).
There is no CPU fallback: if the library is missing or fails to load, importing
this module raises.

Field arguments accept either torch CUDA float64 tensors (device pointers, used
in stream order on torch's current stream) or numpy float64 arrays (host
pointers; the library stages them through device memory and synchronises).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# NEK_LIB_VARIANT=checked loads the build with the device invariant checks (build.py --checked)
LIB_PATH = os.path.join(_PKG, "libnek_checked.so" if os.environ.get("NEK_LIB_VARIANT") == "checked" else "libnek.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(no CPU fallback exists)")
_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

OK, MAXIT, EINVAL, EORDER, EGEOM, ETOPO, ENOTSPD, ENOMEM, ECUDA, ENCCL, ENODEV = 0, 1, -1, -2, -3, -4, -5, -6, -7, -8, -9
_NAMES = {0: "NEK_OK", 1: "NEK_MAXIT", -1: "NEK_EINVAL", -2: "NEK_EORDER", -3: "NEK_EGEOM", -4: "NEK_ETOPO",
          -5: "NEK_ENOTSPD", -6: "NEK_ENOMEM", -7: "NEK_ECUDA", -8: "NEK_ENCCL", -9: "NEK_ENODEV"}

(PLAN_PERM, PLAN_OFFS, PLAN_IFC_PERM, PLAN_IFC_OFFS, PLAN_IFC_GID, PLAN_NEIGHBORS, PLAN_SEND_OFFS, PLAN_SEND_RUN,
 PLAN_CONTRIB_OFFS, PLAN_CONTRIB, PLAN_OWNER, PLAN_ELEM_ORDER) = range(12)
_PLAN_DTYPES = {PLAN_PERM: np.int32, PLAN_OFFS: np.int64, PLAN_IFC_PERM: np.int32, PLAN_IFC_OFFS: np.int64,
                PLAN_IFC_GID: np.int64, PLAN_NEIGHBORS: np.int32, PLAN_SEND_OFFS: np.int64, PLAN_SEND_RUN: np.int32,
                PLAN_CONTRIB_OFFS: np.int64, PLAN_CONTRIB: np.int32, PLAN_OWNER: np.uint8,
                PLAN_ELEM_ORDER: np.int32}


class NekError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class nek_comm(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nccl_id", ctypes.c_ubyte * 128)]


class nek_info_t(ctypes.Structure):
    _fields_ = [("E", ctypes.c_int64), ("N", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("n_local", ctypes.c_int64), ("n_dof", ctypes.c_int64), ("n_masked", ctypes.c_int64),
                ("n_runs", ctypes.c_int64), ("n_perm", ctypes.c_int64), ("n_ifc_runs", ctypes.c_int64),
                ("n_ifc_perm", ctypes.c_int64), ("n_neighbors", ctypes.c_int64), ("halo_doubles", ctypes.c_int64),
                ("n_boundary_elems", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("geom_min_jac", ctypes.c_double), ("transport", ctypes.c_int32), ("l2_keep", ctypes.c_int32),
                ("l2_setaside", ctypes.c_int64), ("l2_setaside_max", ctypes.c_int64)]


class nek_stats_t(ctypes.Structure):
    _fields_ = [("ax_ms", ctypes.c_double), ("gs_ms", ctypes.c_double), ("halo_ms", ctypes.c_double),
                ("vec_ms", ctypes.c_double), ("ax_launches", ctypes.c_int64), ("gs_launches", ctypes.c_int64),
                ("halo_launches", ctypes.c_int64), ("vec_launches", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("ax_elements", ctypes.c_int64), ("ax_bytes", ctypes.c_double), ("axu_ms", ctypes.c_double),
                ("axu_spans", ctypes.c_int64)]


PMG_MAX_LEVELS = 8


class nek_pmg_opts(ctypes.Structure):
    _fields_ = [("nlevels", ctypes.c_int32), ("orders", ctypes.c_int32 * PMG_MAX_LEVELS),
                ("degree", ctypes.c_int32), ("coarse_degree", ctypes.c_int32), ("lanczos_steps", ctypes.c_int32),
                ("lmin_frac", ctypes.c_double), ("lmax_factor", ctypes.c_double), ("coarse_lo", ctypes.c_double),
                ("precision", ctypes.c_int32)]


class nek_pmg_info_t(ctypes.Structure):
    _fields_ = [("nlevels", ctypes.c_int32), ("orders", ctypes.c_int32 * PMG_MAX_LEVELS),
                ("degree", ctypes.c_int32), ("coarse_degree", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("n_local", ctypes.c_int64 * PMG_MAX_LEVELS), ("lam_min", ctypes.c_double * PMG_MAX_LEVELS),
                ("lam_max", ctypes.c_double * PMG_MAX_LEVELS), ("vcycles", ctypes.c_int64)]


_P, _I, _I64, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
_sig = {
    "nek_version": ([], _I),
    "nek_loopback_create": ([_I, _I, ctypes.POINTER(_P)], _I),
    "nek_loopback_comm": ([_P, _I, ctypes.POINTER(nek_comm)], _I),
    "nek_loopback_abort": ([_P], _I),
    "nek_loopback_free": ([_P], _I),
    "nek_last_error": ([], ctypes.c_char_p),
    "nek_comm_unique_id": ([_P], _I),
    "nek_setup": ([ctypes.POINTER(_P), _I64, _I, _P, _P, _P, ctypes.POINTER(nek_comm), _I, _P], _I),
    "nek_ax": ([_P, _D, _D, _P, _P, _P], _I),
    "nek_gs": ([_P, _P, _P], _I),
    "nek_pcg_solve": ([_P, _D, _D, _P, _P, _D, _I, ctypes.POINTER(_I), ctypes.POINTER(_D), _P, _P], _I),
    "nek_free": ([_P], _I),
    "nek_errmsg": ([_P], ctypes.c_char_p),
    "nek_get_info": ([_P, ctypes.POINTER(nek_info_t)], _I),
    "nek_get_gs_map": ([_P, _P, _P], _I),
    "nek_get_geom": ([_P, _P, _P], _I),
    "nek_get_dinv": ([_P, _D, _D, _P, _P], _I),
    "nek_set_timing": ([_P, _I], _I),
    "nek_get_stats": ([_P, ctypes.POINTER(nek_stats_t), _I], _I),
    "nek_set_variant": ([_P, _I], _I),
    "nek_proj_create": ([_P, _I, ctypes.POINTER(_P)], _I),
    "nek_proj_solve": ([_P, _D, _D, _P, _P, _D, _I, ctypes.POINTER(_I), ctypes.POINTER(_D), _P], _I),
    "nek_proj_size": ([_P], _I),
    "nek_proj_reset": ([_P], _I),
    "nek_proj_free": ([_P], _I),
    "nek_pmg_create": ([_P, _P, _D, _D, ctypes.POINTER(nek_pmg_opts), ctypes.POINTER(_P), _P], _I),
    "nek_pmg_apply": ([_P, _P, _P, _P], _I),
    "nek_pmg_solve": ([_P, _P, _P, _D, _I, ctypes.POINTER(_I), ctypes.POINTER(_D), _P, _P], _I),
    "nek_pmg_info": ([_P, ctypes.POINTER(nek_pmg_info_t)], _I),
    "nek_pmg_free": ([_P], _I),
    "nek_makef_create": ([_P, _P, _I, ctypes.POINTER(_P), _P], _I),
    "nek_makef_apply": ([_P, _P, _P, _P, _P, _P, _P, _P], _I),
    "nek_makef_lattice": ([_P], _I),
    "nek_makef_free": ([_P], _I),
    "nek_probe_dfma_tflops": ([_I, ctypes.POINTER(_D)], _I),
    "nek_probe_hbm_gbps": ([_I, _I64, ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_D)], _I),
    "nek_probe_smem_tbps": ([_I, ctypes.POINTER(_D)], _I),
    "nek_plan_create": ([ctypes.POINTER(_P), _I64, _I, _P, _P, _P], _I),
    "nek_plan_surface_gids": ([_P, _P], _I64),
    "nek_plan_set_ranks": ([_P, _I, _I, _P, _P], _I),
    "nek_plan_size": ([_P, _I], _I64),
    "nek_plan_get": ([_P, _I, _P], _I),
    "nek_plan_errmsg": ([_P], ctypes.c_char_p),
    "nek_plan_free": ([_P], None),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_sig)


def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _field_ptr(a, n, name, writable=False, device=None):
    """(pointer, stream) of a float64 field of length n; a CUDA tensor must live on `device`."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or a.size != n or not a.flags.c_contiguous or (writable and not a.flags.writeable):
            raise ValueError(f"{name}: need a C-contiguous float64 array of {n} entries")
        return ctypes.c_void_p(a.ctypes.data), None
    import torch
    if not isinstance(a, torch.Tensor):
        raise TypeError(f"{name}: numpy array or torch tensor expected")
    if a.dtype != torch.float64 or a.numel() != n or not a.is_contiguous():
        raise ValueError(f"{name}: need a contiguous float64 tensor of {n} entries")
    if a.is_cuda:
        if device is not None and a.device.index != device:
            raise ValueError(f"{name}: tensor on cuda:{a.device.index}, context on cuda:{device}")
        return ctypes.c_void_p(a.data_ptr()), torch.cuda.current_stream(a.device).cuda_stream
    return ctypes.c_void_p(a.data_ptr()), None   # host (possibly pinned) tensor


def _stream_of(*streams):
    for s in streams:
        if s is not None:
            return ctypes.c_void_p(s)
    return None


def _check(code, ctx=None):
    if code < 0:
        msg = _lib.nek_errmsg(ctx) if ctx else _lib.nek_last_error()
        raise NekError(code, (msg or b"").decode())
    return code


def version():
    return _lib.nek_version()


def comm_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(_lib.nek_comm_unique_id(buf))
    return bytes(buf)


def comm_from_torch(device=None):
    """A fresh (rank, nranks, nccl_id) triple for nek_setup: rank 0 creates a
    new NCCL unique id, torch.distributed broadcasts it.  Every nek_setup needs
    its own id (an id bootstraps exactly one communicator)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return None
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    t = torch.zeros(128, dtype=torch.uint8, device=dev if dist.get_backend() == "nccl" else "cpu")
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return (rank, world, bytes(t.cpu().numpy().tobytes()))


class Loopback:
    """nek_loopback_*: P virtual ranks in one process on one GPU (include/nek.h).  Drive each rank
    from its own thread with comm=lb.comm(rank); transport 0 = peer-memory (NVLink-path) kernels,
    1 = NCCL-path kernels around staged copies."""

    def __init__(self, nranks, transport=0):
        h = ctypes.c_void_p()
        _check(_lib.nek_loopback_create(int(nranks), int(transport), ctypes.byref(h)))
        self._h = h
        self.nranks = int(nranks)

    def comm(self, rank) -> "nek_comm":
        c = nek_comm()
        _check(_lib.nek_loopback_comm(self._h, int(rank), ctypes.byref(c)))
        return c

    def abort(self):
        if self._h:
            _lib.nek_loopback_abort(self._h)

    def free(self):
        if self._h:
            _lib.nek_loopback_free(self._h)
            self._h = None


class Context:
    """A nek_ctx: one rank's elements, on one GPU."""

    def __init__(self, handle, E, N, device=0):
        self._h = handle
        self.E, self.N = E, N
        self.device = device
        self.n = E * (N + 1) ** 3

    @property
    def handle(self):
        if not self._h:
            raise RuntimeError("context freed")
        return self._h

    def free(self):
        if self._h:
            _lib.nek_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def setup(E, N, xyz, gid, mask=None, comm=None, device=0, stream=None) -> Context:
    """nek_setup: xyz (3, E*(N+1)^3) float64, gid int64, mask uint8 or None (host arrays).
    comm: None or (rank, nranks, nccl_id bytes)."""
    n = int(E) * (int(N) + 1) ** 3
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    gid = np.ascontiguousarray(gid, dtype=np.int64)
    if xyz.size != 3 * n or gid.size != n:
        raise ValueError("xyz must hold 3*E*(N+1)^3 and gid E*(N+1)^3 entries")
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    c = None
    if isinstance(comm, nek_comm):
        c = comm if comm.nranks > 1 else None
    elif comm is not None and comm[1] > 1:
        c = nek_comm()
        c.rank, c.nranks = int(comm[0]), int(comm[1])
        ctypes.memmove(c.nccl_id, bytes(comm[2]), 128)
    h = ctypes.c_void_p()
    st = _lib.nek_setup(ctypes.byref(h), int(E), int(N), _np_ptr(xyz), _np_ptr(gid), _np_ptr(m),
                        ctypes.byref(c) if c is not None else None, int(device),
                        ctypes.c_void_p(stream) if stream else None)
    _check(st)
    return Context(h, int(E), int(N), int(device))


def ax(ctx: Context, h1, h2, u, w):
    """nek_ax: w = M QQ^T (h1 K_L + h2 B_L) M u."""
    pu, su = _field_ptr(u, ctx.n, "u", device=ctx.device)
    pw, sw = _field_ptr(w, ctx.n, "w", writable=True, device=ctx.device)
    _check(_lib.nek_ax(ctx.handle, float(h1), float(h2), pu, pw, _stream_of(su, sw)), ctx.handle)
    return w


def gs(ctx: Context, v):
    """nek_gs: v <- QQ^T v in place."""
    pv, sv = _field_ptr(v, ctx.n, "v", writable=True, device=ctx.device)
    _check(_lib.nek_gs(ctx.handle, pv, _stream_of(sv)), ctx.handle)
    return v


def pcg_solve(ctx: Context, h1, h2, b, x, tol, maxit, want_hist=False):
    """nek_pcg_solve -> (status, iters, relres, hist or None)."""
    pb, sb = _field_ptr(b, ctx.n, "b", device=ctx.device)
    px, sx = _field_ptr(x, ctx.n, "x", writable=True, device=ctx.device)
    it = ctypes.c_int(0)
    rr = ctypes.c_double(0.0)
    hist = np.zeros(int(maxit) + 1) if want_hist else None
    st = _lib.nek_pcg_solve(ctx.handle, float(h1), float(h2), pb, px, float(tol), int(maxit), ctypes.byref(it),
                            ctypes.byref(rr), _np_ptr(hist), _stream_of(sb, sx))
    _check(st, ctx.handle)
    if hist is not None:
        hist = hist[: it.value + 1]
    return st, it.value, rr.value, hist


def free(ctx: Context):
    ctx.free()


def get_info(ctx: Context) -> dict:
    info = nek_info_t()
    _check(_lib.nek_get_info(ctx.handle, ctypes.byref(info)), ctx.handle)
    return {k: getattr(info, k) for k, _ in nek_info_t._fields_}


def get_gs_map(ctx: Context):
    info = get_info(ctx)
    perm = np.zeros(max(info["n_perm"], 1), np.int32)
    offs = np.zeros(info["n_runs"] + 1, np.int64)
    _check(_lib.nek_get_gs_map(ctx.handle, _np_ptr(perm), _np_ptr(offs)), ctx.handle)
    return perm[: info["n_perm"]], offs


def get_geom(ctx: Context):
    P3 = (ctx.N + 1) ** 3
    G = np.zeros((ctx.E, 6, P3))
    wJ = np.zeros(ctx.n)
    _check(_lib.nek_get_geom(ctx.handle, _np_ptr(G), _np_ptr(wJ)), ctx.handle)
    return G, wJ


def get_dinv(ctx: Context, h1, h2, out=None):
    if out is None:
        out = np.zeros(ctx.n)
    p, s = _field_ptr(out, ctx.n, "dinv", writable=True, device=ctx.device)
    _check(_lib.nek_get_dinv(ctx.handle, float(h1), float(h2), p, _stream_of(s)), ctx.handle)
    return out


def set_timing(ctx: Context, on: bool):
    _check(_lib.nek_set_timing(ctx.handle, 1 if on else 0), ctx.handle)


def get_stats(ctx: Context, reset=False) -> dict:
    s = nek_stats_t()
    _check(_lib.nek_get_stats(ctx.handle, ctypes.byref(s), 1 if reset else 0), ctx.handle)
    return {k: getattr(s, k) for k, _ in nek_stats_t._fields_}


def set_variant(ctx: Context, v: int):
    _check(_lib.nek_set_variant(ctx.handle, int(v)), ctx.handle)


class Projection:
    """nek_proj_*: projection of the initial guess onto up to max_vectors prior solutions
    (Fischer)."""

    def __init__(self, ctx: Context, max_vectors: int):
        self.ctx = ctx
        h = ctypes.c_void_p()
        _check(_lib.nek_proj_create(ctx.handle, int(max_vectors), ctypes.byref(h)), ctx.handle)
        self._h = h

    def solve(self, h1, h2, b, x, tol, maxit):
        """-> (status, iters, relres)"""
        pb, sb = _field_ptr(b, self.ctx.n, "b", device=self.ctx.device)
        px, sx = _field_ptr(x, self.ctx.n, "x", writable=True, device=self.ctx.device)
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        st = _lib.nek_proj_solve(self._h, float(h1), float(h2), pb, px, float(tol), int(maxit), ctypes.byref(it),
                                 ctypes.byref(rr), _stream_of(sb, sx))
        _check(st, self.ctx.handle)
        return st, it.value, rr.value

    def size(self):
        return _lib.nek_proj_size(self._h)

    def reset(self):
        _lib.nek_proj_reset(self._h)

    def free(self):
        if self._h:
            _lib.nek_proj_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PMG:
    """nek_pmg_*: p-multigrid V-cycle with Chebyshev smoothing as the PCG preconditioner
    (P:195-198).  xyz: the (3, E*(N+1)^3) coordinates given to setup.  Options (0 =
    default): orders (schedule list), degree, coarse_degree, lanczos_steps, lmin_frac, lmax_factor,
    coarse_lo."""

    def __init__(self, ctx: Context, xyz, h1, h2, orders=None, degree=0, coarse_degree=0, lanczos_steps=0,
                 lmin_frac=0.0, lmax_factor=0.0, coarse_lo=0.0, precision=0):
        self.ctx = ctx
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        if xyz.size != 3 * ctx.n:
            raise ValueError("xyz must hold 3*E*(N+1)^3 entries")
        o = nek_pmg_opts()
        if orders:
            o.nlevels = len(orders)
            for i, v in enumerate(orders):
                o.orders[i] = int(v)
        o.degree, o.coarse_degree, o.lanczos_steps = int(degree), int(coarse_degree), int(lanczos_steps)
        o.lmin_frac, o.lmax_factor, o.coarse_lo = float(lmin_frac), float(lmax_factor), float(coarse_lo)
        o.precision = int(precision)
        h = ctypes.c_void_p()
        _check(_lib.nek_pmg_create(ctx.handle, _np_ptr(xyz), float(h1), float(h2), ctypes.byref(o),
                                   ctypes.byref(h), None), ctx.handle)
        self._h = h

    def apply(self, r, z):
        """z = V(r)."""
        pr, sr = _field_ptr(r, self.ctx.n, "r", device=self.ctx.device)
        pz, sz = _field_ptr(z, self.ctx.n, "z", writable=True, device=self.ctx.device)
        _check(_lib.nek_pmg_apply(self._h, pr, pz, _stream_of(sr, sz)), self.ctx.handle)
        return z

    def solve(self, b, x, tol, maxit, want_hist=False):
        """-> (status, iters, relres, hist or None)"""
        pb, sb = _field_ptr(b, self.ctx.n, "b", device=self.ctx.device)
        px, sx = _field_ptr(x, self.ctx.n, "x", writable=True, device=self.ctx.device)
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        hist = np.zeros(int(maxit) + 1) if want_hist else None
        st = _lib.nek_pmg_solve(self._h, pb, px, float(tol), int(maxit), ctypes.byref(it), ctypes.byref(rr),
                                _np_ptr(hist), _stream_of(sb, sx))
        _check(st, self.ctx.handle)
        if hist is not None:
            hist = hist[: it.value + 1]
        return st, it.value, rr.value, hist

    def info(self) -> dict:
        i = nek_pmg_info_t()
        _check(_lib.nek_pmg_info(self._h, ctypes.byref(i)))
        L = i.nlevels
        return {"nlevels": L, "orders": list(i.orders[:L]), "degree": i.degree, "coarse_degree": i.coarse_degree,
                "precision": i.precision,
                "n_local": list(i.n_local[:L]), "lam_min": list(i.lam_min[:L]), "lam_max": list(i.lam_max[:L]),
                "vcycles": i.vcycles}

    def free(self):
        if self._h:
            _lib.nek_pmg_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def probe_fp64_tflops(device=0) -> float:
    """nek_probe_dfma_tflops: measured FP64 FMA throughput (TFLOP/s)."""
    v = ctypes.c_double(0.0)
    _check(_lib.nek_probe_dfma_tflops(int(device), ctypes.byref(v)))
    return v.value


def probe_hbm_gbps(device=0, nbytes=4 << 30) -> dict:
    """nek_probe_hbm_gbps: FP64 (double2) streaming read / write / copy bandwidth over `nbytes`."""
    r, w, c = ctypes.c_double(0.0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(_lib.nek_probe_hbm_gbps(int(device), int(nbytes), ctypes.byref(r), ctypes.byref(w), ctypes.byref(c)))
    return {"read": r.value, "write": w.value, "copy": c.value}


def probe_smem_tbps(device=0) -> float:
    """nek_probe_smem_tbps: aggregate ld.shared.f64 bandwidth (TB/s)."""
    v = ctypes.c_double(0.0)
    _check(_lib.nek_probe_smem_tbps(int(device), ctypes.byref(v)))
    return v.value


class Makef:
    """nek_makef_*: dealiased advection F_c = -(phi_l, u . grad u_c) on the 3/2-rule Gauss-Legendre
    lattice.  xyz: the (3, E*(N+1)^3) coordinates given to setup."""

    def __init__(self, ctx: Context, xyz, M=0):
        self.ctx = ctx
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        if xyz.size != 3 * ctx.n:
            raise ValueError("xyz must hold 3*E*(N+1)^3 entries")
        h = ctypes.c_void_p()
        _check(_lib.nek_makef_create(ctx.handle, _np_ptr(xyz), int(M), ctypes.byref(h), None), ctx.handle)
        self._h = h
        self.M = _lib.nek_makef_lattice(h)

    def apply(self, u, v, w, fu, fv, fw):
        ps, ss = [], []
        for a, name, wr in ((u, "u", False), (v, "v", False), (w, "w", False), (fu, "fu", True), (fv, "fv", True),
                            (fw, "fw", True)):
            p_, s_ = _field_ptr(a, self.ctx.n, name, writable=wr, device=self.ctx.device)
            ps.append(p_); ss.append(s_)
        _check(_lib.nek_makef_apply(self._h, *ps, _stream_of(*ss)), self.ctx.handle)
        return fu, fv, fw

    def free(self):
        if self._h:
            _lib.nek_makef_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# --------------------------------------------------------------- host plans
class Plan:
    """Host-only gather-scatter / halo plan (nek_plan_*), usable without a GPU."""

    def __init__(self, E, N, gid, mask=None, xyz=None):
        gid = np.ascontiguousarray(gid, dtype=np.int64)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        x = None if xyz is None else np.ascontiguousarray(xyz, dtype=np.float64)
        h = ctypes.c_void_p()
        st = _lib.nek_plan_create(ctypes.byref(h), int(E), int(N), _np_ptr(gid), _np_ptr(m), _np_ptr(x))
        self._h = h
        if st != OK:
            msg = _lib.nek_plan_errmsg(h).decode() if h else ""
            self.free()
            raise NekError(st, msg)

    def surface_gids(self):
        n = _lib.nek_plan_surface_gids(self._h, None)
        out = np.zeros(max(n, 1), np.int64)
        _lib.nek_plan_surface_gids(self._h, _np_ptr(out))
        return out[:n]

    def set_ranks(self, rank, nranks, lists):
        lists = [np.ascontiguousarray(L, dtype=np.int64) for L in lists]
        counts = np.array([L.size for L in lists], np.int64)
        ptrs = (ctypes.c_void_p * nranks)(*[L.ctypes.data for L in lists])
        st = _lib.nek_plan_set_ranks(self._h, int(rank), int(nranks), _np_ptr(counts), ptrs)
        if st != OK:
            raise NekError(st, _lib.nek_plan_errmsg(self._h).decode())

    def get(self, what):
        n = _lib.nek_plan_size(self._h, what)
        out = np.zeros(max(n, 1), _PLAN_DTYPES[what])
        if n > 0:
            _lib.nek_plan_get(self._h, what, _np_ptr(out))
        return out[:n]

    def free(self):
        if self._h:
            _lib.nek_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
