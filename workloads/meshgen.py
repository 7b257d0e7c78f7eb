"""Seeded synthetic input generators (meshes, ids, masks, fields).

This module is shared by the tests, bench.py and smoke(). It holds NONE of the
method's arithmetic: no derivative matrix, no geometric factors, no operator,
no gather-scatter sum, no solver. It only places mesh nodes, numbers them, flags
boundary nodes and evaluates smooth analytic fields at node coordinates.

Conventions:
  E-vector local index  l = e*(N+1)^3 + i + (N+1)*j + (N+1)^2*k, i (r) fastest.
  xyz is (3, E*(N+1)^3) float64: the physical coordinates of every GLL node of
  every element (reading 1 of DESIGN.md: "vertex coordinates" = all GLL nodes,
  because the curved configs need high-order geometry).
  gid is int64, equal on all copies of a node, 0-based.
  mask is uint8, 1 = Dirichlet node.

Node placement: elements are images of [-1,1]^3 with nodes at the order-N
Gauss-Lobatto-Legendre points (Eq. 3). The generator places them with
numpy's Legendre root finder (companion-matrix roots of P_N', polished by Newton
steps through numpy.polynomial.legendre.legval) -- its own route, independent of
both the oracle's and the CUDA library's GLL code. Coordinates are computed ONCE
per global node and gathered to the local copies, so every copy of a node carries
bit-identical coordinates.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
from numpy.polynomial import legendre as _leg


def gll_points(N: int) -> np.ndarray:
    """Ascending GLL points for order N (ends -1, +1; interior = roots of P_N')."""
    if N < 1:
        raise ValueError("N >= 1")
    c = np.zeros(N + 1)
    c[N] = 1.0
    dc = _leg.legder(c)
    if N == 1:
        inner = np.zeros(0)
    else:
        inner = np.sort(np.real(_leg.legroots(dc)))
        d2c = _leg.legder(dc)
        for _ in range(3):  # Newton polish on P_N'
            inner = inner - _leg.legval(inner, dc) / _leg.legval(inner, d2c)
        inner = 0.5 * (inner - inner[::-1])  # exact symmetry
    x = np.concatenate([[-1.0], inner, [1.0]])
    return x


@dataclasses.dataclass
class Mesh:
    E: int
    N: int
    xyz: np.ndarray          # (3, E*Nq^3) float64
    gid: np.ndarray          # (E*Nq^3,) int64
    mask: np.ndarray         # (E*Nq^3,) uint8
    elem: np.ndarray         # (E, 3) int64 element lattice coords (ex, ey, ez)
    shape: tuple             # (Ex, Ey, Ez)
    extent: tuple            # (Lx, Ly, Lz)
    deform: str
    eps: float

    @property
    def Nq(self):
        return self.N + 1

    @property
    def n_local(self):
        return self.E * self.Nq ** 3

    @property
    def n_dof(self):
        """The paper's resolution count n = E*N^3."""
        return self.E * self.N ** 3

    def n_unique(self):
        return int(np.unique(self.gid).size)


def _deform_global(X, Y, Z, extent, deform, eps):
    Lx, Ly, Lz = extent
    xh, yh, zh = X / Lx, Y / Ly, Z / Lz
    if deform in ("none", "affine"):
        return X, Y, Z
    if deform == "bubble":
        # x' = x + eps*b(x)*(1,1,1), b = 64 x(1-x) y(1-y) z(1-z) on the unit box
        # (reading 12). Boundary fixed pointwise; degree 2 per direction.
        b = 64.0 * xh * (1.0 - xh) * yh * (1.0 - yh) * zh * (1.0 - zh)
        return X + eps * Lx * b, Y + eps * Ly * b, Z + eps * Lz * b
    if deform == "sin":
        b = np.sin(np.pi * xh) * np.sin(np.pi * yh) * np.sin(np.pi * zh)
        return X + eps * Lx * b, Y + eps * Ly * b, Z + eps * Lz * b
    if deform == "shear":
        # SPEC S:133 example: x -> x + eps*sin(pi*y)
        return X + eps * Lx * np.sin(np.pi * yh), Y, Z
    raise ValueError(f"unknown deform {deform!r}")


def box_mesh(Ex: int, Ey: int, Ez: int, N: int, deform: str = "bubble", eps: float = 0.05,
             extent=(1.0, 1.0, 1.0), dirichlet: str = "all", jitter: float = 0.0,
             seed: int = 0, zlayers=None) -> Mesh:
    """Structured Ex x Ey x Ez hex box of order N, lexicographic elements
    e = ex + Ex*(ey + Ey*ez), deformed by `deform`.

    dirichlet: "all" (every boundary face), "none", "top" (z = Lz plane only),
    "zends" (z = 0 and z = Lz planes).
    jitter > 0 moves interior element VERTICES randomly (trilinear elements,
    straight edges), used by the patch test; the GLL nodes then follow the
    trilinear map of each element (copies still bit-identical: each global node
    is placed once from one owning element).

    zlayers=(z0, z1) generates only the element layers z0 <= ez < z1 (one
    rank's z-slab) with the global numbering of the full box."""
    Nq = N + 1
    xi = gll_points(N)
    NX, NY, NZ = Ex * N + 1, Ey * N + 1, Ez * N + 1

    def lattice_1d(Ee, L):
        I = np.arange(Ee * N + 1)
        e = np.minimum(I // N, Ee - 1)
        i = I - e * N
        return L * (e + 0.5 * (xi[i] + 1.0)) / Ee

    Lx, Ly, Lz = extent
    if jitter == 0.0:
        gx, gy, gz = lattice_1d(Ex, Lx), lattice_1d(Ey, Ly), lattice_1d(Ez, Lz)
        X, Y, Z = np.meshgrid(gx, gy, gz, indexing="ij")  # (NX, NY, NZ)
    else:
        rng = np.random.default_rng(seed)
        vx = np.linspace(0, Lx, Ex + 1); vy = np.linspace(0, Ly, Ey + 1); vz = np.linspace(0, Lz, Ez + 1)
        VX, VY, VZ = np.meshgrid(vx, vy, vz, indexing="ij")
        V = np.stack([VX, VY, VZ])
        inner = np.zeros(VX.shape, bool)
        inner[1:-1, 1:-1, 1:-1] = True
        h = np.array([Lx / Ex, Ly / Ey, Lz / Ez])
        pert = rng.uniform(-1, 1, size=V.shape) * (jitter * h)[:, None, None, None]
        V = V + pert * inner[None]
        X = np.empty((NX, NY, NZ)); Y = np.empty_like(X); Z = np.empty_like(X)
        I = np.arange(NX); ex = np.minimum(I // N, Ex - 1); ii = I - ex * N
        J = np.arange(NY); ey = np.minimum(J // N, Ey - 1); jj = J - ey * N
        K = np.arange(NZ); ez = np.minimum(K // N, Ez - 1); kk = K - ez * N
        r = 0.5 * (xi[ii] + 1.0); s = 0.5 * (xi[jj] + 1.0); t = 0.5 * (xi[kk] + 1.0)
        R, S, T = np.meshgrid(r, s, t, indexing="ij")
        EX, EY, EZ = np.meshgrid(ex, ey, ez, indexing="ij")
        out = [np.zeros((NX, NY, NZ)) for _ in range(3)]
        for a in (0, 1):
            for b in (0, 1):
                for c in (0, 1):
                    wgt = (R if a else 1 - R) * (S if b else 1 - S) * (T if c else 1 - T)
                    for d in range(3):
                        out[d] += wgt * V[d][EX + a, EY + b, EZ + c]
        X, Y, Z = out
    X, Y, Z = _deform_global(X, Y, Z, extent, deform, eps)

    z0, z1 = (0, Ez) if zlayers is None else zlayers
    E = Ex * Ey * (z1 - z0)
    e = np.arange(E) + Ex * Ey * z0
    ex, ey, ez = e % Ex, (e // Ex) % Ey, e // (Ex * Ey)
    i = np.arange(Nq)
    # local (e, k, j, i) -> global lattice (I, J, K)
    Ig = (ex[:, None, None, None] * N + i[None, None, None, :])
    Jg = (ey[:, None, None, None] * N + i[None, None, :, None])
    Kg = (ez[:, None, None, None] * N + i[None, :, None, None])
    Ig, Jg, Kg = np.broadcast_arrays(Ig, Jg, Kg)
    Ig, Jg, Kg = Ig.reshape(-1), Jg.reshape(-1), Kg.reshape(-1)
    gid = (Ig + NX * (Jg + NY * Kg)).astype(np.int64)
    xyz = np.stack([X[Ig, Jg, Kg], Y[Ig, Jg, Kg], Z[Ig, Jg, Kg]]).astype(np.float64)

    if dirichlet == "all":
        m = (Ig == 0) | (Ig == NX - 1) | (Jg == 0) | (Jg == NY - 1) | (Kg == 0) | (Kg == NZ - 1)
    elif dirichlet == "none":
        m = np.zeros(gid.shape, bool)
    elif dirichlet == "top":
        m = Kg == NZ - 1
    elif dirichlet == "zends":
        m = (Kg == 0) | (Kg == NZ - 1)
    else:
        raise ValueError(dirichlet)
    return Mesh(E=E, N=N, xyz=np.ascontiguousarray(xyz), gid=gid, mask=m.astype(np.uint8),
                elem=np.stack([ex, ey, ez], 1), shape=(Ex, Ey, Ez), extent=tuple(extent),
                deform=deform, eps=eps)


def submesh(mesh: Mesh, elems: np.ndarray) -> Mesh:
    """The elements `elems` (in that order) of `mesh`, keeping global ids."""
    elems = np.asarray(elems, dtype=np.int64)
    P3 = mesh.Nq ** 3
    loc = (elems[:, None] * P3 + np.arange(P3)[None, :]).reshape(-1)
    return Mesh(E=int(elems.size), N=mesh.N, xyz=np.ascontiguousarray(mesh.xyz[:, loc]),
                gid=mesh.gid[loc].copy(), mask=mesh.mask[loc].copy(), elem=mesh.elem[elems].copy(),
                shape=mesh.shape, extent=mesh.extent, deform=mesh.deform, eps=mesh.eps)


def slab_partition(mesh: Mesh, P: int, axis: int = 2) -> list:
    """Contiguous lexicographic element slabs along `axis`."""
    n = mesh.shape[axis]
    if P > n:
        raise ValueError("more ranks than element layers")
    c = mesh.elem[:, axis]
    bounds = [(n * r) // P for r in range(P + 1)]
    return [np.nonzero((c >= bounds[r]) & (c < bounds[r + 1]))[0] for r in range(P)]


def block_partition(mesh: Mesh, px: int, py: int, pz: int) -> list:
    """px*py*pz element blocks (exercises edge and corner sharing)."""
    parts = []
    Ex, Ey, Ez = mesh.shape
    for rz in range(pz):
        for ry in range(py):
            for rx in range(px):
                sel = ((mesh.elem[:, 0] * px // Ex == rx) & (mesh.elem[:, 1] * py // Ey == ry)
                       & (mesh.elem[:, 2] * pz // Ez == rz))
                parts.append(np.nonzero(sel)[0])
    return parts


def smooth_field(mesh: Mesh, seed: int = 0, modes: int = 6, masked: bool = True) -> np.ndarray:
    """A continuous random field: a seeded sum of sinusoids evaluated at node
    coordinates (copies of a node have identical coordinates, hence identical
    values). Zero on Dirichlet nodes when masked."""
    rng = np.random.default_rng(seed)
    x, y, z = mesh.xyz
    Lx, Ly, Lz = mesh.extent
    f = np.zeros(mesh.n_local)
    for _ in range(modes):
        k = rng.uniform(0.5, 3.0, size=3) * np.pi / np.array([Lx, Ly, Lz])
        ph = rng.uniform(0, 2 * np.pi, size=3)
        a = rng.standard_normal()
        f += a * np.sin(k[0] * x + ph[0]) * np.sin(k[1] * y + ph[1]) * np.cos(k[2] * z + ph[2])
    if masked:
        f[mesh.mask != 0] = 0.0
    return f


def random_evector(mesh: Mesh, seed: int = 0) -> np.ndarray:
    """Standard normals per local point (discontinuous across copies)."""
    return np.random.default_rng(seed).standard_normal(mesh.n_local)


def manufactured(mesh: Mesh):
    """u* = sin(pi x) sin(pi y) sin(pi z) and f = 3 pi^2 u* on the unit box
    (-lap u* = f; u* = 0 on the boundary). Returns (u*, f) as E-vectors."""
    x, y, z = mesh.xyz
    u = np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    return u, 3.0 * np.pi ** 2 * u


# ---------------------------------------------------------------- named configs
def config_mesh(cfg: int, **kw) -> Mesh:
    """BASELINE.json configs."""
    if cfg == 1:   # deformed 2x2x2 box, N=3, Dirichlet all faces
        return box_mesh(2, 2, 2, 3, deform="bubble", eps=0.05, dirichlet="all", **kw)
    if cfg == 2:   # BP5-style 16^3, N=7
        return box_mesh(16, 16, 16, 7, deform="bubble", eps=0.05, dirichlet="all", **kw)
    if cfg == 3:   # 32x64x64, N=7
        return box_mesh(32, 64, 64, 7, deform="bubble", eps=0.05, dirichlet="all", **kw)
    raise ValueError(cfg)


# ------------------------------------------------------------- rod bundle
def rod_bundle(npx: int = 17, npy: int = 17, nlayers: int = 3, N: int = 7, pitch: float = 1.26,
               radius: float = 0.475, ntheta: int = 4, nrad: int = 6, dz: float = None,
               dirichlet: str = "pins_walls", z0_layer: int = 0, nlayers_total: int = None) -> Mesh:
    """Rod-bundle-like curved hex mesh (BASELINE config 4, reading 13): npx x npy pin
    cells of side `pitch`, each an O-grid of 4 side blocks x (ntheta x nrad) elements between the
    pin circle of `radius` and the cell square, blended radially; extruded in z by `nlayers`
    element layers (layers z0_layer .. z0_layer+nlayers-1 of nlayers_total).  GLL nodes are placed
    through the analytic map (curved elements); node ids come from coordinate hashing and every
    copy of a node gets the coordinates of its first occurrence (bit-identical copies).

    dirichlet: "pins_walls" (pin surfaces, outer walls, inlet z = 0: velocity-shaped),
               "outlet" (top plane only: pressure-shaped), "none"."""
    if dz is None:
        dz = pitch
    if nlayers_total is None:
        nlayers_total = z0_layer + nlayers
    Nq = N + 1
    xi = gll_points(N)
    h = 0.5 * pitch
    dth = 0.5 * np.pi / ntheta
    R, S = np.meshgrid(xi, xi, indexing="xy")          # R[j, i] = xi_i, S[j, i] = xi_j
    # all cross-section elements at once, ordered (cy, cx, blk, c, a)
    cyv, cxv, bv, cv, av = np.meshgrid(np.arange(npy), np.arange(npx), np.arange(4), np.arange(nrad),
                                       np.arange(ntheta), indexing="ij")
    cyv, cxv, bv, cv, av = (v.reshape(-1, 1, 1) for v in (cyv, cxv, bv, cv, av))
    ox, oy = (cxv + 0.5) * pitch, (cyv + 0.5) * pitch
    th0 = -0.25 * np.pi + bv * 0.5 * np.pi
    # i (r) runs outward from the pin, j (s) counter-clockwise: right-handed with z
    th = th0 + (av + 0.5 * (S[None] + 1.0)) * dth
    srad = (cv + 0.5 * (R[None] + 1.0)) / nrad
    cth, sth = np.cos(th), np.sin(th)
    mm = np.maximum(np.abs(cth), np.abs(sth))
    PX = ox + (1.0 - srad) * radius * cth + srad * h * cth / mm
    PY = oy + (1.0 - srad) * radius * sth + srad * h * sth / mm
    els_xyz = [(PX[e], PY[e]) for e in range(PX.shape[0])]
    nE2 = len(els_xyz)
    E = nE2 * nlayers
    P3 = Nq ** 3
    # cross-section ids by coordinate hashing (tolerance far below the node spacing, far above
    # rounding); every rank builds the same cross-section, so the ids agree across ranks
    pts2 = np.stack([PX.reshape(PX.shape[0], -1), PY.reshape(PY.shape[0], -1)], 1)   # (nE2, 2, Nq^2)
    flat = pts2.transpose(1, 0, 2).reshape(2, -1)
    tol = 1e-7 * pitch
    key = np.round(flat / tol).astype(np.int64)
    _, first, inv = np.unique(key.T, axis=0, return_index=True, return_inverse=True)
    inv = inv.reshape(-1)
    flat = flat[:, first[inv]]                                              # bit-identical copies
    xy_id = inv.reshape(nE2, Nq * Nq)
    pts2 = flat.reshape(2, nE2, Nq * Nq)
    NZ = nlayers_total * N + 1
    xyz = np.empty((3, E * P3))
    gid = np.empty(E * P3, np.int64)
    zt = 0.5 * (xi + 1.0)
    for L in range(nlayers):
        Lg = z0_layer + L
        zl = (Lg + zt) * dz
        sl = slice(L * nE2 * P3, (L + 1) * nE2 * P3)
        xyz[0, sl] = np.broadcast_to(pts2[0][:, None, :], (nE2, Nq, Nq * Nq)).reshape(-1)
        xyz[1, sl] = np.broadcast_to(pts2[1][:, None, :], (nE2, Nq, Nq * Nq)).reshape(-1)
        xyz[2, sl] = np.broadcast_to(zl[None, :, None], (nE2, Nq, Nq * Nq)).reshape(-1)
        K = Lg * N + np.arange(Nq)
        gid[sl] = (xy_id[:, None, :].astype(np.int64) * NZ + K[None, :, None]).reshape(-1)
    x, y, zz = xyz
    ccx = np.clip(np.floor(x / pitch), 0, npx - 1)
    ccy = np.clip(np.floor(y / pitch), 0, npy - 1)
    on_pin = np.abs(np.hypot(x - (ccx + 0.5) * pitch, y - (ccy + 0.5) * pitch) - radius) < 1e-9
    walls = (np.abs(x) < 1e-9) | (np.abs(x - npx * pitch) < 1e-9) | (np.abs(y) < 1e-9) | \
        (np.abs(y - npy * pitch) < 1e-9)
    inlet = np.abs(zz) < 1e-9
    outlet = np.abs(zz - nlayers_total * dz) < 1e-9
    if dirichlet == "pins_walls":
        mask = on_pin | walls | inlet
    elif dirichlet == "outlet":
        mask = outlet
    elif dirichlet == "none":
        mask = np.zeros(E * P3, bool)
    else:
        raise ValueError(dirichlet)
    elem = np.zeros((E, 3), np.int64)
    elem[:, 2] = np.repeat(np.arange(nlayers) + z0_layer, nE2)
    Lx, Ly, Lz = npx * pitch, npy * pitch, nlayers_total * dz
    return Mesh(E=E, N=N, xyz=xyz, gid=gid, mask=mask.astype(np.uint8), elem=elem, shape=(npx, npy, nlayers_total),
                extent=(Lx, Ly, Lz), deform="rod", eps=0.0)
