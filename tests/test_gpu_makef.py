"""GPU parity of the dealiased advection makef (NEXT #4) against the oracle (oracle/makef.py).

Both sides are FP64 on the same 3/2-rule lattice; they differ only in summation order and in how
the Gauss-Legendre nodes and interpolation weights are computed (Newton + barycentric here, numpy's
eigenvalue leggauss + product formula in the oracle), so outputs agree to 1e-12 normwise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.makef import Makef as OMakef  # noqa: E402
from workloads import meshgen as mg  # noqa: E402


@pytest.fixture(scope="module")
def nek():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_19119_b200 import nek as _nek
    return _nek


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def velocity(m, seed):
    return [mg.smooth_field(m, seed=seed + c) for c in range(3)]


@pytest.mark.parametrize("name,mk", [
    ("N7_bubble", lambda: mg.box_mesh(3, 2, 3, 7, deform="bubble")),
    ("N3_sin", lambda: mg.box_mesh(4, 3, 2, 3, deform="sin", eps=0.08)),
    ("N5_jitter", lambda: mg.box_mesh(3, 3, 2, 5, deform="affine", jitter=0.1, seed=4)),
    ("N1", lambda: mg.box_mesh(3, 2, 2, 1, deform="bubble")),
    ("N9", lambda: mg.box_mesh(2, 2, 2, 9, deform="bubble")),
    ("N8_rod", lambda: mg.rod_bundle(2, 2, 1, 8, dirichlet="none")),
])
def test_makef_parity(nek, name, mk):
    m = mk()
    U = velocity(m, 11)
    want = OMakef(m.E, m.N, m.xyz).apply(*U)
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, device=0)
    try:
        K = nek.Makef(ctx, m.xyz)
        assert K.M == (3 * (m.N + 1) + 1) // 2
        F = [np.empty(m.n_local) for _ in range(3)]
        K.apply(*U, *F)
        assert max(rel(a, b) for a, b in zip(F, want)) <= 1e-12
        Ud = [torch.from_numpy(c).cuda() for c in U]
        Fd = [torch.empty_like(Ud[0]) for _ in range(3)]
        K.apply(*Ud, *Fd)
        assert all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(Fd, F))
        Z = [np.zeros(m.n_local) for _ in range(3)]
        K.apply(*Z, *F)
        assert all(np.all(f == 0.0) for f in F)
        K.free()
    finally:
        nek.free(ctx)


def test_makef_full_size_linear_velocity_and_samples(nek):
    """Config 2 size (16^3 elements, N = 7): on an affine map a linear velocity gives the closed form
    F = -w_l J (B c + B^2 x_l) at every node (property at any size), and on the curved bubble mesh
    sampled elements equal the oracle run on just those elements."""
    m = mg.box_mesh(16, 16, 16, 7, deform="affine")
    A = np.array([[1.1, 0.2, 0.0], [-0.1, 0.95, 0.15], [0.05, -0.2, 1.05]])
    m.xyz = A @ m.xyz
    c = np.array([0.3, -0.2, 0.5])
    B = np.array([[0.2, -0.4, 0.1], [0.5, 0.05, -0.3], [-0.1, 0.25, 0.12]])
    U = list(c[:, None] + B @ m.xyz)
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, device=0)
    try:
        K = nek.Makef(ctx, m.xyz)
        F = [np.empty(m.n_local) for _ in range(3)]
        K.apply(*U, *F)
        # w_l J in closed form: GLL weights w_i = 2 / (N (N+1) P_N(xi_i)^2) at the nodes, J = det(A) (h/2)^3
        # of the affine map (element size h = 1/16), independent of the library's geometry
        from numpy.polynomial import legendre as npleg
        xi = mg.gll_points(m.N)
        PN = npleg.legval(xi, [0] * m.N + [1])
        w1 = 2.0 / (m.N * (m.N + 1) * PN ** 2)
        wq = (w1[None, None, :] * w1[None, :, None] * w1[:, None, None]).reshape(-1)    # (k, j, i)
        wJ = np.tile(wq, m.E) * np.linalg.det(A) * (0.5 / 16) ** 3
        adv = (B @ c)[:, None] + B @ (B @ m.xyz)
        for d in range(3):
            want = -wJ * adv[d]
            assert rel(F[d], want) <= 1e-12
        K.free()
    finally:
        nek.free(ctx)
    m = mg.config_mesh(2)
    U = velocity(m, 21)
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, device=0)
    try:
        K = nek.Makef(ctx, m.xyz)
        F = [np.empty(m.n_local) for _ in range(3)]
        K.apply(*U, *F)
        K.free()
    finally:
        nek.free(ctx)
    P3 = 512
    els = np.array([0, 1, 777, 2048, 4095])
    sub = mg.submesh(m, els)
    loc = (els[:, None] * P3 + np.arange(P3)).reshape(-1)
    want = OMakef(sub.E, sub.N, sub.xyz).apply(*[u[loc] for u in U])
    assert max(rel(f[loc], w) for f, w in zip(F, want)) <= 1e-12


def test_makef_errors(nek):
    from paper_2409_19119_b200.nek import NekError
    m = mg.box_mesh(2, 1, 1, 5)
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, device=0)
    try:
        with pytest.raises(NekError) as ei:
            nek.Makef(ctx, m.xyz, M=7)
        assert ei.value.code == -1
    finally:
        nek.free(ctx)
    m = mg.box_mesh(1, 1, 1, 12)
    ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, device=0)
    try:
        with pytest.raises(NekError) as ei:
            nek.Makef(ctx, m.xyz)
        assert ei.value.code == -2
    finally:
        nek.free(ctx)
