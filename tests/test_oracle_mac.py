"""Pins of the oracle's MAC discretisation against closed forms, invariants and
brute force (SURVEY.md §8(c) "What pins each part").  CPU only."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from synth.geometry import slit_2d, duct_3d, random_blobs, dumbbell_2d
from oracle.grid import build_grid
from oracle.mac import Mac
from oracle.decomposition import decompose, masked_faces
from oracle.newton import build_gplmm, newton, direct_solve, solve_steady

H, MU, RHO = 1e-5, 1e-3, 1000.0


def _x_faces(g, x):
    """x-face velocities on the full (nz, ny, nx+1) face array (0 on non-DOF)."""
    fd = g.face_dof[0]
    return np.where(fd >= 0, x[np.where(fd >= 0, fd, 0)], 0.0)


# --------------------------------------------------------------------------
# Closed forms
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13])
@pytest.mark.parametrize("inertia", [False, True])
def test_plane_poiseuille_slit(n, inertia):
    """Discrete plane Poiseuille (A3/A4/A6): u_j = G/(2mu)[y_j(W-y_j)+h^2/4],
    y_j=(j+1/2)h, W=nh, G=dp/((nx+1)h); flux Q = G h^3 (n^3+2n)/(12 mu).
    Convection vanishes (v = 0, du/dx = 0), so Navier-Stokes == Stokes."""
    nx, dp = 9, 3.0
    g = build_grid(slit_2d(nx, n), 2, (False, False), H)
    mac = Mac(g, RHO if inertia else 0.0, MU, p_in=dp, p_out=0.0)
    x = direct_solve(mac, tol=1e-13)
    G = dp / ((nx + 1) * H)
    y = (np.arange(n) + 0.5) * H
    uex = G / (2 * MU) * (y * (n * H - y) + H * H / 4)
    u = _x_faces(g, x)[0]
    assert np.allclose(u, uex[:, None], rtol=1e-12, atol=0)
    Q = u[:, 0].sum() * H
    assert Q == pytest.approx(G * H ** 3 * (n ** 3 + 2 * n) / (12 * MU), rel=1e-12)
    # pressure is linear between the ghost centres
    p = x[g.n_f:].reshape(n, nx)
    pex = dp - G * (np.arange(nx) + 1.0) * H
    assert np.allclose(p, pex[None, :], rtol=1e-11, atol=1e-12 * dp)


def _duct_exact(ny, nz, G):
    """Finite sine series on the cell-centred modes sin(k pi (j+1/2)/n) with
    eigenvalues (4/h^2) sin^2(k pi / 2n) (ghost value -u at the walls)."""
    def modes(n):
        j = np.arange(n)
        ks = np.arange(1, n + 1)
        phi = np.sin(np.outer(ks, j + 0.5) * np.pi / n)        # (k, j)
        lam = 4.0 / H ** 2 * np.sin(ks * np.pi / (2 * n)) ** 2
        nrm = np.where(ks == n, float(n), n / 2.0)
        a = phi.sum(axis=1) / nrm
        return phi, lam, a
    py, ly, ay = modes(ny)
    pz, lz, az = modes(nz)
    u = np.zeros((nz, ny))
    for k in range(ny):
        for l in range(nz):
            u += G * ay[k] * az[l] / (MU * (ly[k] + lz[l])) * np.outer(pz[l], py[k])
    return u


@pytest.mark.parametrize("ny,nz", [(3, 3), (4, 2), (5, 7), (1, 6)])
def test_rectangular_duct(ny, nz):
    nx, dp = 5, 2.0
    g = build_grid(duct_3d(nx, ny, nz), 3, (False, False), H)
    mac = Mac(g, RHO, MU, p_in=dp)
    x = direct_solve(mac, tol=1e-13)
    G = dp / ((nx + 1) * H)
    uex = _duct_exact(ny, nz, G)
    u = _x_faces(g, x)
    for i in range(nx + 1):
        assert np.allclose(u[:, :, i], uex, rtol=1e-11, atol=0)


def test_transient_slit_modes():
    """Backward Euler from rest (A7): each mode obeys
    (rho/dt + mu lam_k) u^{n+1} = (rho/dt) u^n + G a_k."""
    nx, n, dp, dt = 6, 5, 1.0, 2e-4
    g = build_grid(slit_2d(nx, n), 2, (False, False), H)
    mac = Mac(g, RHO, MU, p_in=dp, dt=dt)
    G = dp / ((nx + 1) * H)
    j = np.arange(n)
    ks = np.arange(1, n + 1)
    phi = np.sin(np.outer(ks, j + 0.5) * np.pi / n)
    lam = 4.0 / H ** 2 * np.sin(ks * np.pi / (2 * n)) ** 2
    nrm = np.where(ks == n, float(n), n / 2.0)
    a = phi.sum(axis=1) / nrm
    uh = np.zeros(n)
    x = np.zeros(g.N)
    for step in range(4):
        u_prev = x[:g.n_f].copy()
        x = direct_solve(mac, x, u_prev, tol=1e-13)
        uh = (RHO / dt * uh + G * a) / (RHO / dt + MU * lam)
        u = _x_faces(g, x)[0]
        assert np.allclose(u, (uh @ phi)[:, None], rtol=1e-10, atol=0)
    # the steady state is a fixed point
    xs = direct_solve(Mac(g, RHO, MU, p_in=dp), tol=1e-13)
    x2 = direct_solve(mac, xs, xs[:g.n_f], tol=1e-13)
    assert np.allclose(x2, xs, rtol=1e-11, atol=1e-14)


# --------------------------------------------------------------------------
# Invariants and identities
# --------------------------------------------------------------------------
def _blob_case(dim, periodic, seed=3):
    if dim == 2:
        img = random_blobs(20, 14, 1, 0.6, 2.5, seed)
    else:
        img = random_blobs(10, 9, 8, 0.6, 2.0, seed)
    return build_grid(img, dim, periodic, H)


@pytest.mark.parametrize("dim,periodic", [(2, (False, False)), (2, (True, False)),
                                          (3, (False, False)), (3, (True, True))])
def test_stokes_structure(dim, periodic):
    """F = F^T and Div = -Grad^T bitwise (A3), J(0) = J~_{w=0}."""
    g = _blob_case(dim, periodic)
    mac = Mac(g, RHO, MU, p_in=1.0, p_out=0.2)
    J0 = mac.jacobian(np.zeros(g.N)).tocsr()
    nf = g.n_f
    F = J0[:nf, :nf]
    assert (F - F.T).count_nonzero() == 0
    assert (J0[nf:, :nf] + J0[:nf, nf:].T).count_nonzero() == 0
    assert J0[nf:, nf:].count_nonzero() == 0
    Jt = mac.jacobian_modified(np.zeros(nf), np.zeros(nf, dtype=bool))
    assert (J0 - Jt).count_nonzero() == 0


@pytest.mark.parametrize("dim,periodic", [(2, (False, False)), (3, (True, True))])
def test_fd_jacobian(dim, periodic):
    """Central differences are exact for the quadratic residual when no upwind
    selector switches (A9): ||(r(x+ev)-r(x-ev))/2e - Jv|| small."""
    g = _blob_case(dim, periodic, seed=5)
    mac = Mac(g, RHO, MU, body_force=(3.0, 1.0, 0.5), p_in=1.0, dt=1e-3)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(g.N) * 0.05
    up = rng.standard_normal(g.n_f) * 0.05
    J = mac.jacobian(x)
    for _ in range(10):
        v = rng.standard_normal(g.N)
        e = 1e-7
        fd = (mac.residual(x + e * v, up) - mac.residual(x - e * v, up)) / (2 * e)
        jv = J @ v
        assert np.linalg.norm(fd - jv) <= 1e-6 * np.linalg.norm(jv)


def test_masked_rows_independent_of_wind():
    """J~_w rows of masked faces carry no inertia: independent of w;
    unmasked rows depend on it."""
    g = _blob_case(2, (False, False))
    mac = Mac(g, RHO, MU, p_in=1.0)
    rng = np.random.default_rng(1)
    mask = rng.random(g.n_f) < 0.5
    A1 = mac.jacobian_modified(rng.standard_normal(g.n_f), mask).tocsr()
    A2 = mac.jacobian_modified(rng.standard_normal(g.n_f), mask).tocsr()
    D = (A1 - A2).tocsr()
    rows = np.nonzero(np.diff(D.indptr))[0]
    assert not np.any(mask[rows[rows < g.n_f]])
    assert rows.size > 0
    Afull = mac.jacobian_modified(np.zeros(g.n_f), np.ones(g.n_f, dtype=bool))
    assert (Afull - mac.jacobian(np.zeros(g.N))).count_nonzero() == 0


def test_upwind_hand_coefficients():
    """Uniform wind c > 0 in an open channel: the convective row of an interior
    x-face is rho c (3, -4, 1)/(2h) on (f, f-1, f-2); with c < 0 it mirrors."""
    nx, n = 8, 3
    g = build_grid(slit_2d(nx, n), 2, (False, False), H)
    mac = Mac(g, RHO, MU, p_in=1.0)
    for c in (2.0, -2.0):
        w = np.zeros(g.n_f)
        w[:g.n_face[0]] = c
        C = (mac.jacobian_modified(w) - mac.jacobian(np.zeros(g.N))).tocsr()
        fd = g.face_dof[0]
        f = fd[0, 1, 4]
        row = C.getrow(f).toarray().ravel()
        s = 1 if c > 0 else -1
        exp = {f: 3.0, fd[0, 1, 4 - s]: -4.0, fd[0, 1, 4 - 2 * s]: 1.0}
        for col, k in exp.items():
            assert row[col] == pytest.approx(RHO * abs(c) * k / (2 * H), rel=1e-14)
        assert np.count_nonzero(row) == 3


def test_conservation_navier_stokes():
    """Per-cell divergence and the flux through every x-plane (mass balance)."""
    img = dumbbell_2d(24, 13, 3, 4)
    g = build_grid(img, 2, (False, False), H)
    mac = Mac(g, RHO, MU, p_in=300.0)
    x = direct_solve(mac, tol=1e-13)
    u = _x_faces(g, x)[0]
    qin = u[:, 0].sum() * H
    d = mac.Div @ x[:g.n_f]
    assert np.abs(d).max() <= 1e-8 * qin / H / H
    q = u.sum(axis=0) * H
    assert np.allclose(q, qin, rtol=1e-10)


def test_stokes_newton_one_step_and_permeability():
    """Stokes (rho = 0): r is affine, Newton converges in one step;
    K = mu L U_D / dp is independent of dp."""
    g = _blob_case(2, (False, False), seed=7)
    Ks = []
    for dp in (1.0, 7.5):
        mac = Mac(g, 0.0, MU, p_in=dp)
        dec = decompose(g, 1.0, 3, 1, 2)
        M = build_gplmm(mac, dec)
        rep = {}
        x = newton(mac, M, np.zeros(g.N), tol=1e-10, report=rep)
        assert len(rep["krylov"]) == 1
        u = _x_faces(g, x)[0]
        UD = u[:, -1].sum() / g.ny
        Ks.append(MU * (g.nx + 1) * H * UD / dp)
    assert Ks[0] == pytest.approx(Ks[1], rel=1e-8)


@pytest.mark.parametrize("dim", [2, 3])
def test_newton_gmres_matches_direct(dim):
    """O-def vs O-alg: Newton-FGMRES-gPLMM reaches the splu Newton solution."""
    if dim == 2:
        # (round 1 used random_blobs(28, 16, 1, 0.55, 2.5, 11), a dead-end image
        # with no inlet-to-outlet path: zero velocity made the check vacuous)
        img = random_blobs(33, 20, 1, 0.5, 2.5, 4)
        g = build_grid(img, 2, (False, False), H)
        dec = decompose(g, 0.5, 3, 1, 2)
    else:
        img = random_blobs(12, 10, 10, 0.5, 2.0, 12)
        g = build_grid(img, 3, (True, True), H)
        dec = decompose(g, 0.5, 5, 1, 2)
    mac = Mac(g, RHO, MU, p_in=400.0)
    x, rep = solve_steady(mac, dec)
    assert rep["converged"]
    xs = direct_solve(mac, tol=1e-13)
    out = g.face_dof[0][..., -1]
    assert xs[out[out >= 0]].sum() > 1e-3 * np.abs(xs[:g.n_f]).max()     # through-flow
    nf = g.n_f
    assert np.linalg.norm(x[:nf] - xs[:nf]) <= 1e-7 * np.linalg.norm(xs[:nf])
    assert np.linalg.norm(x[nf:] - xs[nf:]) <= 1e-7 * np.linalg.norm(xs[nf:])
    r = mac.residual(x)
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(mac.b0())
