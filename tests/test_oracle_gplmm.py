"""Pins of the oracle's gPLMM (§3.2.2-§4) against exact identities."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spla

from synth.geometry import slit_2d, random_blobs, load_config, make_image, dumbbell_2d
from oracle.grid import build_grid
from oracle.mac import Mac
from oracle.decomposition import decompose, masked_faces
from oracle.gplmm import GPLMM
from oracle.newton import build_gplmm
from oracle.krylov import fgmres

H, MU, RHO = 1e-5, 1e-3, 1000.0


def _case(dim=2, seed=4):
    if dim == 2:
        img = random_blobs(30, 18, 1, 0.55, 2.5, seed)
        g = build_grid(img, 2, (False, False), H)
        dec = decompose(g, 1.0, 4, 1, 2)
    else:
        img = random_blobs(14, 12, 12, 0.45, 2.0, seed)
        g = build_grid(img, 3, (True, True), H)
        dec = decompose(g, 0.5, 5, 1, 2)
    return g, dec


@pytest.mark.parametrize("dim", [2, 3])
def test_mg_mass_conservation(dim):
    """M_G^{-1} b^_0 is divergence-free in every primary cell and has zero net
    flux through every interface (Eq. restrict_FVM; reading A15,
    structure of A°)."""
    g, dec = _case(dim)
    assert dec.n_p >= 2 and dec.n_c >= 1
    mac = Mac(g, RHO, MU, p_in=200.0)
    x_b = np.zeros(g.N)
    P = build_gplmm(mac, dec, x_b)
    b = -mac.b0()
    z = P.MG(b)
    J = mac.jacobian(x_b)
    div = (J @ z)[g.n_f:]
    void = g.void.reshape(-1)
    prim = dec.label.reshape(-1)[void]
    ifc = dec.iface.reshape(-1)[void]
    scale = np.abs(z[:g.n_f]).max() / H
    assert np.abs(div[prim >= 0]).max() <= 1e-11 * scale
    for j in range(dec.n_c):
        assert abs(div[ifc == j].sum()) <= 1e-11 * scale


def test_shape_vectors_solve_folded_local_problems():
    """Each B column satisfies Abar_ii p + Abar^{p_i}_c e_j = 0 and is supported
    only on primaries adjacent to interface j (Eq. prolong_3)."""
    g, dec = _case(2)
    mac = Mac(g, RHO, MU, p_in=1.0)
    P = build_gplmm(mac, dec)
    A = (P.W.T @ mac.jacobian(np.zeros(g.N)) @ P.W).tocsr()
    Np_f = P.Np_f
    Apc = A[:Np_f, Np_f:Np_f + P.Nc_f] @ P.Qo
    B = P.B.toarray()
    for i in range(dec.n_p):
        s = slice(P.seg[i], P.seg[i + 1])
        res = P.Abar[i] @ B[s] + Apc[s].toarray()
        assert np.abs(res).max() <= 1e-9 * max(1.0, np.abs(Apc[s]).max())
        adj = np.nonzero(np.abs(Apc[s]).sum(axis=0).A1 > 0)[0]
        nzc = np.nonzero(np.abs(B[s]).sum(axis=0) > 0)[0]
        assert set(nzc) <= set(adj)


def test_y_identity_with_fold_and_projection():
    """With the fold kept in the coarse matrix (Eq. iMG, not Remark 1) and
    b = b^_0, the correction coefficients are y == 1 exactly (Eq. coarse_prob
    with B = -Abar^{-1} Abar^p_c, Abar c = b_B).  Remark 1's M_G^{-1} A^ is a
    projection; Eq. iMG's is not (Proposition 1)."""
    img = dumbbell_2d(24, 13, 3, 4)
    g = build_grid(img, 2, (False, False), H)
    dec = decompose(g, 0.0, 1, 1, 2)
    assert dec.n_p == 2 and dec.n_c == 1
    mac = Mac(g, RHO, MU, p_in=2.0)
    A = mac.jacobian(np.zeros(g.N))
    b = -mac.b0()
    Pf = GPLMM(g, dec, A, A, b, use_fold_in_coarse=True)
    xc = sla.lu_solve(Pf.coarse_lu, Pf.Rhat @ b)
    assert np.allclose(xc[dec.n_c:], 1.0, rtol=1e-12)
    assert 0.0 < xc[0] < 2.0          # interface pressure between p_out and p_in
    Pr = GPLMM(g, dec, A, A, b)
    Ad = A.toarray()
    Mr = np.column_stack([Pr.MG(Ad[:, k]) for k in range(g.N)])
    assert np.linalg.norm(Mr @ Mr - Mr) <= 1e-9 * np.linalg.norm(Mr)
    Mf = Pf.Phat @ sla.lu_solve(Pf.coarse_lu, (Pf.Rhat @ Ad))
    assert np.linalg.norm(Mf @ Mf - Mf) >= 1e-6 * np.linalg.norm(Mf)
    # R != P^T
    assert Pr.Rhat.shape == Pr.Phat.T.shape
    assert abs(Pr.Rhat - Pr.Phat.T).sum() > 1e-3


def test_single_primary_is_exact():
    """Straight channel: N^p = 1, N^c = 0, so M_p^{-1} = A^{-1} and
    FGMRES converges in one iteration."""
    g = build_grid(slit_2d(10, 4), 2, (False, False), H)
    dec = decompose(g, 1.0, 2, 1, 2)
    assert dec.n_p == 1 and dec.n_c == 0
    mac = Mac(g, RHO, MU, p_in=5.0)
    P = build_gplmm(mac, dec)
    J = mac.jacobian(np.zeros(g.N))
    b = -mac.b0()
    x, it, ok, _ = fgmres(lambda v: J @ v, b, lambda v: P.apply(v, J), 1e-12 * np.linalg.norm(b))
    assert ok and it == 1


def test_composition_dense_and_smoother_spectrum():
    """Dense Eq. mono_struct / Eq. Mdp equal the operator; the smoother's
    error propagation E_L = I - M_L^{-1} A has spectral radius < 1."""
    g, dec = _case(2, seed=6)
    mac = Mac(g, RHO, MU, p_in=100.0)
    P = build_gplmm(mac, dec)
    J = mac.jacobian(np.zeros(g.N))
    Ad = J.toarray()
    I = np.eye(g.N)
    MG = np.column_stack([P.MG(I[:, k]) for k in range(g.N)])
    Md = np.column_stack([P.Md(I[:, k]) for k in range(g.N)])
    Mp = np.column_stack([P.Mp(I[:, k]) for k in range(g.N)])
    ML = Md + Mp @ (I - Ad @ Md)
    M = MG + ML @ (I - Ad @ MG)
    v = np.random.default_rng(0).standard_normal(g.N)
    assert np.linalg.norm(M @ v - P.apply(v, J)) <= 1e-10 * np.linalg.norm(M @ v)
    rho_L = np.abs(np.linalg.eigvals(I - ML @ Ad)).max()
    assert rho_L < 1.0


def test_gplmm_zero_wind_is_aplmm_s():
    """gPLMM with w = 0 equals aPLMM_S: J~_0 = Stokes, so M_G is
    independent of the mask."""
    g, dec = _case(2)
    mac = Mac(g, RHO, MU, p_in=10.0)
    J0 = mac.jacobian(np.zeros(g.N))
    b = -mac.b0()
    A1 = mac.jacobian_modified(np.zeros(g.n_f), masked_faces(g, dec))
    P1 = GPLMM(g, dec, A1, J0, b)
    P2 = GPLMM(g, dec, J0, J0, b)
    v = np.random.default_rng(2).standard_normal(g.N)
    assert np.array_equal(P1.MG(v), P2.MG(v))


def test_coarse_solver_remark2_and_conservation():
    """Algorithm 1.  Remark 2: for Stokes it converges in
    one Newton iteration and equals M_G^{-1} b^ with the Remark-1 M_G.  Its
    velocity is divergence-free in every primary cell and has zero net flux
    through every interface ('weak' conservation)."""
    from oracle.newton import coarse_solve
    g, dec = _case(3)
    mac0 = Mac(g, 0.0, MU, p_in=150.0)           # Stokes (rho = 0)
    x, rep = coarse_solve(mac0, dec, n_ramp=1)
    assert rep["newton"] == [1]
    P = build_gplmm(mac0, dec)
    xg = P.MG(-mac0.b0())
    assert np.linalg.norm(x - xg) <= 1e-10 * np.linalg.norm(xg)
    mac = Mac(g, RHO, MU, p_in=800.0)
    x, rep = coarse_solve(mac, dec, n_ramp=2)
    assert all(n >= 1 for n in rep["newton"]) and rep["res"][-1] < 1e-6
    div = (mac.jacobian(np.zeros(g.N)) @ x)[g.n_f:]
    void = g.void.reshape(-1)
    prim = dec.label.reshape(-1)[void]
    ifc = dec.iface.reshape(-1)[void]
    scale = np.abs(x[:g.n_f]).max() / H
    assert np.abs(div[prim >= 0]).max() <= 1e-10 * scale
    for j in range(dec.n_c):
        assert abs(div[ifc == j].sum()) <= 1e-10 * scale
