"""ORACLE (test infrastructure only) — Newton drivers.

PAPER.md Eq. Ax=b: J^k delta^k = -r^k, x^{k+1} = x^k + delta^k.
Readings:
* A19 steady pipeline: build M_S = gPLMM with w = 0 (= aPLMM_S) and
  M_L from J(0); Newton step 0 from x = 0 (the Stokes solve); then rebuild
  gPLMM with wind w = u(x^1) (P:555 Stokes fallback) and M_L from J(x^1);
  continue Newton.  No rebuild inside the Newton loop.
* A22 Krylov tolerance ||r^k + J^k delta|| <= 1e-9 ||b_0||.
* A23 Newton tolerance ||r(x^k)|| <= 1e-8 ||b_0||, at most 30 iterations,
  no damping.
* A18 (revised, R9): the preconditioner is a fixed operator during
  the Newton loop: its composition (Eq. mono_struct, Eq. Mdp) uses the same
  A_b = J(x_b) as its local blocks (Eq. Mp_Md), not the current J^k.
"""
from __future__ import annotations

import time

import numpy as np
import scipy.sparse.linalg as spla

from .gplmm import GPLMM
from .decomposition import masked_faces
from .krylov import fgmres


def build_gplmm(mac, dec, x_b=None, mask=None, algebraic=False):
    """gPLMM built from J~_w (w = u(x_b)) and M_L from J(x_b).  algebraic=True
    builds aPLMM instead: M_G from the plain Jacobian J(x_b)
    (no wind linearisation, no inertia mask)."""
    N, nf = mac.N, mac.nf
    xb = np.zeros(N) if x_b is None else x_b
    if mask is None:
        mask = masked_faces(mac.g, dec)
    A_G = mac.jacobian(xb) if algebraic else mac.jacobian_modified(xb[:nf], mask)
    A_L = mac.jacobian(xb)
    bB = -mac.residual(np.zeros(N), np.zeros(nf))       # -r_steady(0, 0)
    if mac.dt > 0.0:
        # r_steady excludes rho u^n/dt (A16); with u = u^n = 0 it is the same
        pass
    return GPLMM(mac.g, dec, A_G, A_L, bB)


def newton(mac, prec, x, u_prev=None, tol=1e-8, ktol=1e-9, m=50, max_newton=30,
           max_krylov=2000, b0n=None, report=None):
    """Newton iterations with a fixed preconditioner.  Returns x."""
    if b0n is None:
        b0n = np.linalg.norm(mac.b0())
    if report is None:
        report = {}
    report.setdefault("krylov", [])
    report.setdefault("res", [])
    report.setdefault("converged", False)
    for k in range(max_newton):
        r = mac.residual(x, u_prev)
        rn = np.linalg.norm(r) / b0n
        report["res"].append(rn)
        if rn <= tol:
            report["converged"] = True
            return x
        J = mac.jacobian(x)
        A = lambda v: J @ v  # noqa: E731
        M = lambda v: prec.apply(v, prec.A_b)  # noqa: E731   (reading A18 / R9: A_b = J(x_b))
        d, it, ok, _ = fgmres(A, -r, M, ktol * b0n, m=m, maxit=max_krylov)
        report["krylov"].append(it)
        x = x + d
    r = mac.residual(x, u_prev)
    rn = np.linalg.norm(r) / b0n
    report["res"].append(rn)
    report["converged"] = rn <= tol
    return x


def solve_steady(mac, dec, tol=1e-8, ktol=1e-9, m=50, max_newton=30, variant="gPLMM"):
    """Steady pipeline A19.  Returns (x, report).
    variant: "gPLMM" (rebuild from J~_w with the Stokes wind after step 0),
    "aPLMM_S" (built once from the Stokes Jacobian, reused for every Newton
    step), "aPLMM_NS" (rebuilt like gPLMM but M_G from J(x^1))."""
    N = mac.N
    rep = {"krylov": [], "res": []}
    b0n = np.linalg.norm(mac.b0())
    t0 = time.perf_counter()
    mask = masked_faces(mac.g, dec)
    MS = build_gplmm(mac, dec, None, mask)
    t1 = time.perf_counter()
    x = np.zeros(N)
    if variant == "aPLMM_S":
        x = newton(mac, MS, x, None, tol, ktol, m, max_newton, b0n=b0n, report=rep)
        t2 = time.perf_counter()
        rep["t_build"] = t1 - t0
        rep["t_sol"] = t2 - t1
        return x, rep
    x = newton(mac, MS, x, None, tol, ktol, m, 1, b0n=b0n, report=rep)
    t2 = time.perf_counter()
    if not rep["converged"]:
        rep["res"].pop()
        del MS                                   # (host memory: one preconditioner alive at a time)
        M = build_gplmm(mac, dec, x, mask, algebraic=(variant == "aPLMM_NS"))
        t3 = time.perf_counter()
        x = newton(mac, M, x, None, tol, ktol, m, max_newton - 1, b0n=b0n, report=rep)
        t4 = time.perf_counter()
    else:
        t3 = t4 = t2
    rep["t_build"] = (t1 - t0) + (t3 - t2)
    rep["t_sol"] = (t2 - t1) + (t4 - t3)
    return x, rep


def direct_solve(mac, x0=None, u_prev=None, tol=1e-10, max_newton=50):
    """O-def: Newton with sparse direct solves (splu) — brute force x*."""
    x = np.zeros(mac.N) if x0 is None else x0.copy()
    b0n = np.linalg.norm(mac.b0())
    for _ in range(max_newton):
        r = mac.residual(x, u_prev)
        if np.linalg.norm(r) <= tol * b0n:
            return x
        J = mac.jacobian(x)
        x = x - spla.splu(J.tocsc()).solve(r)
    return x


def solve_transient(mac, dec, n_steps, x0=None, tol=1e-8, ktol=1e-9, m=50, max_newton=30):
    """Transient pipeline (readings A7, A19; SURVEY config 4: "not in
    between dt steps or Newton iterations"): the preconditioner is built ONCE,
    from the steady-Stokes state x_S (wind w = u(x_S), M_L from J(x_S)),
    with rho/dt included (mac.dt > 0); then each backward-Euler step
    solves r(x; u^n) = 0 by Newton from x = x^n.  x_S is Newton step 0 of the
    steady problem (dt = 0) from rest, i.e. the Stokes solution.
    Returns (x after n_steps, report with per-step Newton/Krylov counts)."""
    from .mac import Mac
    N, nf = mac.N, mac.nf
    steady = Mac(mac.g, mac.rho, mac.mu, body_force=mac.bf, p_in=mac.p_in, p_out=mac.p_out, dt=0.0)
    b0s = np.linalg.norm(steady.b0())
    MS = build_gplmm(steady, dec, None)
    xs = newton(steady, MS, np.zeros(N), None, tol, ktol, m, 1, b0n=b0s)
    P = build_gplmm(mac, dec, xs)
    b0n = np.linalg.norm(mac.b0())
    x = np.zeros(N) if x0 is None else x0.copy()
    rep = {"steps": []}
    for _ in range(n_steps):
        up = x[:nf].copy()
        r = {"krylov": [], "res": []}
        x = newton(mac, P, x, up, tol, ktol, m, max_newton, b0n=b0n, report=r)
        rep["steps"].append(r)
    rep["stokes"] = xs
    return x, rep


def coarse_solve(mac, dec, n_ramp=2, tol=1e-6, max_newton=50):
    """Coarse-scale steady Navier-Stokes solver, Algorithm 1.

    Outer loop over drive increments k = 1..n_ramp (p_in, p_out and b scaled
    by k/n_ramp: the paper ramps Re by raising p_in); wind w =
    velocity of the previous increment (0, the Stokes fallback, for the
    first); M_G built from J~_w (R^, P^; Remark 1); Newton on the coarse
    unknowns only:
        r_c = R^ r~(x^),  J_c = R^ J~^k P^,  delta_c = -J_c^{-1} r_c,
        x^ <- x^ + P^ delta_c   (Eq. coarse_scale_sys, coarse_rJ, coarse_scale_up)
    until ||r_c|| / ||r_c^0|| < tol (1e-6 in the paper).
    Returns (x^, report: Newton counts per increment)."""
    from .mac import Mac
    from .gplmm import GPLMM
    g = mac.g
    mask = masked_faces(g, dec)
    N, nf = mac.N, mac.nf
    x = np.zeros(N)
    rep = {"newton": [], "res": []}
    for k in range(1, n_ramp + 1):
        f = k / n_ramp
        mk = Mac(g, mac.rho, mac.mu, body_force=mac.bf * f, p_in=mac.p_in * f, p_out=mac.p_out * f, dt=0.0)
        w = x[:nf].copy()
        A_G = mk.jacobian_modified(w, mask)
        bB = -mk.residual(np.zeros(N), np.zeros(nf))
        P = GPLMM(g, dec, A_G, None, bB, build_ml=False)
        rc = P.Rhat @ mk.residual_masked(x, mask)
        rc0 = np.linalg.norm(rc)
        it = 0
        while it < max_newton and rc0 > 0:
            Jc = (P.Rhat @ mk.jacobian_masked(x, mask) @ P.Phat).toarray()
            d = -np.linalg.solve(Jc, rc)
            x = x + P.Phat @ d
            rc = P.Rhat @ mk.residual_masked(x, mask)
            it += 1
            if np.linalg.norm(rc) / rc0 < tol:
                break
        rep["newton"].append(it)
        rep["res"].append(np.linalg.norm(rc) / rc0 if rc0 > 0 else 0.0)
    return x, rep


def solve_continuation(mac, dec, n_incr, tol=1e-8, ktol=1e-9, m=50, max_newton=30):
    """Re continuation (homotopy): drive increments
    k = 1..n_incr with p_in, p_out, b scaled by k/n_incr.  Increment 1 is the
    steady pipeline (A19) from rest; increment k >= 2 rebuilds gPLMM at the
    start of the increment with the previous solution as wind and M_L state
    ("rebuilt ... before the Newton loop is entered, but not during")
    and runs Newton from that solution.  Returns (x, report)."""
    from .mac import Mac
    g = mac.g
    mask = masked_faces(g, dec)
    x = None
    rep = {"increments": []}
    for k in range(1, n_incr + 1):
        f = k / n_incr
        mk = Mac(g, mac.rho, mac.mu, body_force=mac.bf * f, p_in=mac.p_in * f, p_out=mac.p_out * f, dt=0.0)
        if k == 1:
            x, r = solve_steady(mk, dec, tol, ktol, m, max_newton)
        else:
            r = {"krylov": [], "res": []}
            M = None                             # (host memory: drop the previous increment's first)
            M = build_gplmm(mk, dec, x, mask)
            x = newton(mk, M, x, None, tol, ktol, m, max_newton, b0n=np.linalg.norm(mk.b0()), report=r)
        rep["increments"].append(r)
    return x, rep
