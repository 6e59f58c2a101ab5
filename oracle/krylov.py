"""ORACLE (test infrastructure only) — right-preconditioned flexible GMRES.

PAPER.md P:760: GMRES with right preconditioning, convergence when
||A x - b|| / ||b_0|| < 1e-9 with b_0 = r(u = 0, p = 0).  Readings (SURVEY
§8(c) A21-A22): flexible variant (the preconditioner is fixed, so FGMRES
and GMRES coincide in exact arithmetic), x_0 = 0, restart m = 50, modified
Gram-Schmidt, Givens rotations; the Arnoldi residual estimate is tested each
iteration and the true residual at exit (restarting if it fails).
"""
from __future__ import annotations

import numpy as np


def fgmres(A, b, Minv, tol_abs, m=50, maxit=2000):
    """Solve A x = b.  ``A`` and ``Minv`` are callables.  Returns
    (x, n_iters, converged, history of |g_{j+1}|)."""
    n = b.shape[0]
    x = np.zeros(n)
    r = b.copy()
    total = 0
    hist = []
    beta = np.linalg.norm(r)
    while True:
        if beta <= tol_abs:
            return x, total, True, hist
        if total >= maxit:
            return x, total, False, hist
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        gv = np.zeros(m + 1)
        gv[0] = beta
        V[0] = r / beta
        j_end = 0
        for j in range(m):
            Z[j] = Minv(V[j])
            w = A(Z[j])
            for i in range(j + 1):                       # MGS
                H[i, j] = np.dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                           # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            gv[j + 1] = -sn[j] * gv[j]
            gv[j] = cs[j] * gv[j]
            total += 1
            j_end = j + 1
            hist.append(abs(gv[j + 1]))
            if abs(gv[j + 1]) <= tol_abs or total >= maxit:
                break
        k = j_end
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):                   # back substitution
            y[i] = (gv[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        x = x + Z[:k].T @ y
        r = b - A(x)
        beta = np.linalg.norm(r)
