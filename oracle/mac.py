"""ORACLE (test infrastructure only) — MAC residual and Jacobians as SciPy CSR.

What it computes (§1 Eq. governing_eqs, Eq. Ax=b P:34-65,
§2, §4 Eq. mod_res) under SURVEY.md §8(c) readings:

  r_u = rho (u - u^n)/dt + rho N(u) - mu L u + G p + g0 - rho b      (faces)
  r_p = Div u                                                        (cells)

* A3  p_in / p_out sit at ghost cell centres h/2 outside x-min / x-max;
      the boundary-face gradient is (p_1 - p_in)/h.  Inlet/outlet dn u = 0 is
      a mirror ghost (value u_f) in viscous and convective stencils.
* A5  N(u) = sum_b c_b(u) D_b(u): c_a = u_f; for b != a, c_b = mean of the
      4 b-faces bounding f's two flanking cells (non-DOF faces count 0; at an
      x-boundary face the single flanking cell's 2 b-faces).  D_b is the
      three-point one-sided upwind derivative
          D_b u = s (3 u_f - 4 V(f - s e_b) + V(f - 2 s e_b)) / (2h),
      s = +1 if c_b >= 0 else -1, with the 1st-order fallback
          D_b u = s (u_f - V(f - s e_b)) / h
      when f - 2 s e_b is neither a DOF nor a zero face.  (The survey's
      formula omits the factor s; without it the s = -1 branch would have the
      wrong sign — DESIGN.md reading R1.)
* A6  L u = sum_b (V(f+e_b) - 2 u_f + V(f-e_b)) / h^2 with the same V rule:
      DOF -> u_m; one solid flank -> 0; both flanks solid -> -u_f;
      beyond inlet/outlet -> u_f; periodic -> wrap.
* A7/A8  backward Euler; body force -rho b_a on every a-face; no volume
      scaling (momentum rows in Pa/m, mass rows in 1/s).
* A9  J = exact derivative of r with the upwind selector frozen:
      dN = sum_b diag(c_b(u)) D_b + diag(D_b u) dc_b/du.
* A10 J~_w (Eq. mod_res): Oseen with wind w (upwind selector from c_b(w)),
      no reaction term, inertia removed on masked faces, rho/dt kept.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .grid import DOF, ZERO, GHOST, MIRROR, VOID, Grid


def _shift(pos, b, o):
    K, J, I = pos
    if b == 0:
        return (K, J, I + o)
    if b == 1:
        return (K, J + o, I)
    return (K + o, J, I)


class Mac:
    """MAC operators on a Grid.  Unknown vector x = [u (n_f); p (n_c)] in
    canonical order (faces first, then cells)."""

    def __init__(self, g: Grid, rho: float, mu: float, body_force=(0.0, 0.0, 0.0),
                 p_in: float = 0.0, p_out: float = 0.0, dt: float = 0.0):
        self.g = g
        self.rho, self.mu, self.dt = float(rho), float(mu), float(dt)
        self.bf = np.array(list(body_force) + [0.0] * (3 - len(body_force)), dtype=float)
        self.p_in, self.p_out = float(p_in), float(p_out)
        self.nf, self.nc, self.N = g.n_f, g.n_c, g.N
        self._build_static()

    # ------------------------------------------------------------------
    def _face_positions(self, a):
        fd = self.g.face_dof[a]
        K, J, I = np.nonzero(fd >= 0)
        return (K, J, I), fd[K, J, I]

    def _build_static(self):
        g, h, nf, nc = self.g, self.g.h, self.nf, self.nc
        dim = g.dim
        self.orient = np.zeros(nf, dtype=np.int64)
        for a in range(dim):
            _, ids = self._face_positions(a)
            self.orient[ids] = a
        # neighbour-value operators S[(b, o)] and "DOF or zero face" flags
        self.S = {}
        self.dz = {}
        for b in range(dim):
            for o in (-2, -1, 1, 2):
                rows, cols, vals = [], [], []
                flag = np.zeros(nf, dtype=bool)
                for a in range(dim):
                    pos, ids = self._face_positions(a)
                    code, idx = g.classify(a, *_shift(pos, b, o))
                    m = code == DOF
                    rows.append(ids[m]); cols.append(idx[m]); vals.append(np.ones(m.sum()))
                    m = code == GHOST
                    rows.append(ids[m]); cols.append(ids[m]); vals.append(-np.ones(m.sum()))
                    m = code == MIRROR
                    rows.append(ids[m]); cols.append(ids[m]); vals.append(np.ones(m.sum()))
                    flag[ids] = (code == DOF) | (code == ZERO)
                self.S[(b, o)] = sp.csr_matrix(
                    (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(nf, nf))
                self.dz[(b, o)] = flag
        I_f = sp.identity(nf, format="csr")
        # viscous Laplacian (A6)
        L = sp.csr_matrix((nf, nf))
        for b in range(dim):
            L = L + (self.S[(b, 1)] - 2.0 * I_f + self.S[(b, -1)]) / (h * h)
        self.L = L.tocsr()
        # advecting-velocity operators C_b (A5)
        self.C = {}
        for b in range(dim):
            rows, cols, vals = [], [], []
            for a in range(dim):
                pos, ids = self._face_positions(a)
                if a == b:
                    rows.append(ids); cols.append(ids); vals.append(np.ones(len(ids)))
                    continue
                (k0, j0, i0), (k1, j1, i1) = g.face_flanks(a, *pos)
                s0 = g.cell_state(k0, j0, i0)
                s1 = g.cell_state(k1, j1, i1)
                nin = (s0 == VOID).astype(float) + (s1 == VOID).astype(float)
                w = 1.0 / (2.0 * nin)
                for (cell, st) in (((k0, j0, i0), s0), ((k1, j1, i1), s1)):
                    for o in (0, 1):
                        fpos = _shift(cell, b, o)
                        code, idx = g.classify(b, *fpos)
                        m = (st == VOID) & (code == DOF)
                        rows.append(ids[m]); cols.append(idx[m]); vals.append(w[m])
            self.C[b] = sp.csr_matrix(
                (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(nf, nf))
        # upwind derivative pieces (A5): D+ (s = +1) and D- (s = -1)
        self.Dp, self.Dm = {}, {}
        for b in range(dim):
            u2 = self.dz[(b, -2)].astype(float)
            D2 = (3.0 * I_f - 4.0 * self.S[(b, -1)] + self.S[(b, -2)]) / (2.0 * h)
            D1 = (I_f - self.S[(b, -1)]) / h
            self.Dp[b] = (sp.diags(u2) @ D2 + sp.diags(1.0 - u2) @ D1).tocsr()
            u2 = self.dz[(b, 2)].astype(float)
            D2 = (3.0 * I_f - 4.0 * self.S[(b, 1)] + self.S[(b, 2)]) / (2.0 * h)
            D1 = (I_f - self.S[(b, 1)]) / h
            self.Dm[b] = (-(sp.diags(u2) @ D2 + sp.diags(1.0 - u2) @ D1)).tocsr()
        # gradient G (n_f x n_c), boundary vector g0, divergence Div (n_c x n_f)
        rows, cols, vals = [], [], []
        g0 = np.zeros(nf)
        for a in range(dim):
            pos, ids = self._face_positions(a)
            (k0, j0, i0), (k1, j1, i1) = g.face_flanks(a, *pos)
            for (cell, sgn) in (((k0, j0, i0), -1.0), ((k1, j1, i1), 1.0)):
                st = g.cell_state(*cell)
                m = st == VOID
                cid = g.cell_dof[cell[0][m], cell[1][m], cell[2][m]] - nf
                rows.append(ids[m]); cols.append(cid); vals.append(np.full(m.sum(), sgn / h))
            if a == 0:
                I = pos[2]
                g0[ids[I == 0]] = -self.p_in / h
                g0[ids[I == g.nx]] = self.p_out / h
        self.G = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(nf, nc))
        self.g0 = g0
        rows, cols, vals = [], [], []
        K, J, I = np.nonzero(g.cell_dof >= 0)
        cid = g.cell_dof[K, J, I] - nf
        for b in range(dim):
            for (o, sgn) in ((0, -1.0), (1, 1.0)):
                code, idx = g.classify(b, *_shift((K, J, I), b, o))
                m = code == DOF
                rows.append(cid[m]); cols.append(idx[m]); vals.append(np.full(m.sum(), sgn / h))
        self.Div = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                 shape=(nc, nf))
        # body force per face row
        self.fb = self.rho * self.bf[self.orient]

    # ------------------------------------------------------------------
    def _conv_parts(self, u_adv):
        """c_b(u_adv) and the upwind operators D_b with s frozen from c_b."""
        out = []
        for b in range(self.g.dim):
            c = self.C[b] @ u_adv
            sp_ = (c >= 0.0).astype(float)
            D = (sp.diags(sp_) @ self.Dp[b] + sp.diags(1.0 - sp_) @ self.Dm[b]).tocsr()
            out.append((c, D))
        return out

    def convection(self, u):
        """N(u) = sum_b c_b(u) D_b(u) u (A5)."""
        n = np.zeros(self.nf)
        for c, D in self._conv_parts(u):
            n += c * (D @ u)
        return n

    def residual(self, x, u_prev=None, inertia=True):
        """r(x) (Eq. Ax=b / Eq. mod_res with w = u)."""
        nf = self.nf
        u, p = x[:nf], x[nf:]
        ru = -self.mu * (self.L @ u) + self.G @ p + self.g0 - self.fb
        if inertia:
            ru = ru + self.rho * self.convection(u)
        if self.dt > 0.0:
            up = np.zeros(nf) if u_prev is None else u_prev
            ru = ru + self.rho * (u - up) / self.dt
        rp = self.Div @ u
        return np.concatenate([ru, rp])

    def residual_masked(self, x, mask):
        """r~ of Eq. mod_res with w = u: the true steady residual with
        the inertia term removed on the masked faces (coarse-scale solver)."""
        nf = self.nf
        u, p = x[:nf], x[nf:]
        keep = (~np.asarray(mask, dtype=bool)).astype(float)
        ru = -self.mu * (self.L @ u) + self.G @ p + self.g0 - self.fb + self.rho * keep * self.convection(u)
        return np.concatenate([ru, self.Div @ u])

    def jacobian_masked(self, x, mask):
        """J~^k: the Newton Jacobian with inertia removed on masked faces."""
        u = x[:self.nf]
        keep = sp.diags((~np.asarray(mask, dtype=bool)).astype(float))
        F = -self.mu * self.L
        for b, (c, D) in enumerate(self._conv_parts(u)):
            F = F + self.rho * keep @ (sp.diags(c) @ D + sp.diags(D @ u) @ self.C[b])
        return self._assemble(F.tocsr())

    def b0(self):
        """b^_0 = r(u = 0, p = 0) with u^n = 0."""
        return self.residual(np.zeros(self.N), np.zeros(self.nf))

    def _assemble(self, F):
        return sp.bmat([[F, self.G], [self.Div, None]], format="csr")

    def stokes_F(self):
        F = -self.mu * self.L
        if self.dt > 0.0:
            F = F + (self.rho / self.dt) * sp.identity(self.nf)
        return F.tocsr()

    def jacobian(self, x):
        """J(x) (A9): exact derivative with the upwind selector frozen."""
        u = x[:self.nf]
        F = self.stokes_F()
        for b, (c, D) in enumerate(self._conv_parts(u)):
            F = F + self.rho * (sp.diags(c) @ D + sp.diags(D @ u) @ self.C[b])
        return self._assemble(F.tocsr())

    def jacobian_modified(self, w, mask=None):
        """J~_w (A10, Eq. mod_res): Oseen with wind w, inertia removed on masked faces."""
        F = self.stokes_F()
        keep = np.ones(self.nf) if mask is None else (~np.asarray(mask, dtype=bool)).astype(float)
        for c, D in self._conv_parts(w):
            F = F + self.rho * (sp.diags(keep * c) @ D)
        return self._assemble(F.tocsr())
