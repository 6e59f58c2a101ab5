"""ORACLE (test infrastructure only) — gPLMM two-level preconditioner by
explicit sparse matrices, a literal transcription of PAPER.md §3.2.2-§4.

* Permutation W (Eq. permute): ``decomposition.w_order``.
* Reduction / fold (Eq. reduce_1, Eq. reduce_2):
      A~^p_p = A^p_p + diag(csum(A^p_f)),
      Abar^{p_i}_{p_i} = A~^{p_i}_{p_i} + diag(sum_{j != i} csum(A~^{p_i}_{p_j})).
* Reduction matrix Q = blockdiag(I, Q°), Q° = blockdiag(1^{c_j}) (Eq. reduce_3).
* Prolongation P = [[B, C], [I, O]] (Eq. prolong_1), shape vectors
      p^{p_i}_{c_j} = -(Abar^{p_i}_{p_i})^{-1} R^{p_i}_p Abar^p_c e^{c_j}
  (Eq. prolong_3; zero automatically for c_j not in C^{p_i}) and correction
  vectors c^{p_i} = (Abar^{p_i}_{p_i})^{-1} b_B^{p_i} (Eq. prolong_2),
  b_B = -r_steady(u = 0, p = 0) permuted.
* Restriction R = [[O, I], [Pi(C^T), O]] (Eq. restrict_FVM).
* Effective P^ = W [Q P; F] with the interface f-rows F given by the
  homogeneous back-substitution of Eq. xf (reading A14), R^ = R Q^T W^T
  (Eq. iMG_PR; the f-block is discarded).
* Coarse matrix (Remark 1, reading A13): A° = R^ A^ P^ with
  A^ = J~_w.  Optionally the un-simplified Eq. iMG with
  A_check = W C(W^T A^ W) W^T (Proposition 1 test).
* Readings A15 (y_i dropped where b_B^{p_i} = 0; Pi(C^T) = 1 on every row of
  p_i) and A17 (M_L local blocks are principal submatrices of J(x_b)).
* Smoother M_dp (Eq. Mdp, Eq. Mp_Md) and the two-level
  composition (Eq. mono_struct, n_st = 1):
      z_G = M_G^{-1} v; s = v - A z_G; z_d = M_d^{-1} s; t = s - A z_d;
      z = z_G + z_d + M_p^{-1} t
  (reading A18, revised in round 2 -- DESIGN.md R9: A = A_b = J(x_b), the same
  A^ the local blocks of Eq. Mp_Md are taken from, because the preconditioner
  is built once before the Newton loop; `apply(v, J)` takes the
  matrix explicitly so tests can also evaluate other compositions).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .decomposition import w_order, subdomain_unknowns


def _ones(n):
    return np.ones(n)


class GPLMM:
    def __init__(self, g, dec, A_G: sp.csr_matrix, A_L: sp.csr_matrix, b_B: np.ndarray,
                 use_fold_in_coarse: bool = False, build_ml: bool = True):
        """A_G = matrix M_G is built from (J~_w); A_L = matrix the smoother's
        local blocks come from (J(x_b)); b_B = -r_steady(0, 0) (canonical)."""
        self.g, self.dec = g, dec
        N = g.N
        self.N = N
        perm, seg = w_order(g, dec)
        self.perm, self.seg = perm, seg
        n_p, n_c = dec.n_p, dec.n_c
        self.n_p, self.n_c = n_p, n_c
        Np_f = int(seg[n_p])
        Nc_f = int(seg[n_p + n_c]) - Np_f
        self.Np_f, self.Nc_f = Np_f, Nc_f
        # W: x^ = W x  (x in permuted order)
        W = sp.csr_matrix((np.ones(N), (perm, np.arange(N))), shape=(N, N))
        self.W = W
        A = (W.T @ A_G @ W).tocsr()
        ip = slice(0, Np_f)
        ic = slice(Np_f, Np_f + Nc_f)
        iF = slice(Np_f + Nc_f, N)
        App, Apc, Apf = A[ip, ip], A[ip, ic], A[ip, iF]
        Acp, Acc, Acf = A[ic, ip], A[ic, ic], A[ic, iF]
        Afp, Afc, Aff = A[iF, ip], A[iF, ic], A[iF, iF]
        # --- Eq. reduce_1 ---
        Atpp = (App + sp.diags(Apf @ _ones(Apf.shape[1]))).tocsr()
        Atcc = (Acc + sp.diags(Acf @ _ones(Acf.shape[1]))).tocsr()
        # --- Eq. reduce_2 ---
        self.Abar = []
        rows_all = Atpp @ _ones(Np_f)
        for i in range(n_p):
            s = slice(int(seg[i]), int(seg[i + 1]))
            Aii = Atpp[s, s]
            off = rows_all[s] - Aii @ _ones(Aii.shape[1])
            self.Abar.append((Aii + sp.diags(off)).tocsc())
        # --- Eq. reduce_3: Q° ---
        ifc_of_cell = np.repeat(np.arange(n_c), np.diff(seg[n_p:n_p + n_c + 1]))
        Qo = sp.csr_matrix((np.ones(Nc_f), (np.arange(Nc_f), ifc_of_cell)), shape=(Nc_f, n_c))
        self.Qo = Qo
        Abar_pc = (Apc @ Qo).tocsc()
        # --- shape vectors B (Eq. prolong_3) and correction vectors (Eq. prolong_2) ---
        bB = W.T @ b_B
        Bcols = []
        Ccols = []
        kept = []
        for i in range(n_p):
            s = slice(int(seg[i]), int(seg[i + 1]))
            lu_bar = spla.splu(self.Abar[i])    # (factor, use, drop: host memory only)
            rhs = Abar_pc[s, :].toarray()
            nz = np.nonzero(np.any(rhs != 0.0, axis=0))[0]      # C^{p_i}
            blk = np.zeros((s.stop - s.start, n_c))
            if nz.size:
                blk[:, nz] = -lu_bar.solve(rhs[:, nz])
            Bcols.append(sp.csr_matrix(blk))
            bi = bB[s]
            if np.any(bi != 0.0):
                kept.append(i)
                Ccols.append(lu_bar.solve(bi))
            else:
                Ccols.append(None)
        self.kept = kept
        self.C_of = {i: Ccols[i] for i in kept}
        B = sp.vstack(Bcols, format="csr") if n_p else sp.csr_matrix((0, n_c))
        nB = len(kept)
        crow, ccol, cval = [], [], []
        for k, i in enumerate(kept):
            s0 = int(seg[i])
            v = Ccols[i]
            crow.append(np.arange(s0, s0 + len(v))); ccol.append(np.full(len(v), k)); cval.append(v)
        Cm = sp.csr_matrix((np.concatenate(cval) if cval else [],
                            (np.concatenate(crow) if crow else [], np.concatenate(ccol) if ccol else [])),
                           shape=(Np_f, nB))
        self.B, self.Cm = B, Cm
        # P = [[B, C], [I, O]]
        P = sp.bmat([[B, Cm], [sp.identity(n_c), sp.csr_matrix((n_c, nB))]], format="csr")
        # R = [[O, I], [Pi(C^T), O]]  (A15: 1 on every row of p_i)
        pr, pc = [], []
        for k, i in enumerate(kept):
            pr.append(np.full(int(seg[i + 1] - seg[i]), k)); pc.append(np.arange(int(seg[i]), int(seg[i + 1])))
        Pi = sp.csr_matrix((np.ones(sum(len(x) for x in pr)),
                            (np.concatenate(pr) if pr else [], np.concatenate(pc) if pc else [])),
                           shape=(nB, Np_f))
        R = sp.bmat([[sp.csr_matrix((n_c, Np_f)), sp.identity(n_c)],
                     [Pi, sp.csr_matrix((nB, n_c))]], format="csr")
        Q = sp.block_diag([sp.identity(Np_f), Qo], format="csr")
        QP = (Q @ P).tocsr()
        # f-rows (Eq. xf, homogeneous; reading A14)
        Nf_f = N - Np_f - Nc_f
        if Nf_f:
            rhs = (sp.hstack([Afp, Afc]) @ QP).tocsc()
            F = -spla.splu(Aff.tocsc()).solve(rhs.toarray())
            F = sp.csr_matrix(F)
        else:
            F = sp.csr_matrix((0, n_c + nB))
        self.Phat = (W @ sp.vstack([QP, F])).tocsr()
        Rt = sp.hstack([(R @ Q.T), sp.csr_matrix((n_c + nB, Nf_f))]).tocsr()
        self.Rhat = (Rt @ W.T).tocsr()
        self.n_coarse = n_c + nB
        # coarse matrix
        if use_fold_in_coarse:
            Cfold = sp.bmat([[sp.block_diag(self.Abar), Apc, None],
                             [Acp, Atcc, None],
                             [Afp, Afc, Aff]], format="csr")
            Acheck = W @ Cfold @ W.T
            self.Acoarse = (self.Rhat @ Acheck @ self.Phat).toarray()
        else:
            self.Acoarse = (self.Rhat @ A_G @ self.Phat).toarray()
        self.coarse_lu = sla.lu_factor(self.Acoarse) if self.n_coarse else None
        # --- smoother local blocks (A17) ---
        if not build_ml:
            return
        A_L = A_L.tocsr()
        # A_b: the system matrix of the composition (Eq. mono_struct / Mdp use
        # the same A^ as the local blocks of Eq. Mp_Md; built once)
        self.A_b = A_L
        self.p_sets = [perm[int(seg[i]):int(seg[i + 1])] for i in range(n_p)]
        self.d_sets = [subdomain_unknowns(g, cells) for cells in dec.dual_cells]
        self.lu_p = [spla.splu(A_L[s][:, s].tocsc()) for s in self.p_sets]
        self.lu_d = [spla.splu(A_L[s][:, s].tocsc()) for s in self.d_sets]

    # ------------------------------------------------------------------
    def MG(self, v):
        """M_G^{-1} v = P^ (A°)^{-1} R^ v (Eq. iMG with Remark 1)."""
        if self.n_coarse == 0:
            return np.zeros(self.N)
        bc = self.Rhat @ v
        xc = sla.lu_solve(self.coarse_lu, bc)
        return self.Phat @ xc

    def Mp(self, v):
        z = np.zeros(self.N)
        for s, lu in zip(self.p_sets, self.lu_p):
            z[s] += lu.solve(v[s])
        return z

    def Md(self, v):
        z = np.zeros(self.N)
        for s, lu in zip(self.d_sets, self.lu_d):
            z[s] += lu.solve(v[s])
        return z

    def ML(self, v, J):
        """M_dp^{-1} v = M_d^{-1} v + M_p^{-1}(v - J M_d^{-1} v) (Eq. Mdp)."""
        zd = self.Md(v)
        return zd + self.Mp(v - J @ zd)

    def apply(self, v, J):
        """M^{-1} v (Eq. mono_struct, n_st = 1, M_l = M_dp)."""
        zG = self.MG(v)
        s = v - J @ zG
        zd = self.Md(s)
        t = s - J @ zd
        return zG + zd + self.Mp(t)
