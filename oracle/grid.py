"""ORACLE (test infrastructure only) — MAC grid, clean-up and canonical DOFs.

Follows PAPER.md §2 P:115-117 ("MAC finite difference method, with velocity
unknowns defined at cell faces and pressure unknowns at cell centers";
no-slip on the void-solid interface, inlet/outlet pressure on the left/right
external boundaries) with SURVEY.md §8(b)/(c) readings:

* D1  void components (face connectivity, periodic axes wrapped) that touch
      neither the x-min nor the x-max plane become solid.
* A1  one cell per voxel, spacing h.
* A2  faces with a solid flank carry u = 0 and are not unknowns.
* A4  non-periodic lateral boundaries are solid (no-slip) outside the image.
* Canonical order: x-face DOFs by i + (nx+1)(j + ny k), then y-face DOFs
  by i + nx(j + ny k) (face j is the low-y face of cell (i,j,k)), then z-faces
  likewise, then cells by i + nx(j + ny k).

Arrays are indexed [k, j, i] (x fastest).  ``dim`` = 2 images have nz = 1
and no z-faces.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.ndimage as ndi
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

# face classification codes (SURVEY §8(c) A5 "neighbour value rule")
DOF, ZERO, GHOST, MIRROR = 0, 1, 2, 3
# cell states
VOID, SOLID, OUT = 0, 1, 2


def _periodic_union(labels: np.ndarray, periodic_axes) -> np.ndarray:
    """Merge connected-component labels across periodic faces (label 0 = bg)."""
    n = int(labels.max())
    if n == 0:
        return labels
    pairs = []
    for ax in periodic_axes:
        a = np.take(labels, 0, axis=ax)
        b = np.take(labels, -1, axis=ax)
        m = (a > 0) & (b > 0)
        pairs.append(np.stack([a[m], b[m]], axis=1))
    if not pairs:
        return labels
    pairs = np.concatenate(pairs, axis=0)
    if pairs.size == 0:
        return labels
    g = sp.coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(n + 1, n + 1))
    _, comp = connected_components(g, directed=False)
    comp = comp.astype(np.int64) + 1
    comp[0] = 0
    out = comp[labels]
    out[labels == 0] = 0
    return out


def clean_void(solid: np.ndarray, periodic_y: bool, periodic_z: bool) -> np.ndarray:
    """D1: keep void components touching x = 0 or x = nx-1 (face connectivity,
    periodic axes wrapped).  Returns the cleaned ``void`` bool array."""
    void = solid == 0
    nz = void.shape[0]
    if nz == 1:
        lab2, _ = ndi.label(void[0])
        per = [0] if periodic_y else []
        lab = _periodic_union(lab2, per)[None]
    else:
        lab, _ = ndi.label(void)
        per = []
        if periodic_z:
            per.append(0)
        if periodic_y:
            per.append(1)
        lab = _periodic_union(lab, per)
    keep = np.union1d(np.unique(lab[..., 0]), np.unique(lab[..., -1]))
    keep = keep[keep > 0]
    return np.isin(lab, keep) & void


@dataclass
class Grid:
    """Void-space MAC grid with canonical DOF numbering."""
    void: np.ndarray            # (nz, ny, nx) bool, after D1
    dim: int
    periodic: tuple             # (py, pz)
    h: float
    face_dof: list = field(default_factory=list)   # per axis a: int64 array, -1 if not DOF
    cell_dof: np.ndarray = None
    n_face: list = field(default_factory=list)
    n_f: int = 0
    n_c: int = 0
    N: int = 0

    @property
    def shape(self):
        return self.void.shape

    @property
    def nx(self):
        return self.void.shape[2]

    @property
    def ny(self):
        return self.void.shape[1]

    @property
    def nz(self):
        return self.void.shape[0]

    # ------------------------------------------------------------------
    def cell_state(self, K, J, I):
        """State of cell (K,J,I) (arrays, any range): VOID/SOLID/OUT.
        x outside the image is OUT (treated as neither void nor solid);
        lateral outside is wrapped if periodic, else SOLID (A4)."""
        K = np.asarray(K, dtype=np.int64)
        J = np.asarray(J, dtype=np.int64)
        I = np.asarray(I, dtype=np.int64)
        nz, ny, nx = self.shape
        st = np.full(np.broadcast(K, J, I).shape, SOLID, dtype=np.int8)
        K, J, I = np.broadcast_arrays(K, J, I)
        Jw = J % ny if self.periodic[0] else J
        Kw = K % nz if (self.periodic[1] and self.dim == 3) else K
        inx = (I >= 0) & (I < nx)
        iny = (Jw >= 0) & (Jw < ny)
        inz = (Kw >= 0) & (Kw < nz)
        ok = inx & iny & inz
        st[ok] = np.where(self.void[Kw[ok], Jw[ok], I[ok]], VOID, SOLID)
        st[(~inx) & iny & inz] = OUT
        return st

    def face_flanks(self, a, K, J, I):
        """Low and high flanking cell coordinates of face (a, K, J, I)."""
        if a == 0:
            return (K, J, I - 1), (K, J, I)
        if a == 1:
            return (K, J - 1, I), (K, J, I)
        return (K - 1, J, I), (K, J, I)

    def classify(self, a, K, J, I):
        """Return (code, dof_index) for faces of orientation a at (K,J,I).

        DOF: both flanks void, or an x-boundary face next to a void cell.
        ZERO: exactly one solid flank (u = 0, wall-normal).
        GHOST: both flanks solid (tangential wall -> ghost value -u_f).
        MIRROR: beyond the inlet/outlet planes (dn u = 0 -> value u_f).
        """
        K = np.asarray(K, dtype=np.int64)
        J = np.asarray(J, dtype=np.int64)
        I = np.asarray(I, dtype=np.int64)
        K, J, I = np.broadcast_arrays(K, J, I)
        nz, ny, nx = self.shape
        code = np.full(K.shape, GHOST, dtype=np.int8)
        idx = np.full(K.shape, -1, dtype=np.int64)
        if a == 0:
            mirror = (I < 0) | (I > nx)
        else:
            mirror = (I < 0) | (I >= nx)
        (k0, j0, i0), (k1, j1, i1) = self.face_flanks(a, K, J, I)
        s0 = self.cell_state(k0, j0, i0)
        s1 = self.cell_state(k1, j1, i1)
        nsolid = (s0 == SOLID).astype(np.int8) + (s1 == SOLID).astype(np.int8)
        isdof = ((s0 == VOID) & (s1 == VOID)) | ((s0 == VOID) & (s1 == OUT)) | ((s0 == OUT) & (s1 == VOID))
        code[nsolid == 1] = ZERO
        code[nsolid == 2] = GHOST
        code[isdof] = DOF
        code[mirror] = MIRROR
        d = isdof & ~mirror
        if d.any():
            Jw = J % ny if self.periodic[0] else J
            Kw = K % nz if (self.periodic[1] and self.dim == 3) else K
            idx[d] = self.face_dof[a][Kw[d], Jw[d], I[d]]
        return code, idx


def build_grid(solid: np.ndarray, dim: int, periodic, h: float, clean: bool = True) -> Grid:
    """Clean the image (D1) and number DOFs canonically."""
    periodic = (bool(periodic[0]), bool(periodic[1]) and dim == 3)
    void = clean_void(solid, *periodic) if clean else (solid == 0)
    if not void.any():
        raise ValueError("non-percolating geometry (PMNS_ENONPERC)")
    g = Grid(void=void, dim=dim, periodic=periodic, h=h)
    nz, ny, nx = void.shape
    shapes = [(nz, ny, nx + 1), (nz, ny, nx), (nz, ny, nx)][:dim]
    off = 0
    g.face_dof = []
    for a in range(dim):
        g.face_dof.append(np.full(shapes[a], -1, dtype=np.int64))
    for a in range(dim):
        K, J, I = np.indices(shapes[a])
        (k0, j0, i0), (k1, j1, i1) = g.face_flanks(a, K, J, I)
        s0 = g.cell_state(k0, j0, i0)
        s1 = g.cell_state(k1, j1, i1)
        isdof = ((s0 == VOID) & (s1 == VOID)) | ((s0 == VOID) & (s1 == OUT)) | ((s0 == OUT) & (s1 == VOID))
        n = int(isdof.sum())
        fd = g.face_dof[a]
        fd[isdof] = np.arange(off, off + n)      # C order == canonical linear id order
        g.n_face.append(n)
        off += n
    g.n_f = off
    cd = np.full(void.shape, -1, dtype=np.int64)
    g.n_c = int(void.sum())
    cd[void] = np.arange(off, off + g.n_c)
    g.cell_dof = cd
    g.N = off + g.n_c
    return g


def dof_positions(g: Grid):
    """For each DOF in canonical order: (type, k, j, i) with type 0..dim-1 for
    faces of that orientation and type 3 for cells."""
    out = np.zeros((g.N, 4), dtype=np.int64)
    for a in range(g.dim):
        m = g.face_dof[a] >= 0
        K, J, I = np.nonzero(m)
        ids = g.face_dof[a][m]
        out[ids] = np.stack([np.full_like(K, a), K, J, I], axis=1)
    K, J, I = np.nonzero(g.cell_dof >= 0)
    ids = g.cell_dof[K, J, I]
    out[ids] = np.stack([np.full_like(K, 3), K, J, I], axis=1)
    return out
