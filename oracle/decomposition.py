"""ORACLE (test infrastructure only) — pore decomposition D2-D10.

PAPER.md §3.2.1 P:156 ("modified watershed segmentation ... on a binary-image
representation of Omega"; details deferred to an external reference),
§3.2.2 P:163-164 (interfaces = thinnest 4/6-connected separating collection;
face partition), P:156 (dual grids = successive morphological dilations of
each interface, N^d = N^c), P:557 (inertia removed on faces within a few
layers of each interface).  The paper does not specify the algorithm, so this
module implements SURVEY.md §8(c) D2-D10 (our specification; DESIGN.md lists
every reading).  PARITY UNPINNED against the paper for the exact labelling:
pinned only by invariants and hand-built fixtures (tests/test_oracle_decomp.py).

D2  D(v) = exact squared Euclidean distance (integer) from void voxel v to the
    nearest solid voxel centre; periodic axes use the minimum image,
    non-periodic lateral walls are a solid layer outside the image, outside
    along x counts as void.
D3  immersion: levels of D in descending order; at each level, grow existing
    basins into unlabelled voxels of that level by synchronous BFS rounds (a
    voxel takes the smallest label among neighbours labelled in previous
    rounds), then leftover components become new basins numbered in order of
    their smallest linear index.
D4  peak P_a = max D over basin a; saddle s_ab = max over face-adjacent pairs
    (u in a, v in b) of min(D(u), D(v)).
D5  merge repeatedly the pair with the smallest key
    sqrt(min(P_a,P_b)) - sqrt(s_ab) < h_m (ties by (min label, max label)),
    the lower-peak basin into the other (tie: larger label into smaller);
    then basins with < n_min voxels (smallest size first, ties by label) into
    the neighbour of largest saddle (ties: smallest label).
D6  relabel basins 0..N^p-1 by smallest linear index.
D7  a voxel with a face neighbour of smaller label b' is an interface voxel of
    pair (a*, b) (a* = its smallest neighbour label); interface voxels leave
    their basin.  Interfaces = 26-connected (8 in 2D) components of each
    pair's voxels, numbered by (a*, b, smallest linear index).  A basin left
    empty is merged (D5 small-basin rule) and D6-D7 are redone.
D8  dual j = geodesic (face-connected, periodic, within void) dilation of
    interface j by k_d steps.
D9  mask band: DOF faces with a flanking cell at geodesic distance <= band
    from an interface cell.
D10 a DOF face flanked by >= 1 cell of primary i belongs to i; otherwise it
    is an interface f-face owned by its lowest-id flanking interface cell's
    interface.
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass

import numpy as np
import scipy.ndimage as ndi
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .grid import Grid, VOID, OUT, DOF, ZERO, GHOST

BIG = np.int64(1) << 40


# ----------------------------------------------------------------------------
# voxel graph helpers
# ----------------------------------------------------------------------------
def face_neighbours(g: Grid):
    """Flat indices of the 2*dim face neighbours of every voxel (-1 = none,
    i.e. outside a non-periodic boundary).  Shape (nvox, 2*dim)."""
    nz, ny, nx = g.shape
    K, J, I = np.indices(g.shape).reshape(3, -1)
    out = []
    for b in range(g.dim):
        for o in (-1, 1):
            k, j, i = K.copy(), J.copy(), I.copy()
            if b == 0:
                i = i + o
                ok = (i >= 0) & (i < nx)
            elif b == 1:
                j = j + o
                if g.periodic[0]:
                    j %= ny
                ok = (j >= 0) & (j < ny)
            else:
                k = k + o
                if g.periodic[1]:
                    k %= nz
                ok = (k >= 0) & (k < nz)
            f = np.where(ok, (k * ny + np.where(ok, j, 0)) * nx + np.where(ok, i, 0), -1)
            out.append(f)
    return np.stack(out, axis=1)


def box_neighbours(g: Grid, flat):
    """26- (8 in 2D) neighbours of the given flat voxels, periodic-aware,
    -1 outside.  Shape (len(flat), 26 or 8)."""
    nz, ny, nx = g.shape
    k0, j0, i0 = np.unravel_index(flat, g.shape)
    offs = []
    rz = (-1, 0, 1) if g.dim == 3 else (0,)
    for dk in rz:
        for dj in (-1, 0, 1):
            for di in (-1, 0, 1):
                if dk == 0 and dj == 0 and di == 0:
                    continue
                offs.append((dk, dj, di))
    out = np.empty((len(flat), len(offs)), dtype=np.int64)
    for c, (dk, dj, di) in enumerate(offs):
        k, j, i = k0 + dk, j0 + dj, i0 + di
        if g.periodic[0]:
            j = j % ny
        if g.periodic[1]:
            k = k % nz
        ok = (i >= 0) & (i < nx) & (j >= 0) & (j < ny) & (k >= 0) & (k < nz)
        out[:, c] = np.where(ok, (np.where(ok, k, 0) * ny + np.where(ok, j, 0)) * nx + np.where(ok, i, 0), -1)
    return out


def squared_edt(g: Grid) -> np.ndarray:
    """D2: exact integer squared EDT of void voxels (0 on solid)."""
    void = g.void
    nz, ny, nx = void.shape
    P = 8
    while True:
        pads = []
        modes = []
        arr = void.astype(np.uint8)
        # lateral axes: z (axis 0, 3D only), y (axis 1)
        padw = [(0, 0), (0, 0), (0, 0)]
        if g.dim == 3:
            padw[0] = (P, P) if g.periodic[1] else (1, 1)
        padw[1] = (P, P) if g.periodic[0] else (1, 1)
        a = arr
        # periodic axes: wrap; non-periodic lateral: solid layer (0)
        for ax in (0, 1):
            if padw[ax] == (0, 0):
                continue
            per = g.periodic[1] if ax == 0 else g.periodic[0]
            w = [(0, 0)] * 3
            w[ax] = padw[ax]
            a = np.pad(a, w, mode="wrap") if per else np.pad(a, w, mode="constant", constant_values=0)
        if not (a == 0).any():
            D = np.where(void, BIG, 0).astype(np.int64)
            return D
        _, inds = ndi.distance_transform_edt(a, return_indices=True)
        oz, oy = padw[0][0], padw[1][0]
        Kp, Jp, Ip = np.indices(a.shape)
        d2 = ((Kp - inds[0]) ** 2 + (Jp - inds[1]) ** 2 + (Ip - inds[2]) ** 2).astype(np.int64)
        D = d2[oz:oz + nz, oy:oy + ny, :]
        D = np.where(void, D, 0)
        need = False
        if g.periodic[0] and D.max() > P * P:
            need = True
        if g.dim == 3 and g.periodic[1] and D.max() > P * P:
            need = True
        if not need:
            return D.astype(np.int64)
        P *= 2


# ----------------------------------------------------------------------------
@dataclass
class Decomposition:
    label: np.ndarray          # (nz,ny,nx) int64: primary id >= 0, -1 otherwise (solid or interface)
    iface: np.ndarray          # (nz,ny,nx) int64: interface id >= 0, -1 otherwise
    basin: np.ndarray          # (nz,ny,nx) int64: basin id before interface removal (-1 solid)
    n_p: int
    n_c: int
    dual_cells: list           # per dual j: sorted flat voxel indices
    mask_cells: np.ndarray     # (nz,ny,nx) bool: within band of an interface cell
    n_raw_basins: int = 0


def watershed(g: Grid, D: np.ndarray, nbr: np.ndarray):
    """D3: level-synchronous immersion.  Returns raw basin labels (flat)."""
    void = g.void.reshape(-1)
    Df = D.reshape(-1)
    nv = void.size
    label = np.full(nv, -1, dtype=np.int64)
    vox = np.nonzero(void)[0]
    # void-only neighbour table
    nb_void = np.where(nbr >= 0, nbr, 0)
    nb_ok = (nbr >= 0) & void[nb_void]
    order = np.argsort(-Df[vox], kind="stable")
    vs = vox[order]
    dv = Df[vs]
    bounds = np.nonzero(np.diff(dv))[0] + 1
    groups = np.split(vs, bounds)
    nlab = 0
    INF = np.iinfo(np.int64).max
    for grp in groups:
        remaining = np.sort(grp)
        while remaining.size:
            nbs = nbr[remaining]
            okm = nb_ok[remaining]
            nl = np.where(okm, label[np.where(okm, nbs, 0)], -1)
            nl = np.where(nl >= 0, nl, INF)
            m = nl.min(axis=1)
            grow = m < INF
            if not grow.any():
                break
            label[remaining[grow]] = m[grow]
            remaining = remaining[~grow]
        if remaining.size:
            # connected components among the leftover voxels of this level
            pos = np.full(nv, -1, dtype=np.int64)
            pos[remaining] = np.arange(remaining.size)
            nbs = nbr[remaining]
            okm = nb_ok[remaining]
            pn = np.where(okm, pos[np.where(okm, nbs, 0)], -1)
            r, c = np.nonzero(pn >= 0)
            gr = sp.coo_matrix((np.ones(len(r)), (r, pn[r, c])), shape=(remaining.size,) * 2)
            nc, comp = connected_components(gr, directed=False)
            # number components by smallest linear index (remaining is sorted)
            first = np.full(nc, -1, dtype=np.int64)
            seen = np.zeros(nc, dtype=bool)
            rank = 0
            for idx in range(remaining.size):
                cc = comp[idx]
                if not seen[cc]:
                    seen[cc] = True
                    first[cc] = rank
                    rank += 1
            label[remaining] = nlab + first[comp]
            nlab += nc
    return label, nlab


def _saddles(label, Df, nbr, void):
    """D4: peaks and saddles of a labelling (flat arrays)."""
    vox = np.nonzero(void)[0]
    res = {}
    for c in range(nbr.shape[1]):
        nb = nbr[vox, c]
        ok = nb >= 0
        u = vox[ok]
        v = nb[ok]
        ok2 = void[v]
        u, v = u[ok2], v[ok2]
        la, lb = label[u], label[v]
        m = la < lb
        u, v, la, lb = u[m], v[m], la[m], lb[m]
        val = np.minimum(Df[u], Df[v])
        if la.size == 0:
            continue
        key = la * (label.max() + 1) + lb
        o = np.lexsort((val, key))
        key, val = key[o], val[o]
        last = np.r_[np.nonzero(np.diff(key))[0], key.size - 1]
        for k_, v_ in zip(key[last], val[last]):
            k_ = int(k_)
            if res.get(k_, -1) < v_:
                res[k_] = int(v_)
    L = int(label.max()) + 1
    S = {}
    for k_, v_ in res.items():
        a, b = divmod(k_, L)
        S.setdefault(a, {})[b] = v_
        S.setdefault(b, {})[a] = v_
    return S


def merge_basins(label, nlab, Df, nbr, void, h_m, n_min):
    """D4-D5 on raw labels; returns final labels (flat, relabelled D6)."""
    vox = np.nonzero(void)[0]
    P = np.full(nlab, -1, dtype=np.int64)
    np.maximum.at(P, label[vox], Df[vox])
    size = np.bincount(label[vox], minlength=nlab).astype(np.int64)
    S = _saddles(label, Df, nbr, void)
    for a in range(nlab):
        S.setdefault(a, {})
    parent = np.arange(nlab)
    alive = np.ones(nlab, dtype=bool)
    P = [int(x) for x in P]
    size = [int(x) for x in size]

    def key(a, b):
        return math.sqrt(float(min(P[a], P[b]))) - math.sqrt(float(S[a][b]))

    def merge(src, dst):
        parent[src] = dst
        alive[src] = False
        P[dst] = max(P[dst], P[src])
        size[dst] += size[src]
        for c, s in S[src].items():
            if c == dst:
                continue
            cur = S[dst].get(c, -1)
            if s > cur:
                S[dst][c] = s
                S[c][dst] = s
            del S[c][src]
        del S[dst][src]
        S[src] = {}

    heap = []
    for a in range(nlab):
        for b in S[a]:
            if a < b:
                heap.append((key(a, b), a, b))
    heapq.heapify(heap)
    while heap:
        k, a, b = heapq.heappop(heap)
        if not (alive[a] and alive[b] and b in S[a]):
            continue
        if key(a, b) != k:
            continue
        if not k < h_m:
            break
        if P[a] < P[b]:
            src, dst = a, b
        elif P[b] < P[a]:
            src, dst = b, a
        else:
            src, dst = max(a, b), min(a, b)
        merge(src, dst)
        for c in S[dst]:
            heapq.heappush(heap, (key(dst, c), min(dst, c), max(dst, c)))
    # small basins
    heap = [(size[a], a) for a in range(nlab) if alive[a] and size[a] < n_min]
    heapq.heapify(heap)
    while heap:
        s, a = heapq.heappop(heap)
        if not alive[a] or size[a] != s or size[a] >= n_min:
            continue
        if not S[a]:
            continue
        b = min(S[a].items(), key=lambda kv: (-kv[1], kv[0]))[0]
        merge(a, b)
        if size[b] < n_min:
            heapq.heappush(heap, (size[b], b))
    # resolve to representatives
    root = parent.copy()
    for _ in range(64):
        nr = root[root]
        if np.array_equal(nr, root):
            break
        root = nr
    lab = np.full(label.shape, -1, dtype=np.int64)
    lab[vox] = root[label[vox]]
    return relabel(lab, vox)


def relabel(lab, vox):
    """D6: renumber labels 0.. by smallest linear index."""
    out = np.full(lab.shape, -1, dtype=np.int64)
    vals = lab[vox]
    _, first_idx = np.unique(vals, return_index=True)
    order = np.argsort(vox[first_idx])
    uniq = vals[first_idx][order]
    mp = {int(u): i for i, u in enumerate(uniq)}
    lut = np.full(int(vals.max()) + 1, -1, dtype=np.int64)
    for u, i in mp.items():
        lut[u] = i
    out[vox] = lut[vals]
    return out


def interfaces(g: Grid, lab, nbr, void):
    """D7: interface voxels and their ids.  Returns (iface flat array, n_c,
    pair list)."""
    vox = np.nonzero(void)[0]
    nb = nbr[vox]
    okm = (nb >= 0) & void[np.where(nb >= 0, nb, 0)]
    nl = np.where(okm, lab[np.where(okm, nb, 0)], np.iinfo(np.int64).max)
    mn = nl.min(axis=1)
    cand = mn < lab[vox]
    cv = vox[cand]
    pa = mn[cand]
    pb = lab[cv]
    iface = np.full(lab.shape, -1, dtype=np.int64)
    if cv.size == 0:
        return iface, 0
    # 26/8-connected components within each pair
    pos = np.full(lab.shape, -1, dtype=np.int64)
    pos[cv] = np.arange(cv.size)
    bn = box_neighbours(g, cv)
    pn = np.where(bn >= 0, pos[np.where(bn >= 0, bn, 0)], -1)
    r, c = np.nonzero(pn >= 0)
    q = pn[r, c]
    same = (pa[r] == pa[q]) & (pb[r] == pb[q])
    gr = sp.coo_matrix((np.ones(same.sum()), (r[same], q[same])), shape=(cv.size,) * 2)
    ncomp, comp = connected_components(gr, directed=False)
    # order components by (a*, b, smallest linear index); cv is sorted ascending
    first = np.full(ncomp, -1, dtype=np.int64)
    for idx in range(cv.size - 1, -1, -1):
        first[comp[idx]] = cv[idx]
    ca = np.zeros(ncomp, dtype=np.int64)
    cb = np.zeros(ncomp, dtype=np.int64)
    ca[comp] = pa
    cb[comp] = pb
    order = np.lexsort((first, cb, ca))
    rank = np.empty(ncomp, dtype=np.int64)
    rank[order] = np.arange(ncomp)
    iface[cv] = rank[comp]
    return iface, ncomp


def geodesic_dilate(seed_flat, nbr, void, steps):
    cur = np.unique(seed_flat)
    front = cur
    for _ in range(steps):
        nb = nbr[front].reshape(-1)
        nb = nb[nb >= 0]
        nb = nb[void[nb]]
        new = np.setdiff1d(np.unique(nb), cur, assume_unique=True)
        if new.size == 0:
            break
        cur = np.union1d(cur, new)
        front = new
    return cur


def floating_faces(g: Grid, prim_flat, iface_flat):
    """D7b test: bool per face DOF.  For each primary and orientation a, the
    primary's a-faces form a graph (edges: same-orientation face neighbours
    f +- e_b owned by the same primary).  A face is *anchored* if one of its
    2*dim neighbour positions is a wall face (ZERO or GHOST).  Faces of a
    component without an anchored face are *floating*: after the fold of
    Eq. reduce_1/2 their viscous rows see only themselves, so the folded block
    Abar^{p_i}_{p_i} has a zero-resistance mode (singular).  Reading D7b."""
    fl = face_flank_cells(g)
    pf = np.full(g.n_f, -1, dtype=np.int64)
    for s_ in range(2):
        f = fl[:, s_]
        ok = f >= 0
        lp = np.where(ok, prim_flat[np.where(ok, f, 0)], -1)
        pf = np.where(lp >= 0, lp, pf)
    anch = np.zeros(g.n_f, dtype=bool)
    rows, cols = [], []
    for a in range(g.dim):
        fd = g.face_dof[a]
        K, J, I = np.nonzero(fd >= 0)
        ids = fd[K, J, I]
        for b in range(g.dim):
            for o in (-1, 1):
                pos = [K, J, I]
                ax = 2 - b
                pos[ax] = pos[ax] + o
                code, idx = g.classify(a, *pos)
                anch[ids] |= (code == ZERO) | (code == GHOST)
                m = code == DOF
                rows.append(ids[m]); cols.append(idx[m])
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    keep = (pf[r] >= 0) & (pf[r] == pf[c])
    G = sp.coo_matrix((np.ones(keep.sum()), (r[keep], c[keep])), shape=(g.n_f, g.n_f))
    ncomp, comp = connected_components(G, directed=False)
    ca = np.zeros(ncomp, dtype=bool)
    np.logical_or.at(ca, comp, anch)
    return (pf >= 0) & (~ca[comp]), fl


def repair_floating(g: Grid, lab, iface, nbr, void):
    """D7b: while floating faces exist, every primary cell flanking one joins
    the interface with the smallest id among interface cells in its 26- (8-)
    neighbourhood (synchronous rounds; cells with none wait a round)."""
    iface = iface.copy()
    while True:
        prim = np.where(iface >= 0, -1, lab)
        flt, fl = floating_faces(g, prim, iface)
        if not flt.any():
            return iface, True
        cells = np.unique(fl[flt].reshape(-1))
        cells = cells[cells >= 0]
        cells = cells[prim[cells] >= 0]
        bn = box_neighbours(g, cells)
        nid = np.where(bn >= 0, iface[np.where(bn >= 0, bn, 0)], -1)
        nid = np.where(nid >= 0, nid, np.iinfo(np.int64).max)
        mn = nid.min(axis=1)
        ok = mn < np.iinfo(np.int64).max
        if not ok.any():
            raise RuntimeError("D7b: floating faces with no adjacent interface")
        iface[cells[ok]] = mn[ok]


def decompose(g: Grid, h_m: float, n_min: int, dual_layers: int = 2, mask_band: int = 2) -> Decomposition:
    """Run D2-D9 (D10 face labels are derived in ``face_owner``)."""
    void = g.void.reshape(-1)
    nbr = face_neighbours(g)
    D = squared_edt(g).reshape(-1)
    raw, nraw = watershed(g, D.reshape(g.shape), nbr)
    lab = merge_basins(raw, nraw, D, nbr, void, h_m, n_min)
    vox = np.nonzero(void)[0]

    def first_empty(iface_):
        prim_ = np.where(iface_ >= 0, -1, lab)
        cnt = np.bincount(prim_[vox][prim_[vox] >= 0], minlength=int(lab.max()) + 1)
        e = np.nonzero(cnt == 0)[0]
        return int(e[0]) if e.size else -1

    while True:
        iface, n_c = interfaces(g, lab, nbr, void)           # D7
        a = first_empty(iface)
        if a < 0:
            iface, _ = repair_floating(g, lab, iface, nbr, void)   # D7b
            a = first_empty(iface)
            if a < 0:
                break
        # a basin left empty: merge it by the D5 small-basin rule, redo D6-D7
        S = _saddles(lab, D, nbr, void)
        b = min(S[a].items(), key=lambda kv: (-kv[1], kv[0]))[0]
        lab = relabel(np.where(lab == a, b, lab), vox)
    n_p = int(lab.max()) + 1
    prim = np.where(iface >= 0, -1, lab)
    # D8 duals
    duals = []
    for j in range(n_c):
        seed = np.nonzero(iface == j)[0]
        duals.append(geodesic_dilate(seed, nbr, void, dual_layers))
    # D9 band: multi-source BFS distance from interface cells
    dist = np.full(void.size, -1, dtype=np.int64)
    front = np.nonzero(iface >= 0)[0]
    dist[front] = 0
    for d in range(1, mask_band + 1):
        nb = nbr[front].reshape(-1)
        nb = nb[nb >= 0]
        nb = np.unique(nb[void[nb]])
        nb = nb[dist[nb] < 0]
        dist[nb] = d
        front = nb
    mask_cells = (dist >= 0).reshape(g.shape)
    return Decomposition(label=prim.reshape(g.shape), iface=iface.reshape(g.shape),
                         basin=lab.reshape(g.shape), n_p=n_p, n_c=n_c, dual_cells=duals,
                         mask_cells=mask_cells, n_raw_basins=nraw)


# ----------------------------------------------------------------------------
# D10 and unknown sets
# ----------------------------------------------------------------------------
def face_flank_cells(g: Grid):
    """For every face DOF (canonical id 0..n_f-1): flat index of its two flank
    cells (-1 if outside/solid).  Cached on the grid."""
    cached = getattr(g, "_flank_cache", None)
    if cached is not None:
        return cached
    nz, ny, nx = g.shape
    out = np.full((g.n_f, 2), -1, dtype=np.int64)
    for a in range(g.dim):
        fd = g.face_dof[a]
        K, J, I = np.nonzero(fd >= 0)
        ids = fd[K, J, I]
        for s, cell in enumerate(g.face_flanks(a, K, J, I)):
            k, j, i = cell
            st = g.cell_state(k, j, i)
            m = st == VOID
            kk, jj = k.copy(), j.copy()
            if g.periodic[0]:
                jj = jj % ny
            if g.periodic[1]:
                kk = kk % nz
            out[ids[m], s] = (kk[m] * ny + jj[m]) * nx + i[m]
    g._flank_cache = out
    return out


def face_owner(g: Grid, dec: Decomposition):
    """D10: per face DOF: (primary id or -1, interface id or -1)."""
    fl = face_flank_cells(g)
    lab = dec.label.reshape(-1)
    ifc = dec.iface.reshape(-1)
    p = np.full(g.n_f, -1, dtype=np.int64)
    c = np.full(g.n_f, -1, dtype=np.int64)
    big = np.iinfo(np.int64).max
    for s in range(2):
        f = fl[:, s]
        ok = f >= 0
        lp = np.where(ok, lab[np.where(ok, f, 0)], -1)
        p = np.where(lp >= 0, lp, p)
    ci = np.full(g.n_f, big, dtype=np.int64)
    for s in range(2):
        f = fl[:, s]
        ok = f >= 0
        li = np.where(ok, ifc[np.where(ok, f, 0)], -1)
        ci = np.where((li >= 0) & (li < ci), li, ci)
    c = np.where((p < 0) & (ci < big), ci, -1)
    return p, c, fl


def w_order(g: Grid, dec: Decomposition):
    """The permutation W (Eq. permute) as an index array:
    ``perm[w] = canonical index`` with unknowns grouped by primary grid
    (cells and faces, canonical order inside), then interface cells (by
    interface), then interface f-faces (by owning interface).  Also returns
    segment boundaries."""
    p, c, _ = face_owner(g, dec)
    nf = g.n_f
    cell_ids = g.cell_dof.reshape(-1)
    lab = dec.label.reshape(-1)
    ifc = dec.iface.reshape(-1)
    vox = np.nonzero(g.void.reshape(-1))[0]
    # per unknown: group key
    grp = np.empty(g.N, dtype=np.int64)
    grp[:nf] = np.where(p >= 0, p, dec.n_p + dec.n_c + c)
    cg = np.where(lab[vox] >= 0, lab[vox], dec.n_p + ifc[vox])
    grp[cell_ids[vox]] = cg
    perm = np.lexsort((np.arange(g.N), grp))
    counts = np.bincount(grp, minlength=dec.n_p + 2 * dec.n_c)
    seg = np.concatenate([[0], np.cumsum(counts)])
    return perm, seg


def subdomain_unknowns(g: Grid, cells_flat):
    """Unknown set of a subdomain (P:522-537 reading D10): its cells plus every
    DOF face with >= 1 flanking cell in it.  Canonical indices, sorted."""
    fl = face_flank_cells(g)
    inset = np.zeros(g.void.size, dtype=bool)
    inset[cells_flat] = True
    m = np.zeros(g.n_f, dtype=bool)
    for s in range(2):
        f = fl[:, s]
        ok = f >= 0
        m |= ok & inset[np.where(ok, f, 0)]
    faces = np.nonzero(m)[0]
    cells = g.cell_dof.reshape(-1)[cells_flat]
    return np.sort(np.concatenate([faces, cells]))


def masked_faces(g: Grid, dec: Decomposition):
    """D9: bool per face DOF."""
    fl = face_flank_cells(g)
    mc = dec.mask_cells.reshape(-1)
    m = np.zeros(g.n_f, dtype=bool)
    for s in range(2):
        f = fl[:, s]
        ok = f >= 0
        m |= ok & mc[np.where(ok, f, 0)]
    return m
