"""Pins of the oracle decomposition (D1-D10).  The paper does not specify the
watershed, so these are invariants, brute force and fixtures only —
"parity unpinned" against the paper for the exact labelling."""
import itertools

import numpy as np
import pytest

from synth.geometry import slit_2d, random_blobs, dumbbell_2d, load_config, make_image
from oracle.grid import build_grid, clean_void
from oracle.decomposition import (decompose, squared_edt, face_owner, w_order, floating_faces,
                                  face_neighbours, subdomain_unknowns, masked_faces)

H = 1e-5


def _brute_edt(g):
    nz, ny, nx = g.shape
    sol = []
    for k, j, i in itertools.product(range(nz), range(ny), range(nx)):
        if not g.void[k, j, i]:
            sol.append((k, j, i))
    # lateral wall layers (non-periodic) are solid
    ext = []
    if not g.periodic[0]:
        for k, i in itertools.product(range(nz), range(-3, nx + 3)):
            ext += [(k, -1, i), (k, ny, i)]
    if g.dim == 3 and not g.periodic[1]:
        for j, i in itertools.product(range(-1, ny + 1), range(-3, nx + 3)):
            ext += [(-1, j, i), (nz, j, i)]
    S = np.array(sol + ext, dtype=np.int64).reshape(-1, 3)
    D = np.zeros(g.shape, dtype=np.int64)
    for k, j, i in itertools.product(range(nz), range(ny), range(nx)):
        if not g.void[k, j, i]:
            continue
        d = S - np.array([k, j, i])
        if g.periodic[0]:
            d[:, 1] = np.minimum(np.abs(d[:, 1]), ny - np.abs(d[:, 1]))
        if g.dim == 3 and g.periodic[1]:
            d[:, 0] = np.minimum(np.abs(d[:, 0]), nz - np.abs(d[:, 0]))
        D[k, j, i] = (d ** 2).sum(axis=1).min()
    return D


@pytest.mark.parametrize("dim,per,seed", [(2, (False, False), 1), (2, (True, False), 2),
                                          (3, (True, True), 3), (3, (False, False), 4), (3, (True, False), 5)])
def test_edt_brute_force(dim, per, seed):
    if dim == 2:
        img = random_blobs(17, 13, 1, 0.7, 2.0, seed)
    else:
        img = random_blobs(9, 8, 7, 0.7, 1.7, seed)
    g = build_grid(img, dim, per, H, clean=False)
    assert np.array_equal(squared_edt(g), _brute_edt(g))


def test_cleanup_removes_isolated_void():
    img = np.ones((1, 7, 9), dtype=np.uint8)
    img[0, 3, :] = 0          # channel
    img[0, 1, 4] = 0          # isolated pocket
    v = clean_void(img, False, False)
    assert v[0, 3].all() and not v[0, 1, 4]
    img2 = np.ones((1, 5, 5), dtype=np.uint8)
    img2[0, 2, 2] = 0
    with pytest.raises(ValueError):
        build_grid(img2, 2, (False, False), H)


def test_fixtures_channel_and_dumbbell():
    """Straight channel: N^p = 1, N^c = 0; dumbbell: N^p = 2, N^c = 1."""
    g = build_grid(slit_2d(12, 5), 2, (False, False), H)
    dec = decompose(g, 1.0, 3)
    assert (dec.n_p, dec.n_c) == (1, 0)
    g = build_grid(dumbbell_2d(24, 13, 3, 4), 2, (False, False), H)
    dec = decompose(g, 0.0, 1)
    assert (dec.n_p, dec.n_c) == (2, 1)
    # the interface sits in the throat: its cells have x inside the neck
    k, j, i = np.nonzero(dec.iface == 0)
    assert i.min() >= 8 and i.max() <= 15


@pytest.mark.parametrize("case", ["blob2", "blob3", "cfg1"])
def test_decomposition_invariants(case):
    if case == "blob2":
        g = build_grid(random_blobs(40, 24, 1, 0.55, 3.0, 9), 2, (False, False), H)
        dec = decompose(g, 1.0, 5, 1, 2)
    elif case == "blob3":
        g = build_grid(random_blobs(20, 16, 16, 0.4, 2.5, 9), 3, (True, True), H)
        dec = decompose(g, 0.5, 10, 1, 2)
    else:
        cfg = load_config("cfg1")
        g = build_grid(make_image(cfg), 2, (False, False), H)
        dec = decompose(g, cfg["ws_merge_h"], cfg["ws_min_cells"], cfg["dual_layers"], cfg["mask_band"])
    void = g.void.reshape(-1)
    lab = dec.label.reshape(-1)
    ifc = dec.iface.reshape(-1)
    # every void voxel is exactly one of primary / interface; solid is neither
    assert np.all((lab >= 0) ^ (ifc >= 0) == void)
    assert np.all(lab[~void] == -1) and np.all(ifc[~void] == -1)
    # separator: no face-adjacent pair of cells in different primaries
    nbr = face_neighbours(g)
    for c in range(nbr.shape[1]):
        nb = nbr[:, c]
        ok = (nb >= 0) & (lab >= 0)
        other = np.where(ok, lab[np.where(ok, nb, 0)], -1)
        assert np.all((other < 0) | (other == lab) | ~ok)
    # N^d = N^c, duals contain their interfaces
    assert len(dec.dual_cells) == dec.n_c
    for j, d in enumerate(dec.dual_cells):
        assert set(np.nonzero(ifc == j)[0]) <= set(d)
    # every primary non-empty, every interface non-empty
    assert np.all(np.bincount(lab[lab >= 0], minlength=dec.n_p) > 0)
    assert np.all(np.bincount(ifc[ifc >= 0], minlength=dec.n_c) > 0)
    # D10: every face DOF has exactly one owner
    p, c, _ = face_owner(g, dec)
    assert np.all((p >= 0) ^ (c >= 0))
    # D7b: no floating faces
    flt, _ = floating_faces(g, lab, ifc)
    assert not flt.any()
    # W is a permutation with contiguous primary segments equal to the
    # subdomain unknown sets
    perm, seg = w_order(g, dec)
    assert np.array_equal(np.sort(perm), np.arange(g.N))
    for i in range(dec.n_p):
        cells = np.nonzero(lab == i)[0]
        assert np.array_equal(np.sort(perm[seg[i]:seg[i + 1]]), subdomain_unknowns(g, cells))
    # mask covers every face touching an interface cell
    m = masked_faces(g, dec)
    fl = face_owner(g, dec)[2]
    touch = np.zeros(g.n_f, dtype=bool)
    for s in range(2):
        f = fl[:, s]
        ok = f >= 0
        touch |= ok & (ifc[np.where(ok, f, 0)] >= 0)
    assert np.all(m[touch])
