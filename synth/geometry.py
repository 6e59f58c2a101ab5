"""Seeded binary voxel images (1 = solid grain, 0 = void), x-fastest.

Recipes follow SURVEY.md §8(d) "Synthetic inputs"; they stand in for the
paper's images (PD4/GLD4 disk packs, the Granular pack),
which are not available.  Arrays are numpy ``uint8`` of shape (nz, ny, nx)
(C order => x fastest), nz = 1 for 2D images.

Nothing here computes anything of the method (no flow, no decomposition).
"""
from __future__ import annotations

import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CFG_DIR = os.path.join(os.path.dirname(_HERE), "configs")

CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


def config_path(name: str) -> str:
    return os.path.join(_CFG_DIR, f"{name}.json")


def load_config(name: str) -> dict:
    """Read configs/<name>.json (geometry recipe + physical constants)."""
    with open(config_path(name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# Recipes
# --------------------------------------------------------------------------
def disk_pack_2d(n: int, n_disks: int, r_lo: float, r_hi: float, seed: int,
                 max_tries: int = 100000) -> np.ndarray:
    """20 non-overlapping disks in an n x n image (BASELINE config 1).

    Radii r ~ U[r_lo, r_hi] (drawn, then sorted descending); centres uniform in
    [0, n)^2; a centre is rejected if its distance to an accepted centre is
    < r_i + r_j + 1.  A voxel is solid iff its centre (i+.5, j+.5) lies inside
    a disk (disks are clipped at the image edge, not wrapped).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    radii = np.sort(rng.uniform(r_lo, r_hi, size=n_disks))[::-1]
    centres = []
    for r in radii:
        for _ in range(max_tries):
            c = rng.uniform(0.0, float(n), size=2)
            ok = True
            for (c2, r2) in centres:
                if np.hypot(c[0] - c2[0], c[1] - c2[1]) < r + r2 + 1.0:
                    ok = False
                    break
            if ok:
                centres.append((c, r))
                break
    yy, xx = np.meshgrid(np.arange(n) + 0.5, np.arange(n) + 0.5, indexing="ij")
    solid = np.zeros((n, n), dtype=bool)
    for (c, r) in centres:
        solid |= (xx - c[0]) ** 2 + (yy - c[1]) ** 2 <= r * r
    return solid.astype(np.uint8)[None, :, :]


def _stamp_sphere(solid: np.ndarray, c: np.ndarray, r: float) -> int:
    """Set solid voxels whose centres are within r of c (periodic wrap in all
    axes for generation).  Returns the number of voxels newly made solid."""
    nz, ny, nx = solid.shape
    lo = np.floor(c - r - 0.5).astype(np.int64)
    hi = np.ceil(c + r - 0.5).astype(np.int64)
    ix = np.arange(lo[0], hi[0] + 1)
    iy = np.arange(lo[1], hi[1] + 1)
    iz = np.arange(lo[2], hi[2] + 1)
    dz = (iz + 0.5 - c[2])[:, None, None]
    dy = (iy + 0.5 - c[1])[None, :, None]
    dx = (ix + 0.5 - c[0])[None, None, :]
    inside = dx * dx + dy * dy + dz * dz <= r * r
    sub = np.ix_(iz % nz, iy % ny, ix % nx)
    before = solid[sub].copy()
    after = before | inside
    solid[sub] = after
    return int(after.sum() - before.sum())


def boolean_spheres_3d(n: int, phi_target: float, radius_sampler, seed: int) -> np.ndarray:
    """Boolean model: spheres with uniform centres in [0, n)^3 (wrapped
    periodically) added one at a time until porosity <= phi_target."""
    rng = np.random.Generator(np.random.PCG64(seed))
    solid = np.zeros((n, n, n), dtype=bool)
    total = n ** 3
    n_solid = 0
    while (total - n_solid) / total > phi_target:
        c = rng.uniform(0.0, float(n), size=3)
        r = float(radius_sampler(rng))
        n_solid += _stamp_sphere(solid, c, r)
    return solid.astype(np.uint8)


def make_image(cfg: dict) -> np.ndarray:
    """Build the image described by a config dict's ``geometry`` entry."""
    g = cfg["geometry"]
    kind = g["kind"]
    if kind == "crop":   # the corner n^3 (or nx x ny x nz) block of another config's image
        src = make_image(load_config(g["of"]))
        nz, ny, nx = g["shape"]
        return np.ascontiguousarray(src[:nz, :ny, :nx])
    seed = int(g["seed"])
    if kind == "disks2d":
        return disk_pack_2d(g["n"], g["n_disks"], g["r_lo"], g["r_hi"], seed)
    if kind == "spheres3d":
        dist = g["radius"]
        if dist["kind"] == "const":
            rv = float(dist["r"])
            sampler = lambda rng: rv  # noqa: E731
        elif dist["kind"] == "uniform":
            a, b = float(dist["lo"]), float(dist["hi"])
            sampler = lambda rng: rng.uniform(a, b)  # noqa: E731
        elif dist["kind"] == "lognormal":
            mu, sig = float(dist["mu_log"]), float(dist["sigma_log"])
            lo, hi = float(dist["clip_lo"]), float(dist["clip_hi"])
            sampler = lambda rng: min(max(rng.lognormal(mu, sig), lo), hi)  # noqa: E731
        else:
            raise ValueError(dist["kind"])
        return boolean_spheres_3d(g["n"], g["phi"], sampler, seed)
    if kind in FIXTURES:
        return FIXTURES[kind](**{k: v for k, v in g.items() if k not in ("kind", "seed")})
    raise ValueError(kind)


# --------------------------------------------------------------------------
# Small analytic fixtures (tests)
# --------------------------------------------------------------------------
def slit_2d(nx: int, n: int) -> np.ndarray:
    """Straight channel of n void rows between no-slip lateral walls (the
    walls are the image boundary)."""
    return np.zeros((1, n, nx), dtype=np.uint8)


def duct_3d(nx: int, ny: int, nz: int) -> np.ndarray:
    """Rectangular duct: all void, walls are the lateral image boundary."""
    return np.zeros((nz, ny, nx), dtype=np.uint8)


def dumbbell_2d(nx: int = 24, ny: int = 13, neck: int = 3, neck_len: int = 4) -> np.ndarray:
    """Two square pores joined by a thin straight throat (SPEC S:122 fixture)."""
    s = np.ones((ny, nx), dtype=np.uint8)
    half = (nx - neck_len) // 2
    s[1:ny - 1, 0:half] = 0
    s[1:ny - 1, nx - half:nx] = 0
    c = ny // 2
    s[c - neck // 2:c - neck // 2 + neck, half:nx - half] = 0
    return s[None]


def random_blobs(nx: int, ny: int, nz: int, phi: float, r: float, seed: int) -> np.ndarray:
    """Small Boolean-sphere image for parity tests (non-cubic allowed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    solid = np.zeros((nz, ny, nx), dtype=bool)
    total = solid.size
    n_solid = 0
    while (total - n_solid) / total > phi:
        c = rng.uniform(0.0, 1.0, size=3) * np.array([nx, ny, nz], dtype=float)
        if nz == 1:
            c[2] = 0.5
            # 2D: disks
            lo = np.floor(c - r - 0.5).astype(np.int64)
            hi = np.ceil(c + r - 0.5).astype(np.int64)
            ix = np.arange(lo[0], hi[0] + 1)
            iy = np.arange(lo[1], hi[1] + 1)
            dx = (ix + 0.5 - c[0])[None, :]
            dy = (iy + 0.5 - c[1])[:, None]
            inside = dx * dx + dy * dy <= r * r
            sub = np.ix_(iy % ny, ix % nx)
            before = solid[0][sub].copy()
            after = before | inside
            solid[0][sub] = after
            n_solid += int(after.sum() - before.sum())
        else:
            n_solid += _stamp_sphere(solid, c, r)
    return solid.astype(np.uint8)


def gyroid(nx: int, ny: int, nz: int, lx: float = 1.0, ly: float = 1.5, lz: float = 1.0,
           freq: float = 12.0) -> np.ndarray:
    """Gyroid: void where
    sin(f x)cos(f y) + sin(f y)cos(f z) + sin(f z)cos(f x) > 0 at the voxel
    centre, coordinates in the paper's units (domain 1 x 1.5 x 1 cm, f = 12);
    points on the surface are solid."""
    x = (np.arange(nx) + 0.5) / nx * lx
    y = (np.arange(ny) + 0.5) / ny * ly
    z = (np.arange(nz) + 0.5) / nz * lz
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    f = freq
    v = np.sin(f * X) * np.cos(f * Y) + np.sin(f * Y) * np.cos(f * Z) + np.sin(f * Z) * np.cos(f * X)
    return (v <= 0.0).astype(np.uint8)


FIXTURES = {
    "gyroid": gyroid,
    "slit2d": slit_2d,
    "duct3d": duct_3d,
    "dumbbell2d": dumbbell_2d,
    "blobs": random_blobs,
}
