"""Bit-exact parity of the library's host setup (C++: clean-up, EDT, watershed,
merge, interfaces, D7b, duals, mask, W order) with the oracle (readings D1-D10).
Runs on CPU through a host-only pmns context (device = -1)."""
import numpy as np
import pytest

from synth.geometry import load_config, make_image, random_blobs, dumbbell_2d, slit_2d
from oracle.grid import build_grid
from oracle.decomposition import decompose, w_order, masked_faces


def _cfg(dim, per, hm, nmin, kd=1, band=2):
    return dict(dim=dim, periodic=list(per), h=1e-5, rho=1000.0, mu=1e-3, body_force=[0, 0, 0],
                p_in=1.0, p_out=0.0, dt=0.0, ws_merge_h=hm, ws_min_cells=nmin, dual_layers=kd, mask_band=band)


CASES = {
    "cfg1": lambda: (load_config("cfg1"), make_image(load_config("cfg1"))),
    "cfg2": lambda: (load_config("cfg2"), make_image(load_config("cfg2"))),
    "blob2d": lambda: (_cfg(2, (False, False), 1.0, 5), random_blobs(40, 24, 1, 0.55, 3.0, 9)),
    "blob2d_per": lambda: (_cfg(2, (True, False), 0.5, 3, 2, 3), random_blobs(33, 20, 1, 0.5, 2.5, 4)),
    "blob3d": lambda: (_cfg(3, (True, True), 0.5, 10), random_blobs(20, 16, 16, 0.4, 2.5, 9)),
    "blob3d_walls": lambda: (_cfg(3, (False, False), 0.25, 4, 2, 2), random_blobs(15, 13, 11, 0.5, 2.2, 6)),
    "blob3d_mixed": lambda: (_cfg(3, (True, False), 0.75, 6), random_blobs(18, 12, 14, 0.45, 2.4, 8)),
    "dumbbell": lambda: (_cfg(2, (False, False), 0.0, 1), dumbbell_2d(24, 13, 3, 4)),
    "slit": lambda: (_cfg(2, (False, False), 1.0, 3), slit_2d(12, 5)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_host_setup_bit_exact(name):
    pytest.importorskip("ctypes")
    from paper_2510_22077_b200 import Solver
    cfg, img = CASES[name]()
    s = Solver(cfg, img, device=-1)
    L = s.export_layout()
    q = s.query()
    g = build_grid(img, cfg["dim"], cfg["periodic"], cfg["h"])
    dec = decompose(g, cfg["ws_merge_h"], cfg["ws_min_cells"], cfg["dual_layers"], cfg["mask_band"])
    assert (q["n_c"], q["n_f"], q["N"]) == (g.n_c, g.n_f, g.N)
    assert (q["n_p"], q["n_iface"]) == (dec.n_p, dec.n_c)
    assert q["raw_basins"] == dec.n_raw_basins
    assert np.array_equal(L["label"], dec.label.reshape(-1).astype(np.int32))
    assert np.array_equal(L["iface"], dec.iface.reshape(-1).astype(np.int32))
    perm, seg = w_order(g, dec)
    assert np.array_equal(L["perm"], perm)
    assert len(L["duals"]) == len(dec.dual_cells)
    for a, b in zip(L["duals"], dec.dual_cells):
        assert np.array_equal(a, b)
    assert np.array_equal(L["mask"], masked_faces(g, dec))
    s.close()
