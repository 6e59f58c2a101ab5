"""Calibrate the drive of a config too large for the oracle to decompose at full size (config 5): the oracle's Stokes
solve on a seeded-corner crop gives Re per unit pressure gradient (Re is linear in G at Stokes; the same procedure as
scripts/calibrate.py --crop), and the full-size statistics (N, N^p, N^c) come from a host-only library context
(pmns_create with device = -1: the integer set-up is bit-exact against the oracle, tests/test_setup_parity.py).
Writes configs/<name>.json.  Usage: python scripts/calibrate_big.py cfg5 96 0.5 50"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from synth.geometry import load_config, make_image, config_path  # noqa: E402
from oracle.grid import build_grid  # noqa: E402
from oracle.mac import Mac  # noqa: E402
from oracle.decomposition import decompose  # noqa: E402
from oracle.newton import build_gplmm, newton  # noqa: E402
from scripts.calibrate import geometry_stats, reynolds  # noqa: E402

name, crop, hm, nmin = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
cfg = load_config(name)
t0 = time.time()
img = make_image(cfg)
print(f"image {img.shape} in {time.time() - t0:.1f} s, phi {1.0 - img.mean():.4f}", flush=True)
sub = np.ascontiguousarray(img[:crop, :crop, :crop])
g = build_grid(sub, cfg["dim"], cfg["periodic"], cfg["h"])
phi, Vs, Aw = geometry_stats(g, sub)
dec = decompose(g, hm, nmin, cfg["dual_layers"], cfg["mask_band"])
mac = Mac(g, cfg["rho"], cfg["mu"], p_in=1.0, p_out=0.0)
MS = build_gplmm(mac, dec, None)
x = newton(mac, MS, np.zeros(g.N), None, max_newton=1)
Re1, UD1 = reynolds(g, mac, x, phi, Vs, Aw)
G1 = 1.0 / ((g.nx + 1) * g.h)
G = cfg["Re_target"] / Re1 * G1
print(f"crop {crop}^3: N {g.N}, phi {phi:.4f}, Re per unit G {Re1 / G1:.4e} ({time.time() - t0:.1f} s)", flush=True)
cfg["p_in"] = G * (img.shape[2] + 1) * cfg["h"]
cfg["p_out"] = 0.0
cfg["body_force"] = [0.0, 0.0, 0.0]
cfg["ws_merge_h"] = hm
cfg["ws_min_cells"] = nmin
cfg["calibrated"] = True
cfg["calibration"] = dict(kind="crop", crop=crop, crop_N=int(g.N), crop_phi=float(phi),
                          crop_Re_per_unit_G=float(Re1 / G1), G=float(G),
                          script="scripts/calibrate_big.py (oracle/ for the crop solve; library host set-up for the "
                                 "full-size counts)")
from paper_2510_22077_b200 import Solver  # noqa: E402
t1 = time.time()
s = Solver(cfg, img, device=-1)
q = s.query()
cfg["stats"] = dict(N=int(q["N"]), n_c=int(q["n_c"]), n_f=int(q["n_f"]), phi=float(1.0 - img.mean()),
                    N_p=int(q["n_p"]), N_c=int(q["n_iface"]), host_setup_s=round(time.time() - t1, 1))
s.close()
with open(config_path(name), "w") as f:
    json.dump(cfg, f, indent=1)
print(json.dumps({k: cfg[k] for k in ("p_in", "ws_merge_h", "ws_min_cells", "stats")}), flush=True)
