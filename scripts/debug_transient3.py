"""Debug helper: the 3D transient fixture of tests/test_gpu_parity.py alone."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth.geometry import random_blobs  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

cfg = dict(dim=3, periodic=[True, True], h=1e-5, rho=1000.0, mu=1e-3, body_force=[0.0, 0.0, 0.0],
           p_in=400.0, p_out=0.0, dt=2e-4, ws_merge_h=0.5, ws_min_cells=4, dual_layers=1, mask_band=2)
img = random_blobs(15, 13, 11, 0.5, 2.2, 6)
if os.environ.get("WARM"):   # dirty the caching allocator first (as a previous test would)
    from synth.geometry import load_config, make_image
    c1 = load_config("cfg1")
    s0 = Solver(c1, make_image(c1), device=0)
    x0 = torch.zeros(s0.N, dtype=torch.float64, device="cuda")
    s0.solve_steady(x0)
    s0.close()
if os.environ.get("PRE2D"):   # the 2D transient fixture first, as in the test order
    cfg2d = dict(cfg, dim=2, periodic=[False, False], p_in=300.0, dt=5e-4, ws_min_cells=3)
    s1 = Solver(cfg2d, random_blobs(33, 20, 1, 0.5, 2.5, 4), device=0)
    x1 = torch.zeros(s1.N, dtype=torch.float64, device="cuda")
    print("2d", s1.solve_transient(x1, 3)[0])
    s1.close()
    if os.environ.get("RELEASE"):
        from paper_2510_22077_b200._lib import release_cache
        release_cache()
s = Solver(cfg, img, device=0)
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
st, rep = s.solve_transient(x, 3)
print("status", st, rep["step_newton"])
