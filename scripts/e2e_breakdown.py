"""Time the end-to-end path (create / solve_steady_host / destroy) of bench.py's
e2e leg phase by phase.  Run with PMNS_TRACE=1 for the library's own laps."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from synth.geometry import load_config, make_image
from paper_2510_22077_b200 import Solver

cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
img = make_image(cfg)
torch.cuda.init()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Solver(cfg, img, device=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    xh = np.zeros(s.N)
    st, rep = s.solve_steady_host(xh)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    s.close()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"e2e {it}: create {1e3*(t1-t0):.1f} ms solve {1e3*(t2-t1):.1f} ms destroy {1e3*(t3-t2):.1f} ms "
          f"(mg {rep['t_mg_ms']:.1f} ml {rep['t_ml_ms']:.1f} sol {rep['t_sol_ms']:.1f}) krylov {rep['krylov_iters']}",
          flush=True)
