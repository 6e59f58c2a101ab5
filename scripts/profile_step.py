"""One warm-up steady solve then one measured steady solve of a config through
the C ABI (for ncu launch lists / captures; never a bench number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = load_config(name)
s = Solver(cfg, make_image(cfg), device=0)
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
for _ in range(reps):
    st, rep = s.solve_steady(x)
torch.cuda.synchronize()
print(name, "status", st, "newton", rep["newton_iters"], "krylov", rep["krylov_iters"],
      "t_mg", round(rep["t_mg_ms"]), "t_ml", round(rep["t_ml_ms"]), "t_sol", round(rep["t_sol_ms"]),
      "launches", rep["kernel_launches"])
s.close()
