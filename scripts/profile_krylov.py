"""Profiling driver (ncu --profile-from-start off): the Krylov phase of one
Newton step of a config, bracketed by cudaProfilerStart/Stop.

Usage: python scripts/profile_krylov.py cfg3 [wind]
Builds gPLMM (x_b = 0, or with `wind`: a first Stokes step supplies x_b and
the wind, as in the bench pipeline), then runs one Newton step (its FGMRES
solve: every a2-a10 kernel) inside the profiler range.  Prints one JSON line
(Krylov count, time).  Not a bench number."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver, default_opts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
wind = len(sys.argv) > 2 and sys.argv[2] == "wind"
cfg = load_config(name)
s = Solver(cfg, make_image(cfg), device=0)
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
s.build_preconditioner(None)
if wind:
    s.newton_solve(x, opts=default_opts(max_newton=1))
    s.build_preconditioner(x)
torch.cuda.synchronize()
t0 = time.perf_counter()
torch.cuda.profiler.start()
st, rep = s.newton_solve(x, opts=default_opts(max_newton=1))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(json.dumps({"config": name, "wind": wind, "krylov": rep["krylov_iters"][:rep["newton_iters"]],
                  "s": time.perf_counter() - t0, "launches": rep["kernel_launches"]}))
s.close()
