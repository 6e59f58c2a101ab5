"""Trace the second (warm) run of a config's bench pipeline (PMNS_TRACE=1 PMNS_GPUTIME=1 on stderr): per-build
phases, per-level assembly sub-phases and allocator statistics as they occur inside a whole solve.
Usage: python scripts/trace_solve.py cfg3"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
n_incr = int(cfg.get("n_incr", 1)) if cfg.get("pipeline") == "continuation" else 1
s = Solver(cfg, make_image(cfg), device=0)
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
for it in range(3):
    if it == 2:
        os.environ["PMNS_TRACE"] = "1"
        os.environ["PMNS_GPUTIME"] = "1"
    x.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, rep = s.solve_continuation(x, n_incr) if n_incr > 1 else s.solve_steady(x)
    torch.cuda.synchronize()
    print(f"solve {it}: {time.perf_counter() - t0:.3f} s  t_mg {rep['t_mg_ms']:.0f} t_ml {rep['t_ml_ms']:.0f} "
          f"t_sol {rep['t_sol_ms']:.0f} ms  builds {rep['builds']}", flush=True)
s.close()
