"""Warm a context with two steady solves, then trace a third one
(PMNS_TRACE=1 PMNS_GPUTIME=1 set only for it; output on stderr)."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
from synth.geometry import load_config, make_image
from paper_2510_22077_b200 import Solver
import torch

cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
img = make_image(cfg)
s = Solver(cfg, img, device=0)
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
for _ in range(2):
    s.solve_steady(x)
torch.cuda.synchronize()
os.environ["PMNS_TRACE"] = "1"
os.environ["PMNS_GPUTIME"] = "1"
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    print(f"---- traced solve {it} ----", file=sys.stderr, flush=True)
    st, rep = s.solve_steady(x)
    torch.cuda.synchronize()
    print(rep["t_mg_ms"], rep["t_ml_ms"], rep["t_sol_ms"], flush=True)
