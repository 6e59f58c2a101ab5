"""Trace one warm preconditioner build of a config (PMNS_TRACE=1 PMNS_GPUTIME=1 PMNS_VERBOSE=1 on stderr).
Usage: python scripts/trace_build.py cfg3 [n_warm]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = Solver(cfg, make_image(cfg), device=0)
print("memory plan", s.memory_plan(), flush=True)
for _ in range(nw):
    t0 = time.perf_counter()
    s.build_preconditioner(None)
    torch.cuda.synchronize()
    print(f"warm build {time.perf_counter() - t0:.3f} s", flush=True)
os.environ["PMNS_TRACE"] = "1"
os.environ["PMNS_GPUTIME"] = "1"
os.environ["PMNS_VERBOSE"] = "1"
t0 = time.perf_counter()
s.build_preconditioner(None)
torch.cuda.synchronize()
print(f"traced build {time.perf_counter() - t0:.3f} s", flush=True)
s.close()
