"""Profiling driver (ncu --profile-from-start off): one WARM preconditioner build of a config inside
cudaProfilerStart/Stop (two untimed builds first, so the allocator cache and the layouts are warm).
Usage: python scripts/profile_build.py cfg3"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
s = Solver(cfg, make_image(cfg), device=0)
for _ in range(2):
    s.build_preconditioner(None)
torch.cuda.synchronize()
t0 = time.perf_counter()
torch.cuda.profiler.start()
s.build_preconditioner(None)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled build {time.perf_counter() - t0:.3f} s", flush=True)
s.close()
