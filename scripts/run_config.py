"""Run one steady solve of a config through the C ABI and print sizes, timings
and iteration counts (feasibility / scaling checks; not a bench number).

Usage: python scripts/run_config.py cfg3 [key=value ...]   (overrides, e.g. body_force=2600,0,0)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver, default_opts  # noqa: E402

name = sys.argv[1]
cfg = load_config(name)
optkw = {}
n_incr = 0
n_steps = 0
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    if k == "continuation":
        n_incr = int(v)
        continue
    if k == "transient":
        n_steps = int(v)
        continue
    if k in ("max_krylov", "max_newton", "restart"):
        optkw[k] = int(v)
        continue
    if k == "variant":
        optkw[k] = v
        continue
    cfg[k] = [float(x) for x in v.split(",")] if "," in v else float(v)
t0 = time.time()
img = make_image(cfg)
t1 = time.time()
s = Solver(cfg, img, device=0)
t2 = time.time()
q = s.query()
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t3 = time.time()
if n_steps:
    st, rep = s.solve_transient(x, n_steps, default_opts(**optkw))
elif n_incr:
    st, rep = s.solve_continuation(x, n_incr, default_opts(**optkw))
else:
    st, rep = s.solve_steady(x, default_opts(**optkw))
torch.cuda.synchronize()
t4 = time.time()
q = s.query()
out = dict(config=name, status=st, N=q["N"], n_c=q["n_c"], N_p=q["n_p"], N_c=q["n_iface"], n_coarse=q["n_coarse"],
           raw_basins=q["raw_basins"], image_s=round(t1 - t0, 2), setup_s=round(t2 - t1, 2),
           solve_s=round(t4 - t3, 2), newton=rep["newton_iters"], krylov=rep["krylov_iters"],
           res=rep["res_hist"][-1], t_mg_ms=round(rep["t_mg_ms"]), t_ml_ms=round(rep["t_ml_ms"]),
           t_sol_ms=round(rep["t_sol_ms"]), ms_per_krylov=round(rep["t_sol_ms"] / max(1, rep["total_krylov"]), 3),
           mp_GB=round(q["mp_bytes"] / 1e9, 2), md_GB=round(q["md_bytes"] / 1e9, 2),
           coarse_MB=round(q["coarse_bytes"] / 1e6, 1), max_mem_GB=round(torch.cuda.max_memory_allocated() / 1e9, 2),
           overrides=sys.argv[2:], builds=rep["builds"], res_hist=rep["res_hist"][:rep["newton_iters"] + 1],
           n_steps=rep.get("n_steps"), step_newton=rep.get("step_newton"))
print(json.dumps(out))
s.close()
