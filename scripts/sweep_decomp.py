"""Diagnostic: Krylov count of the Stokes step (Newton step 0 with M_S) of a
config under decomposition / drive overrides, through the C ABI on one GPU.
Not a bench number; used to decide DESIGN readings (R2, R5) on config 3.

Usage: python scripts/sweep_decomp.py cfg3 'ws_merge_h=1.0,ws_min_cells=100' 'dual_layers=2' ...
Each argument is one run: comma-separated key=value overrides of the config
(geometry.* keys override the geometry recipe, e.g. geometry.radius.r=6).
Prints one JSON line per run.
"""
import copy
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver, default_opts  # noqa: E402


def _set(cfg, key, val):
    parts = key.split(".")
    d = cfg
    for p in parts[:-1]:
        d = d[p]
    old = d.get(parts[-1])
    if isinstance(old, list):
        d[parts[-1]] = [float(x) for x in val.split(":")]
    elif isinstance(old, int) and not isinstance(old, bool):
        d[parts[-1]] = int(val)
    elif isinstance(old, str):
        d[parts[-1]] = val
    else:
        d[parts[-1]] = float(val)


def main():
    name = sys.argv[1]
    base = load_config(name)
    img_cache = {}
    for spec in sys.argv[2:] or [""]:
        cfg = copy.deepcopy(base)
        opt = {"max_newton": 1}
        n_incr = 0
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=", 1)
            if k in ("max_newton", "restart", "max_krylov"):
                opt[k] = int(v)
            elif k == "continuation":
                n_incr = int(v)
            elif k == "variant":
                opt[k] = v
            else:
                _set(cfg, k, v)
        key = json.dumps(cfg["geometry"], sort_keys=True)
        if key not in img_cache:
            img_cache[key] = make_image(cfg)
        img = img_cache[key]
        t0 = time.time()
        s = Solver(cfg, img, device=0)
        q = s.query()
        x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
        if n_incr:
            st, rep = s.solve_continuation(x, n_incr, default_opts(**opt))
        else:
            st, rep = s.solve_steady(x, default_opts(**opt))
        torch.cuda.synchronize()
        q = s.query()
        print(json.dumps(dict(spec=spec, status=st, N=q["N"], N_p=q["n_p"], N_c=q["n_iface"],
                              dual_unknowns=q["dual_unknowns"], krylov=rep["krylov_iters"],
                              res=rep["res_hist"], t=round(time.time() - t0, 1),
                              t_mg_ms=round(rep["t_mg_ms"]), t_ml_ms=round(rep["t_ml_ms"]),
                              t_sol_ms=round(rep["t_sol_ms"]), mp_GB=round(q["mp_bytes"] / 1e9, 2),
                              ms_per_it=round(rep["t_sol_ms"] / max(1, rep["total_krylov"]), 2),
                              step_newton=rep.get("step_newton"))), flush=True)
        s.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
