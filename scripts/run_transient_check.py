"""Run a config's transient pipeline on the GPU (pmns_solve_transient) and check the final time
step with the ORACLE's residual: after n_steps steps (state x^n) one more step is taken from u^n = x^n, and
||r(x^{n+1}; u^n)|| / ||b0|| is evaluated by oracle/mac.py (assembled CSR residual, backward Euler).

Usage: python scripts/run_transient_check.py cfg4h [n_steps]
Prints one JSON line (sizes, memory plan, timings, Newton / Krylov counts per step, the oracle residual)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver, default_opts  # noqa: E402

name = sys.argv[1]
cfg = load_config(name)
n_steps = int(sys.argv[2]) if len(sys.argv) > 2 else int(cfg["n_steps"])
img = make_image(cfg)
t0 = time.time()
s = Solver(cfg, img, device=0)
t_setup = time.time() - t0
q = s.query()
plan = s.memory_plan()
print(json.dumps({"config": name, "N": q["N"], "N_p": q["n_p"], "N_c": q["n_iface"], "setup_s": round(t_setup, 1),
                  "mp_GB": plan["mp_bytes"] / 1e9, "md_GB": plan["md_bytes"] / 1e9}), flush=True)
x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.time()
st, rep = s.solve_transient(x, n_steps, default_opts())
torch.cuda.synchronize()
t_solve = time.time() - t0
out = dict(config=name, status=st, N=q["N"], N_p=q["n_p"], N_c=q["n_iface"], setup_s=round(t_setup, 1),
           solve_s=round(t_solve, 1), n_steps=rep["n_steps"], step_newton=rep["step_newton"],
           krylov=rep["krylov_iters"], total_krylov=rep["total_krylov"], t_mg_ms=round(rep["t_mg_ms"]),
           t_ml_ms=round(rep["t_ml_ms"]), t_sol_ms=round(rep["t_sol_ms"]),
           ms_per_krylov=round(rep["t_sol_ms"] / max(1, rep["total_krylov"]), 3),
           unknown_iters_per_s=q["N"] * rep["total_krylov"] / max(t_solve, 1e-9),
           mp_GB=round(s.query()["mp_bytes"] / 1e9, 2), md_GB=round(s.query()["md_bytes"] / 1e9, 2))
print(json.dumps(out), flush=True)
if st == 0:
    # one more step from u^n = x^n with the preconditioner already built (newton_solve), checked by the oracle
    up = x.clone()
    st2, rep2 = s.newton_solve(x, u_prev=up, opts=default_opts())
    xc = torch.empty_like(x)
    uc = torch.empty_like(x)
    s.permute(x, xc, to_canonical=True)
    s.permute(up, uc, to_canonical=True)
    torch.cuda.synchronize()
    xg, ug = xc.cpu().numpy(), uc.cpu().numpy()
    s.close()
    from oracle.grid import build_grid
    from oracle.mac import Mac
    g = build_grid(img, cfg["dim"], cfg["periodic"], cfg["h"])
    mac = Mac(g, cfg["rho"], cfg["mu"], body_force=cfg["body_force"], p_in=cfg["p_in"], p_out=cfg["p_out"],
              dt=cfg["dt"])
    r = mac.residual(xg, ug[:g.n_f])
    b0 = np.linalg.norm(mac.b0())
    nf = g.n_f
    print(json.dumps(dict(check="oracle residual of the extra step", status=st2, krylov=rep2["krylov_iters"],
                          res_gpu=rep2["res_hist"][-1], oracle_res=float(np.linalg.norm(r) / b0),
                          oracle_res_momentum=float(np.linalg.norm(r[:nf]) / b0),
                          oracle_res_mass=float(np.linalg.norm(r[nf:]) / b0), ok=bool(np.linalg.norm(r) <= 1e-8 * b0))),
          flush=True)
