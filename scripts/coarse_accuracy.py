"""Coarse-scale solver (Algorithm 1) vs the full Newton-FGMRES
solution on one config: speed-up and the paper's error metrics
E_2^p (pressure, % of sup|p_t|) and E_K (permeability K = mu L U_D / dp,
P:699-702), plus E_2 of the outlet-plane x-velocity.  Measurement script:
uses only the product library and the canonical layout rules."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n_ramp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = load_config(name)
img = make_image(cfg)
s = Solver(cfg, img, device=0)
q = s.query()
N, n_c, n_f = q["N"], q["n_c"], q["n_f"]
L = s.export_layout()
void = ((L["label"] >= 0) | (L["iface"] >= 0)).reshape(img.shape)


def canon(xd):
    out = torch.empty_like(xd)
    s.permute(xd, out, to_canonical=True)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def outlet_velocities(xc):
    nz, ny, nx = void.shape
    left = np.zeros((nz, ny, nx + 1), bool)
    right = np.zeros((nz, ny, nx + 1), bool)
    left[:, :, 1:] = void
    right[:, :, :nx] = void
    dof = (left & right) | (right & (np.arange(nx + 1) == 0)) | (left & (np.arange(nx + 1) == nx))
    ids = np.cumsum(dof.reshape(-1)).reshape(dof.shape) - 1
    m = dof[:, :, nx]
    return xc[ids[:, :, nx][m]]


x = torch.zeros(N, dtype=torch.float64, device="cuda")
s.solve_steady(x)                      # warm-up
torch.cuda.synchronize()
t0 = time.time()
st, rep = s.solve_steady(x)
torch.cuda.synchronize()
t_full = time.time() - t0
xt = canon(x)
s.coarse_solve(x, n_ramp)              # warm-up
torch.cuda.synchronize()
t0 = time.time()
st2, rep2 = s.coarse_solve(x, n_ramp)
torch.cuda.synchronize()
t_coarse = time.time() - t0
xa = canon(x)
pt, pa = xt[n_f:], xa[n_f:]
E2p = 100 * np.sqrt(np.mean((np.abs(pt - pa) / np.abs(pt).max()) ** 2))
ut, ua = outlet_velocities(xt), outlet_velocities(xa)
E2u = 100 * np.sqrt(np.mean((np.abs(ut - ua) / np.abs(ut).max()) ** 2))
EK = 100 * abs(ut.sum() - ua.sum()) / abs(ut.sum())    # K is proportional to the outlet flux at fixed dp
out = dict(config=name, n_ramp=n_ramp, t_full_s=round(t_full, 3), t_coarse_s=round(t_coarse, 3),
           speedup=round(t_full / t_coarse, 2), full_krylov=rep["krylov_iters"], coarse_newton=rep2["step_newton"],
           E2_p_pct=round(E2p, 3), E2_uout_pct=round(E2u, 3), E_K_pct=round(EK, 3),
           K_over=bool(ua.sum() > ut.sum()), coarse_res=rep2["res_hist"][:rep2["n_steps"]])
print(json.dumps(out))
s.close()
