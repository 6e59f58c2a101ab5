"""Write tests/golden/<cfg>_<case>.json using ONLY oracle/ (and synth/ for the
image): expected values for the full-size GPU parity tests, which cannot run
the oracle at these sizes inside a test.

Cases
  stokes   Newton step 0 of the steady pipeline (reading A19): build M_S
           (gPLMM with w = 0), one FGMRES solve of J(0) d = -r(0) (P:760
           tolerance 1e-9 ||b0||, restart 50).  Records the Krylov count,
           ||r(x^1)||/||b0||, ||u||, ||p|| of x^1 and seeded samples of x^1.
  steady   the whole A19 steady pipeline (Newton counts, Krylov counts per
           step, residual history, norms and samples of the solution).
  continuation  the Re-continuation pipeline (oracle/newton.py
           solve_continuation) with n_incr increments (cfg "n_incr", default
           4): Newton / Krylov counts per increment, residuals, norms and
           samples of the final solution.
  transient  the transient pipeline (oracle/newton.py
           solve_transient: steady Stokes state, ONE gPLMM build with rho/dt,
           then cfg "n_steps" backward-Euler steps, one Newton solve each):
           Newton / Krylov counts per time step, residuals, norms and samples
           of the final state.
  nnz      Sum of nnz(L+U) of SuperLU's factors of every M_p and M_d block
           of J(0) (M_S) and J(x^1) (gPLMM): the algorithmic-byte basis of
           SURVEY 8(d)'s B_Mp / B_Md.  Needs the Stokes solution x^1.

Also records host-side timings (build / solve), nproc and the threads used.

Usage: python scripts/oracle_golden.py cfg3 stokes nnz
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth.geometry import load_config, make_image  # noqa: E402
from oracle.grid import build_grid  # noqa: E402
from oracle.mac import Mac  # noqa: E402
from oracle.decomposition import decompose, masked_faces  # noqa: E402
from oracle.newton import build_gplmm, newton, solve_steady, solve_continuation, solve_transient  # noqa: E402

N_SAMPLES = 4096


def samples(x, nf, seed):
    """Seeded sample positions (canonical order) of u and p and their values."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nc = x.size - nf
    iu = np.sort(rng.choice(nf, size=min(N_SAMPLES, nf), replace=False))
    ip = np.sort(rng.choice(nc, size=min(N_SAMPLES, nc), replace=False)) + nf
    return dict(u_idx=iu.tolist(), u_val=x[iu].tolist(), p_idx=ip.tolist(), p_val=x[ip].tolist())


def field_stats(x, nf):
    return dict(u_norm=float(np.linalg.norm(x[:nf])), p_norm=float(np.linalg.norm(x[nf:])))


def _nnz_worker(A):
    import scipy.sparse.linalg as spla
    lu = spla.splu(A)
    return int(lu.L.nnz + lu.U.nnz - lu.shape[0])


def lu_nnz_pool(g, dec, A_L, nproc):
    """Same counts as lu_nnz(build_gplmm(...)) -- SuperLU's factors of the
    principal blocks of A_L on every primary and dual set (oracle/gplmm.py
    A17) -- factored in a process pool (nothing else is needed from them)."""
    import multiprocessing as mp
    from oracle.decomposition import w_order, subdomain_unknowns
    perm, seg = w_order(g, dec)
    A_L = A_L.tocsr()
    p_sets = [perm[int(seg[i]):int(seg[i + 1])] for i in range(dec.n_p)]
    d_sets = [subdomain_unknowns(g, cells) for cells in dec.dual_cells]
    blocks = [A_L[s][:, s].tocsc() for s in p_sets]
    dblocks = [A_L[s][:, s].tocsc() for s in d_sets]
    with mp.get_context("fork").Pool(nproc) as pool:
        mp_n = pool.map(_nnz_worker, blocks, chunksize=1)
        md_n = pool.map(_nnz_worker, dblocks, chunksize=1)
    return dict(mp_nnz=int(sum(mp_n)), md_nnz=int(sum(md_n)), mp_rows=int(sum(len(s) for s in p_sets)),
                md_rows=int(sum(len(s) for s in d_sets)), n_p=len(p_sets), n_d=len(d_sets))


def lu_nnz(P):
    """Sum of nnz(L) + nnz(U) - n over SuperLU factors (unit-diagonal L not stored twice)."""
    mp = sum(int(lu.L.nnz + lu.U.nnz - lu.shape[0]) for lu in P.lu_p)
    md = sum(int(lu.L.nnz + lu.U.nnz - lu.shape[0]) for lu in P.lu_d)
    return dict(mp_nnz=mp, md_nnz=md, mp_rows=int(sum(len(s) for s in P.p_sets)),
                md_rows=int(sum(len(s) for s in P.d_sets)), n_p=len(P.p_sets), n_d=len(P.d_sets))


def main(name, cases):
    cfg = load_config(name)
    img = make_image(cfg)
    t0 = time.perf_counter()
    g = build_grid(img, cfg["dim"], cfg["periodic"], cfg["h"])
    dec = decompose(g, cfg["ws_merge_h"], cfg["ws_min_cells"], cfg["dual_layers"], cfg["mask_band"])
    mac = Mac(g, cfg["rho"], cfg["mu"], body_force=cfg["body_force"], p_in=cfg["p_in"] or 0.0,
              p_out=cfg["p_out"] or 0.0, dt=0.0)
    t_setup = time.perf_counter() - t0
    meta = dict(config=name, N=int(g.N), n_f=int(g.n_f), n_c=int(g.n_c), N_p=int(dec.n_p), N_c=int(dec.n_c),
                nproc=os.cpu_count(), threads=os.environ.get("OMP_NUM_THREADS", "default"),
                t_setup_s=round(t_setup, 2), script="scripts/oracle_golden.py (oracle/ only)")
    print(json.dumps(meta), flush=True)
    out_dir = os.environ.get("PMNS_GOLDEN_DIR", os.path.join(ROOT, "tests", "golden"))
    os.makedirs(out_dir, exist_ok=True)
    nproc = os.cpu_count() or 1
    xs = None
    if "stokes" in cases or "nnz" in cases:
        b0n = float(np.linalg.norm(mac.b0()))
        t1 = time.perf_counter()
        MS = build_gplmm(mac, dec, None, masked_faces(g, dec))
        t2 = time.perf_counter()
        rep = {"krylov": [], "res": []}
        xs = newton(mac, MS, np.zeros(g.N), None, max_newton=1, b0n=b0n, report=rep)
        t3 = time.perf_counter()
        out = dict(meta, case="stokes", b0_norm=b0n, krylov=rep["krylov"], res=rep["res"],
                   t_build_s=round(t2 - t1, 2), t_sol_s=round(t3 - t2, 2), **field_stats(xs, g.n_f),
                   **samples(xs, g.n_f, 20251022))
        del MS
        if "nnz" in cases:
            out["nnz_MS"] = lu_nnz_pool(g, dec, mac.jacobian(np.zeros(g.N)), nproc)
        with open(os.path.join(out_dir, f"{name}_stokes.json"), "w") as f:
            json.dump(out, f)
        print(json.dumps({k: v for k, v in out.items() if not k.endswith(("_idx", "_val"))}), flush=True)
    if "nnz" in cases:
        t1 = time.perf_counter()
        nn = dict(meta, case="nnz", nnz_gplmm=lu_nnz_pool(g, dec, mac.jacobian(xs), nproc),
                  t_build_s=round(time.perf_counter() - t1, 2))
        with open(os.path.join(out_dir, f"{name}_factor_nnz.json"), "w") as f:
            json.dump(nn, f, indent=1)
        print(json.dumps(nn), flush=True)
    if "continuation" in cases:
        n_incr = int(cfg.get("n_incr", 4))
        t1 = time.perf_counter()
        x, rep = solve_continuation(mac, dec, n_incr)
        incs = rep["increments"]
        out = dict(meta, case="continuation", n_incr=n_incr, krylov=[r["krylov"] for r in incs],
                   res=[r["res"] for r in incs], converged=bool(incs[-1].get("converged", False)),
                   t_total_s=round(time.perf_counter() - t1, 2), **field_stats(x, g.n_f),
                   **samples(x, g.n_f, 20251024))
        with open(os.path.join(out_dir, f"{name}_continuation.json"), "w") as f:
            json.dump(out, f)
        print(json.dumps({k: v for k, v in out.items() if not k.endswith(("_idx", "_val"))}), flush=True)
    if "transient" in cases:
        n_steps = int(cfg["n_steps"])
        mac_t = Mac(g, cfg["rho"], cfg["mu"], body_force=cfg["body_force"], p_in=cfg["p_in"] or 0.0,
                    p_out=cfg["p_out"] or 0.0, dt=cfg["dt"])
        t1 = time.perf_counter()
        x, rep = solve_transient(mac_t, dec, n_steps)
        out = dict(meta, case="transient", n_steps=n_steps, dt=cfg["dt"], krylov=[r["krylov"] for r in rep["steps"]],
                   res=[r["res"] for r in rep["steps"]], t_total_s=round(time.perf_counter() - t1, 2),
                   **field_stats(x, g.n_f), **samples(x, g.n_f, 20251025))
        with open(os.path.join(out_dir, f"{name}_transient.json"), "w") as f:
            json.dump(out, f)
        print(json.dumps({k: v for k, v in out.items() if not k.endswith(("_idx", "_val"))}), flush=True)
    if "steady" in cases:
        t1 = time.perf_counter()
        x, rep = solve_steady(mac, dec)
        out = dict(meta, case="steady", krylov=rep["krylov"], res=rep["res"], converged=bool(rep["converged"]),
                   t_build_s=round(rep["t_build"], 2), t_sol_s=round(rep["t_sol"], 2),
                   t_total_s=round(time.perf_counter() - t1, 2), **field_stats(x, g.n_f),
                   **samples(x, g.n_f, 20251023))
        with open(os.path.join(out_dir, f"{name}_steady.json"), "w") as f:
            json.dump(out, f)
        print(json.dumps({k: v for k, v in out.items() if not k.endswith(("_idx", "_val"))}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1], set(sys.argv[2:]) or {"stokes"})
