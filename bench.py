#!/usr/bin/env python
"""Benchmark: gPLMM-preconditioned Newton-FGMRES on B200 (arXiv 2510.22077).

One STEP = one complete steady solve of the configured workload through the
C ABI, i.e. every hot-path row of SURVEY §8(a) (a1-a11, B1, B2): config 3
(the default, the largest single-GPU config) reaches Re ~10 by the paper's
Re continuation (pmns_solve_continuation, 4 drive increments: increment 1 =
build M_S -> Stokes step -> gPLMM with the Stokes wind -> Newton; each later
increment rebuilds gPLMM from the previous solution); config 2
is the A19 steady pipeline (pmns_solve_steady).  Every Newton solve runs to
||r||/||b0|| <= 1e-8.  Setup (S1/S2: decomposition,
numbering, upload) happens once in pmns_create, outside the timed region.

metric: void-unknown x Krylov-iterations per second over the whole step
(builds included) = N * sum(FGMRES iterations) / T_step, summed over ranks.

Roofline: M_p apply, J apply, M_d, whole M^{-1} and whole
FGMRES iteration, each as SURVEY's ALGORITHMIC bytes (SuperLU nnz of the
same local blocks, oracle-written under tests/golden/) over CUDA-event time
on the solve stream; the builder's stored bytes are reported beside them.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pmns|reference] [--config cfg3]
N > 1 is launched by torchrun (one process per GPU) and partitions ONE
problem over the ranks (strong scaling).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "void-unknown*Krylov-iters/s (gPLMM Newton-FGMRES, fp64)"
UNIT = "unknown*iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pmns", choices=["pmns", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ----------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.lines = []

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def mark(self, timeout=5.0):
        """Wait for the sampler's first line (nvidia-smi's start-up is outside
        the timed region), then keep only the samples taken from now on."""
        t0 = time.time()
        while self.p is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)
        self.m = len(self.lines)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        m = getattr(self, "m", 0)
        timed = self.lines[m:] if len(self.lines) > m else self.lines
        for ln in timed:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# oracle (CPU baseline / reference arm): the oracle's own per-iteration
# operations timed on a seeded sample of the workload's subdomains
# ----------------------------------------------------------------------------
def _solve_block(args):
    """Factor one oracle local block (untimed) and time its solves (one
    SuperLU triangular solve pair per FGMRES iteration, as GPLMM.Mp/Md do)."""
    import scipy.sparse.linalg as spla
    A, reps = args
    lu = spla.splu(A)
    v = np.random.default_rng(0).standard_normal(A.shape[0])
    t0 = time.perf_counter()
    for _ in range(reps):
        lu.solve(v)
    return (time.perf_counter() - t0) / reps, int(lu.L.nnz + lu.U.nnz - A.shape[0])


def oracle_prepare(cfg, img, n_sample=24, seed=11):
    """Oracle setup (decomposition, J(0) as CSR) and a seeded sample of primary
    and dual blocks (the oracle's own principal submatrices, oracle/gplmm.py
    A17); nothing here is timed."""
    from threadpoolctl import threadpool_limits
    from oracle.grid import build_grid
    from oracle.mac import Mac
    from oracle.decomposition import decompose, w_order, subdomain_unknowns
    with threadpool_limits(1):
        g = build_grid(img, cfg["dim"], cfg["periodic"], cfg["h"])
        dec = decompose(g, cfg["ws_merge_h"], cfg["ws_min_cells"], cfg["dual_layers"], cfg["mask_band"])
        mac = Mac(g, cfg["rho"], cfg["mu"], body_force=cfg["body_force"], p_in=cfg["p_in"],
                  p_out=cfg["p_out"], dt=cfg.get("dt") or 0.0)
        J = mac.jacobian(np.zeros(g.N)).tocsr()
        perm, seg = w_order(g, dec)
        rng = np.random.Generator(np.random.PCG64(seed))
        ip = np.sort(rng.choice(dec.n_p, size=min(n_sample, dec.n_p), replace=False))
        idd = np.sort(rng.choice(dec.n_c, size=min(n_sample, dec.n_c), replace=False)) if dec.n_c else []
        pb = [J[perm[int(seg[i]):int(seg[i + 1])]][:, perm[int(seg[i]):int(seg[i + 1])]].tocsc() for i in ip]
        db = []
        for j in idd:
            s_ = subdomain_unknowns(g, dec.dual_cells[j])
            db.append(J[s_][:, s_].tocsc())
    return dict(g=g, dec=dec, J=J, pb=pb, db=db, n_p=dec.n_p, n_d=dec.n_c)


def oracle_iter_time(prep, cores, j_mean=25, reps=3):
    """Seconds per FGMRES iteration of the oracle (Newton step 0, M_S local
    blocks), from its own operations: SuperLU solves of the sampled primary
    and dual blocks scaled to all N^p + N^d blocks (unbiased: mean x count),
    3 CSR J applies (a6, a8, a10), and MGS over j_mean + 1 basis vectors
    (oracle/krylov.py).  M_G ("negligible") is not charged, which
    favours the baseline.  cores > 1: the independent block solves run in a
    process pool (multiprocessing over subdomains)."""
    import multiprocessing as mp
    from threadpoolctl import threadpool_limits
    N = prep["g"].N
    jobs = [(A, reps) for A in prep["pb"]] + [(A, reps) for A in prep["db"]]
    npb = len(prep["pb"])
    with threadpool_limits(1):
        if cores > 1:
            # solves timed inside `cores` concurrent workers (memory-bandwidth
            # contention included); perfect load balance over the blocks is
            # assumed, which favours the baseline
            with mp.get_context("fork").Pool(cores) as pool:
                res = pool.map(_solve_block, jobs, chunksize=1)
        else:
            res = [_solve_block(j) for j in jobs]
        tp = np.mean([r[0] for r in res[:npb]]) * prep["n_p"] / cores if npb else 0.0
        td = np.mean([r[0] for r in res[npb:]]) * prep["n_d"] / cores if len(res) > npb else 0.0
        v = np.random.default_rng(1).standard_normal(N)
        t0 = time.perf_counter()
        for _ in range(reps):
            prep["J"] @ v
        tj = (time.perf_counter() - t0) / reps
        V = np.random.default_rng(2).standard_normal((4, N))
        t0 = time.perf_counter()
        for _ in range(reps):
            w = V[0].copy()
            for i in range(1, 4):
                h = np.dot(w, V[i])
                w = w - h * V[i]
        tm = (time.perf_counter() - t0) / (reps * 3) * (j_mean + 1)
    return tp + td + 3 * tj + tm, dict(t_mp=tp, t_md=td, t_j=tj, t_mgs=tm)


def oracle_baseline(prep, cores):
    t, parts = oracle_iter_time(prep, cores)
    N = prep["g"].N
    return N / t, parts


def check_converged(st, rep):
    """Every warm-up, timed and e2e step must converge (a capped solve would
    inflate N * sum(Krylov) / T)."""
    if st != 0 or not rep["converged"]:
        print(json.dumps({"error": "solve did not converge", "status": st, "krylov": rep["krylov_iters"],
                          "res_hist": rep["res_hist"]}), flush=True)
        sys.exit(3)


# ----------------------------------------------------------------------------
# SURVEY 8(d) algorithmic bytes
# ----------------------------------------------------------------------------
def golden_nnz(name):
    """SuperLU nnz(L+U) of every M_p / M_d block of J(0) (M_S) and J(x^1)
    (gPLMM), written by scripts/oracle_golden.py (oracle/ only): the byte basis
    of SURVEY 8(d)'s B_Mp / B_Md.  None if the config has no such record."""
    out = {}
    try:
        out["MS"] = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}_stokes.json")))["nnz_MS"]
        out["G"] = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}_factor_nnz.json")))["nnz_gplmm"]
    except Exception:
        return None
    return out


def alg_bytes(q, nnz, krylov, restart):
    """Per-apply and per-iteration algorithmic bytes:
    B_J = 8(2N + n_f) (+8N fused), B_Mp = 8 nnz(LU_p) + 24 N_prim,
    B_Md = 8 nnz(LU_d) + 24 sum n_d, B_MG = 16N + prolongation rows + coarse
    inverse (stored), B_M = B_MG + 2 B_J(fused) + B_Md + B_Mp,
    B_Arn(j) = 32N(j+1) + 16N, B_iter = B_J + B_M + B_Arn(j).  Step 0 applies
    M_S (J(0) blocks), later Newton steps gPLMM (J(x^1) blocks)."""
    N, nf = q["N"], q["n_f"]
    bj = 8 * (2 * N + nf)
    bjf = bj + 8 * N
    bmg = 16 * N + q["prolong_bytes"] + q["coarse_bytes"]
    tot = dict(mp=0.0, md=0.0, m=0.0, it=0.0, n=0)
    for k, its in enumerate(krylov):
        key = "MS" if k == 0 else "G"
        bmp = 8 * nnz[key]["mp_nnz"] + 24 * nnz[key]["mp_rows"]
        bmd = 8 * nnz[key]["md_nnz"] + 24 * nnz[key]["md_rows"]
        bm = bmg + 2 * bjf + bmd + bmp
        for i in range(its):
            j = i % restart
            tot["mp"] += bmp
            tot["md"] += bmd
            tot["m"] += bm
            tot["it"] += bj + bm + 32 * N * (j + 1) + 16 * N
            tot["n"] += 1
    return bj, bjf, tot


# ----------------------------------------------------------------------------
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from synth.geometry import load_config, make_image
    cfg = load_config(a.config)
    img = make_image(cfg)
    n_incr = int(cfg.get("n_incr", 1)) if cfg.get("pipeline") == "continuation" else 1
    n_tsteps = int(cfg.get("n_steps", 0)) if (cfg.get("pipeline") == "transient" or not cfg.get("steady", True)) else 0
    config = {"workload": f"{a.config}: {cfg['geometry']}", "N_unknowns": None,
              "steady": n_tsteps == 0, "Re_target": cfg["Re_target"],
              "pipeline": (f"transient (P:840-843): steady Stokes state, ONE gPLMM build with rho/dt, {n_tsteps} "
                           f"backward-Euler steps of dt = {cfg['dt']:.3e} s, one Newton solve each" if n_tsteps else
                           f"Re continuation, {n_incr} drive increments (P:763, P:918), gPLMM rebuilt per increment"
                           if n_incr > 1 else "steady A19: M_S Stokes step, gPLMM rebuild, Newton"),
              "l2": "inputs larger than L2: each step streams the stored local inverses (>> 126 MB)"}
    ncores = os.cpu_count() or 1

    if a.impl == "reference":
        if rank != 0:
            return
        t0 = time.perf_counter()
        prep = oracle_prepare(cfg, img)
        t_prep = time.perf_counter() - t0
        for _ in range(a.warmup):
            oracle_iter_time(prep, ncores, reps=1)
        ts = []
        for _ in range(a.steps):
            t, parts = oracle_iter_time(prep, ncores)
            ts.append(t)
        N = prep["g"].N
        val = N / float(np.mean(ts))
        config["N_unknowns"] = int(N)
        sample = (f"oracle (NumPy/SciPy, SuperLU) on {a.config}, {ncores} cores: seconds per FGMRES iteration of "
                  f"Newton step 0 from its own operations -- SuperLU solves of {len(prep['pb'])} seeded primary and "
                  f"{len(prep['db'])} dual blocks of J(0) in a {ncores}-process pool, scaled by "
                  f"N^p={prep['n_p']}, N^d={prep['n_d']}; 3 CSR J applies; MGS over 26 vectors. M_G and all builds "
                  f"excluded (favours the baseline). setup {t_prep:.0f} s untimed")
        out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * float(np.mean(ts)),
               "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
               "dtype": "f64", "data": f"synthetic (seeded sphere pack, BASELINE {a.config})", "config": config,
               "cpu_baseline": {"value": val, "unit": UNIT, "cores": ncores, "kind": "oracle", "sample": sample,
                                "parts_s": parts},
               "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2510_22077_b200 import Solver
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    from paper_2510_22077_b200._lib import comm_unique_id

    def _partition(solver):
        """N > 1: one problem partitioned over the ranks: each GPU
        owns a z-slab of primaries with their interfaces and dual grids; the
        Krylov phase exchanges halos over NCCL (strong scaling)."""
        if world == 1:
            return
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        solver.set_comm(rank, world, obj[0])

    def solve(solver, xv):
        if n_tsteps:
            xv.zero_()   # every bench step starts the transient from rest
            return solver.solve_transient(xv, n_tsteps)
        return solver.solve_continuation(xv, n_incr) if n_incr > 1 else solver.solve_steady(xv)

    t0 = time.perf_counter()
    s = Solver(cfg, img, device=local)
    _partition(s)
    t_setup = time.perf_counter() - t0
    q = s.query()
    N = q["N"]
    config["N_unknowns"] = int(N)
    config["N_p"] = int(q["n_p"])
    config["N_c"] = int(q["n_iface"])
    config["parallelism"] = (f"z-slabs over {world} GPUs: owned primaries/interfaces/duals, NCCL halo exchanges "
                             f"for J and M_d, distributed CGS2, coarse-RHS allreduce (DESIGN.md 8)"
                             if world > 1 else "1 GPU")
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    # clocks sampler started before the last warm-up step, so nvidia-smi's own
    # start-up (NVML init) does not fall into the timed region
    clk = Clocks(local)
    for w in range(a.warmup):
        if w == a.warmup - 1:
            s.profile(True)   # last warm-up step fills the library's timing-event pool
            clk.start()
        st, rep = solve(s, x)
        check_converged(st, rep)
    torch.cuda.synchronize()
    s.profile(True)           # clear (events recycled) and record the timed steps
    if clk.p is None:
        clk.start()
    clk.mark()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    reps = []
    for _ in range(a.steps):
        st, rep = solve(s, x)
        check_converged(st, rep)
        reps.append(rep)
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    from paper_2510_22077_b200.dist import max_over_ranks
    ms = max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    iters = sum(r["total_krylov"] for r in reps)
    value = N * iters / (ms / 1e3)   # one problem on all ranks (strong scaling for N > 1)
    launches = sum(r["kernel_launches"] for r in reps)
    # live rooflines (CUDA events on the solve stream, production graph path):
    # achieved = SURVEY 8(d) ALGORITHMIC bytes (SuperLU nnz of the same local
    # blocks, written by the oracle) / device time; the builder's stored bytes
    # are reported beside them
    cnt, kms, kbytes = s.profile_query(3)   # whole M_p applies (one CUDA graph each)
    jc, jms, jbytes = s.profile_query(2)    # J applies (bytes = B_J, fused where fused)
    dc, dms, dbytes = s.profile_query(4)    # whole M_d applies
    mc, mms, _ = s.profile_query(5)         # whole M^{-1} applies
    s.profile(False)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    q = s.query()
    nnz = golden_nnz(a.config)
    r0 = reps[-1]
    kry = r0["krylov_iters"][:r0["newton_iters"]]
    if nnz:
        bj, bjf, tot = alg_bytes(q, nnz, kry, 50)
        alg_mp = tot["mp"] / tot["n"]
        alg_md = tot["md"] / tot["n"]
        alg_m = tot["m"] / tot["n"]
        alg_it = tot["it"] / tot["n"]
        basis = "SURVEY 8(d) algorithmic bytes: SuperLU nnz(L+U) of the same blocks (tests/golden, oracle-written)"
    else:
        alg_mp, alg_md, alg_m, alg_it = kbytes / max(cnt, 1), dbytes / max(dc, 1), None, None
        basis = "stored bytes (no oracle nnz record for this config)"
    gbs = lambda by, t_ms: by / t_ms / 1e6 if t_ms else None   # noqa: E731
    achieved = gbs(alg_mp, kms / cnt) if cnt else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", f"traffic_{a.config}.json")))
        traffic = prof.get("mp_apply_dram_bytes_per_apply")
    except Exception:
        pass
    t_it_ms = sum(r["t_sol_ms"] for r in reps) / max(1, iters)
    roof = {"bound": "hbm",
            "kernel": "M_p apply (a9): the nested-dissection level sweeps (gemv_rows_kernel + nd_update_kernel, "
                      "one CUDA graph), timed per apply",
            "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic,
            "bytes_basis": basis,
            "algorithmic_bytes_per_launch": alg_mp, "stored_bytes_per_launch": kbytes / cnt if cnt else None,
            "frac_on_stored_bytes": gbs(kbytes / cnt, kms / cnt) / peak if cnt else None,
            "launches": cnt, "unit_of_launch": "one M_p apply",
            "share_of_step": (kms / ms) if ms else None,
            "jacobian_apply": {"achieved": gbs(jbytes / jc, jms / jc) if jc else None,
                               "frac": gbs(jbytes / jc, jms / jc) / peak if jc else None,
                               "bytes_per_launch": jbytes / jc if jc else None, "launches": jc,
                               "share_of_step": jms / ms if ms else None},
            "md_apply": {"achieved": gbs(alg_md, dms / dc) if dc else None,
                         "frac": gbs(alg_md, dms / dc) / peak if dc else None,
                         "frac_on_stored_bytes": gbs(dbytes / dc, dms / dc) / peak if dc else None,
                         "share_of_step": dms / ms if ms else None},
            "preconditioner_apply": {"achieved": gbs(alg_m, mms / mc) if (mc and alg_m) else None,
                                     "frac": gbs(alg_m, mms / mc) / peak if (mc and alg_m) else None,
                                     "bytes_per_launch": alg_m, "launches": mc,
                                     "ms_per_launch": mms / mc if mc else None},
            "fgmres_iteration": {"achieved": gbs(alg_it, t_it_ms) if alg_it else None,
                                 "frac": gbs(alg_it, t_it_ms) / peak if alg_it else None,
                                 "bytes_per_iteration": alg_it, "ms_per_iteration": t_it_ms}}
    # the build (B1/B2: nested-dissection factorisations of M_p, the folded Abar and M_d) is the other large
    # share of the step: a dense fp64 contraction on the DMMA tensor path, reported against the measured
    # cuBLAS DGEMM rate of this pool's B200 (profiles/r02_dgemm_rates.txt: 35.5 TF/s at n = 8192; the guides give
    # no measured fp64 peak, the programming guide's nominal figure is 45 TF/s)
    try:
        plan = s.memory_plan()
        nb_ = sum(r["builds"] for r in reps)
        t_build_ms = sum(r["t_ml_ms"] + r["t_mg_ms"] for r in reps)
        fl = 2.0 * plan["mp_flops"] + plan["md_flops"]
        roof["build_factorisation"] = {
            "bound": "tensor (fp64 DMMA, mma.sync.m8n8k4.f64)", "flops_per_build": fl,
            "flops_basis": "2m^3 + 2m^2 b + 2 b^2 m per front (explicit pivot-block inverse, W12, Schur update) "
                           "for M_p and the folded Abar, plus M_d; L21 and the multi-RHS solves not counted",
            "builds": nb_, "ms_per_build": t_build_ms / max(nb_, 1),
            "achieved": fl * nb_ / (t_build_ms / 1e3) / 1e12 if t_build_ms else None, "unit": "TFLOP/s",
            "peak": 35.5, "peak_source": "measured cuBLAS DGEMM 8192^3 on this pool's B200 "
                                         "(profiles/r02_dgemm_rates.txt); nominal 45 (programming guide)",
            "frac": (fl * nb_ / (t_build_ms / 1e3) / 1e12) / 35.5 if t_build_ms else None,
            "share_of_step": t_build_ms / ms if ms else None}
    except Exception as e:  # noqa: BLE001
        roof["build_factorisation"] = {"error": str(e)}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic (seeded Boolean sphere pack, BASELINE {a.config}; no paper dataset available)",
           "config": config, "gpu_launches": launches, "clocks": clocks, "roofline": roof,
           "solve": {"newton_iters": r0["newton_iters"], "krylov_iters": r0["krylov_iters"],
                     "res_hist": r0["res_hist"], "t_mg_ms": r0["t_mg_ms"], "t_ml_ms": r0["t_ml_ms"],
                     "t_sol_ms": r0["t_sol_ms"], "t_setup_s": t_setup,
                     "theta_sol": N * r0["total_krylov"] / (r0["t_sol_ms"] / 1e3),
                     "stored_bytes": {k: q2 for k, q2 in q.items() if k.endswith("_bytes")}}}
    s.close()   # the e2e contexts below need the device memory (config 3: ~100 GB per build)
    # end-to-end through the C ABI with host buffers: create from the host image,
    # solve with host output (H2D/D2H inside), destroy
    e2e_steps = min(a.steps, 2)
    xh = np.zeros(N)
    te = 0.0
    e_it = 0
    for _ in range(e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = Solver(cfg, img, device=local)
        _partition(s2)
        st2, rep2 = (s2.solve_transient_host(xh, n_tsteps) if n_tsteps
                     else s2.solve_continuation_host(xh, n_incr))
        check_converged(st2, rep2)
        h2d = s2.query()["h2d_bytes"]
        s2.close()
        torch.cuda.synchronize()
        te += time.perf_counter() - t0
        e_it += rep2["total_krylov"]
    te = max_over_ranks(te * 1e3, device="cuda") / 1e3
    out["e2e"] = {"value": N * e_it / te, "unit": UNIT,
                  "h2d_bytes_per_step": int(h2d + img.nbytes), "d2h_bytes_per_step": int(8 * N),
                  "includes": "pmns_create (host setup + upload) + pmns_solve_continuation_host / "
                              "pmns_solve_transient_host (pipeline of the config, H2D/D2H inside) + pmns_destroy"}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        t0 = time.perf_counter()
        prep = oracle_prepare(cfg, img)
        t_prep = time.perf_counter() - t0
        v1, p1 = oracle_baseline(prep, 1)
        vn, pn = oracle_baseline(prep, ncores)
        out["cpu_baseline"] = {
            "value": vn, "unit": UNIT, "cores": ncores, "kind": "oracle",
            "value_1core": v1, "parts_s_1core": p1, "parts_s": pn,
            "sample": (f"oracle on {a.config}: seconds per FGMRES iteration (Newton step 0) from its own "
                       f"operations -- SuperLU solves of {len(prep['pb'])} seeded primary + {len(prep['db'])} dual "
                       f"blocks of J(0) (concurrently in a {ncores}-process pool for `value`; serially for "
                       f"value_1core), scaled by N^p={prep['n_p']}, N^d={prep['n_d']}; 3 CSR J applies; MGS over "
                       f"26 vectors; M_G and builds not charged (favours the baseline); setup {t_prep:.0f} s "
                       f"untimed")}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
