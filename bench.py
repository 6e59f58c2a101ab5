#!/usr/bin/env python
"""Benchmark: gPLMM-preconditioned Newton-FGMRES on B200 (arXiv 2510.22077).

One STEP = one complete steady solve of the configured workload through the
C ABI (pmns_solve_steady: build M_S -> Newton step 0 (Stokes) -> rebuild
gPLMM with the Stokes wind -> Newton to ||r||/||b0|| <= 1e-8), i.e. every
hot-path row of SURVEY §8(a) (a1-a11, B1, B2).  Setup (S1/S2: decomposition,
numbering, upload) happens once in pmns_create, outside the timed region.

metric: void-unknown x Krylov-iterations per second over the whole step
(builds included) = N * sum(FGMRES iterations) / T_step, summed over ranks.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pmns|reference] [--config cfg2]
N > 1 is launched by torchrun (one process per GPU): round 1 runs
independent replicas of the workload on each rank (weak scaling; the slab
decomposition is not built yet — DESIGN.md §8).
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
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=25)
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
# oracle (CPU baseline / reference arm)
# ----------------------------------------------------------------------------
def oracle_prepare(cfg, img):
    from threadpoolctl import threadpool_limits
    from oracle.grid import build_grid
    from oracle.mac import Mac
    from oracle.decomposition import decompose
    from oracle.newton import build_gplmm
    with threadpool_limits(1):
        g = build_grid(img, cfg["dim"], cfg["periodic"], cfg["h"])
        dec = decompose(g, cfg["ws_merge_h"], cfg["ws_min_cells"], cfg["dual_layers"], cfg["mask_band"])
        mac = Mac(g, cfg["rho"], cfg["mu"], body_force=cfg["body_force"], p_in=cfg["p_in"],
                  p_out=cfg["p_out"], dt=cfg.get("dt") or 0.0)
        P = build_gplmm(mac, dec, None)
        J = mac.jacobian(np.zeros(g.N))
        b = -mac.residual(np.zeros(g.N))
    return g, mac, P, J, b


def oracle_iters(prep, n_iters):
    """Time n_iters right-preconditioned FGMRES(MGS) iterations of Newton
    step 0 (the oracle as it stands, 1 thread)."""
    from threadpoolctl import threadpool_limits
    from oracle.krylov import fgmres
    g, mac, P, J, b = prep
    with threadpool_limits(1):
        t0 = time.perf_counter()
        _, it, _, _ = fgmres(lambda v: J @ v, b, lambda v: P.apply(v, J), 0.0, m=50, maxit=n_iters)
        t1 = time.perf_counter()
    return it, t1 - t0


# ----------------------------------------------------------------------------
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from synth.geometry import load_config, make_image
    cfg = load_config(a.config)
    img = make_image(cfg)
    config = {"workload": f"{a.config}: {cfg['geometry']}", "N_unknowns": None,
              "steady": True, "Re_target": cfg["Re_target"],
              "l2": "inputs larger than L2: each step streams the stored local inverses (>> 126 MB)"}

    if a.impl == "reference":
        if rank != 0:
            return
        prep = oracle_prepare(cfg, img)
        g = prep[0]
        per = max(1, a.cpu_iters // 5)
        for _ in range(a.warmup):
            oracle_iters(prep, per)
        tot_it, tot_t = 0, 0.0
        for _ in range(a.steps):
            it, t = oracle_iters(prep, per)
            tot_it += it
            tot_t += t
        val = g.N * tot_it / tot_t
        config["N_unknowns"] = int(g.N)
        sample = (f"oracle (NumPy/SciPy SuperLU, 1 thread) on {a.config}: each step = {per} FGMRES iterations of "
                  f"Newton step 0 with the prebuilt M_S (build excluded, so this favours the baseline)")
        out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tot_t / a.steps,
               "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
               "dtype": "f64", "data": "synthetic (seeded Boolean sphere pack, BASELINE config 2)", "config": config,
               "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
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
        """N > 1: one steady problem partitioned over the ranks:
        each GPU owns a slab of primaries, NCCL all-reduces the owned M_p output
        and shape vectors (strong scaling)."""
        if world == 1:
            return
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        solver.set_comm(rank, world, obj[0])

    t0 = time.perf_counter()
    s = Solver(cfg, img, device=local)
    _partition(s)
    t_setup = time.perf_counter() - t0
    q = s.query()
    N = q["N"]
    config["N_unknowns"] = int(N)
    config["N_p"] = int(q["n_p"])
    config["N_c"] = int(q["n_iface"])
    config["parallelism"] = (f"primary slabs over {world} GPUs (owned M_p/Abar fronts, NCCL all-reduce)"
                             if world > 1 else "1 GPU")
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    # clocks sampler started before the last warm-up step, so nvidia-smi's own
    # start-up (NVML init) does not fall into the timed region
    clk = Clocks(local)
    for w in range(a.warmup):
        if w == a.warmup - 1:
            s.profile(True)   # last warm-up step fills the library's timing-event pool
            clk.start()
        st, rep = s.solve_steady(x)
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
        st, rep = s.solve_steady(x)
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
    # live roofline of the dominant kernel: the M_p local-solve GEMV sweeps (a9;
    # gemv_rows_kernel over the nested-dissection front levels), every launch
    # timed with CUDA events on the solve stream; bytes = stored operator rows
    # streamed + x gathers + y writes per launch
    cnt, kms, kbytes = s.profile_query(3)   # whole M_p applies (one CUDA graph each)
    jc, jms, jbytes = s.profile_query(2)
    dc, dms, dbytes = s.profile_query(4)   # whole M_d applies
    s.profile(False)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    achieved = (kbytes / cnt) / (kms / cnt) / 1e6 if cnt else None   # bytes/ms -> GB/s
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "r01_traffic.json")))
        traffic = prof.get("mp_apply_dram_bytes_per_apply")
    except Exception:
        pass
    roof = {"bound": "hbm",
            "kernel": "M_p apply (a9): the nested-dissection level sweeps, gemv_rows_kernel + nd_update_kernel "
                      "in one CUDA graph, timed per apply",
            "achieved": achieved,
            "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic,
            "algorithmic_bytes_per_launch": kbytes // cnt if cnt else None, "launches": cnt,
            "unit_of_launch": "one M_p apply (15 GEMV + 7 update kernels of the captured graph)",
            "share_of_step": (kms / ms) if ms else None,
            "others": {"jacobian_apply_GBps": (jbytes / jms / 1e6) if jc else None,
                       "md_apply_GBps": (dbytes / dms / 1e6) if dc else None,
                       "jacobian_share": jms / ms if ms else None, "md_share": dms / ms if ms else None}}
    r0 = reps[-1]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded Boolean sphere pack, BASELINE config 2; no paper dataset available)",
           "config": config, "gpu_launches": launches, "clocks": clocks, "roofline": roof,
           "solve": {"newton_iters": r0["newton_iters"], "krylov_iters": r0["krylov_iters"],
                     "res_hist": r0["res_hist"], "t_mg_ms": r0["t_mg_ms"], "t_ml_ms": r0["t_ml_ms"],
                     "t_sol_ms": r0["t_sol_ms"], "t_setup_s": t_setup,
                     "theta_sol": N * r0["total_krylov"] / (r0["t_sol_ms"] / 1e3),
                     "stored_bytes": {k: q2 for k, q2 in s.query().items() if k.endswith("_bytes")}}}
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
        st2, rep2 = s2.solve_steady_host(xh)
        h2d = s2.query()["h2d_bytes"]
        s2.close()
        torch.cuda.synchronize()
        te += time.perf_counter() - t0
        e_it += rep2["total_krylov"]
    te = max_over_ranks(te * 1e3, device="cuda") / 1e3
    out["e2e"] = {"value": N * e_it / te, "unit": UNIT,
                  "h2d_bytes_per_step": int(h2d + img.nbytes), "d2h_bytes_per_step": int(8 * N),
                  "includes": "pmns_create (host setup + upload) + pmns_solve_steady_host + pmns_destroy"}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        prep = oracle_prepare(cfg, img)
        it, t = oracle_iters(prep, a.cpu_iters)
        out["cpu_baseline"] = {"value": N * it / t, "unit": UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"oracle on {a.config}: {it} FGMRES(MGS) iterations of Newton step 0 "
                                         f"with the prebuilt M_S, 1 thread ({t:.1f} s; build excluded)"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
