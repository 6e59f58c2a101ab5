"""Communication volume of the slab-owned Krylov phase from the host-side plan
(pmns_halo_plan on a host-only context: no GPU needed), and a MODELLED parallel efficiency -- not a measurement:
N > 1 could not be run on hardware in this round.

Per FGMRES iteration a rank receives its forward halo 3 times (s, z_d, z) and sends its dual partial sums once
(reverse halo), 8 bytes per slot, plus 4 small allreduces (coarse RHS: 8 n_coarse bytes; CGS2: 8 (j+1) bytes twice;
the norm).  Model: T_iter(N) = T_iter(1) * max_r share_r + bytes_r / BW + 7 * latency, share_r = the rank's share
of sum n_i^(4/3) over its owned primaries (a proxy for the M_p bytes it streams; its share of sum n_i^2, the dense
front flops, bounds the build's efficiency),
BW = 900 GB/s per direction (NVLink 5), latency = 10 us per exchange or allreduce.

Usage: python scripts/halo_model.py cfg3 9.1 [cfg4 ms_per_iter ...]   (ms per iteration measured on 1 GPU, or 0)
Prints one JSON line per (config, world)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

BW = 900e9
LAT = 10e-6
args = sys.argv[1:]
for name, t1 in zip(args[0::2], args[1::2]):
    t1 = float(t1) * 1e-3
    cfg = load_config(name)
    s = Solver(cfg, make_image(cfg), device=-1)
    q = s.query()
    lay = s.export_layout()
    lab = lay["label"]
    n_p = q["n_p"]
    # unknowns per primary ~ 4 x its cells (faces shared): the balance weight n_i^2 uses the segment sizes, which
    # the host-only context does not export; cells^2 is the same criterion up to a constant
    cells = np.bincount(lab[lab >= 0], minlength=n_p).astype(float)
    for world in (2, 4, 8):
        worst_bytes, worst_share, rows = 0, 0.0, []
        for r in range(world):
            plan, ranges = s.halo_plan(r, world)
            fwd = sum(len(v) for (p, k), v in plan.items() if k == "fwd_recv")
            rev = sum(len(v) for (p, k), v in plan.items() if k == "rev_send")
            snd = sum(len(v) for (p, k), v in plan.items() if k == "fwd_send")
            by = 8 * (3 * max(fwd, snd) + rev)
            worst_bytes = max(worst_bytes, by)
            rows.append(ranges[0][1] - ranges[0][0])
        # the library's cuts (primary_cuts: bottleneck-optimal contiguous ranges) recovered from the owned row
        # counts: unknowns per primary ~ cells x (primary rows / primary cells)
        crow = np.concatenate([[0.0], np.cumsum(cells)]) * (float(sum(rows)) / max(cells.sum(), 1.0))
        cuts = [0] + [int(np.argmin(np.abs(crow - c))) for c in np.cumsum(rows)]
        cuts[-1] = n_p
        n2, n43 = cells ** 2, cells ** (4.0 / 3.0)
        shares_build = [n2[cuts[k]:cuts[k + 1]].sum() / n2.sum() for k in range(world)]
        shares_apply = [n43[cuts[k]:cuts[k + 1]].sum() / n43.sum() for k in range(world)]
        worst_share = max(shares_apply)
        t_comm = worst_bytes / BW + 7 * LAT
        out = dict(config=name, world=world, N=q["N"], N_p=n_p, N_c=q["n_iface"],
                   max_rank_exchange_bytes_per_iter=int(worst_bytes),
                   exchange_bytes_over_8N=round(worst_bytes / (8.0 * q["N"]), 4),
                   owned_primary_rows=rows, max_share_apply_n43=round(max(shares_apply), 4),
                   max_share_build_n2=round(max(shares_build), 4),
                   t_comm_us=round(t_comm * 1e6, 1), kind="model (not measured)")
        if t1 > 0:
            tN = t1 * worst_share + t_comm
            out["t_iter_1gpu_ms"] = t1 * 1e3
            out["t_iter_model_ms"] = round(tN * 1e3, 3)
            out["efficiency_model_krylov"] = round(t1 / (world * tN), 3)
            out["efficiency_bound_build"] = round(1.0 / (world * max(shares_build)), 3)
        print(json.dumps(out), flush=True)
    s.close()
