"""Memory plan of a config's local operators for a list of decomposition parameters
(pmns_memory_plan: structural nested-dissection plans only, no numeric build).

Usage: python scripts/memplan.py cfg4 h_m:n_min [h_m:n_min ...]
Prints one JSON line per (h_m, n_min): N^p, N^c, stored M_p / M_d bytes, factorisation
flops, the largest primary block and front.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from synth.geometry import load_config, make_image  # noqa: E402
from paper_2510_22077_b200 import Solver  # noqa: E402

name = sys.argv[1]
cfg0 = load_config(name)
img = make_image(cfg0)
for spec in sys.argv[2:]:
    hm, nmin = spec.split(":")
    cfg = dict(cfg0)
    cfg["ws_merge_h"] = float(hm)
    cfg["ws_min_cells"] = int(nmin)
    for k, v in (("p_in", 1000.0), ("dt", 0.0)):
        if cfg.get(k) is None:
            cfg[k] = v
    t0 = time.time()
    s = Solver(cfg, img, device=0)
    q = s.query()
    t1 = time.time()
    m = s.memory_plan()
    t2 = time.time()
    out = {"config": name, "h_m": float(hm), "n_min": int(nmin), "N": q["N"], "N_p": q["n_p"], "N_c": q["n_iface"],
           "dual_unknowns": q["dual_unknowns"], "t_create_s": round(t1 - t0, 1), "t_plan_s": round(t2 - t1, 1)}
    out.update(m)
    out["mp_GB"] = round(m["mp_bytes"] / 1e9, 2)
    out["md_GB"] = round(m["md_bytes"] / 1e9, 2)
    out["stencil_mean_run"] = round(q["N"] / max(m["stencil_runs"], 1), 2)
    print(json.dumps(out), flush=True)
    s.close()
