"""Standalone J-apply bandwidth at an HBM-bound size.

Usage: python scripts/bench_jacobian.py cfg4 [reps] [key=value ...]
Creates the context (setup only; no preconditioner), then times `reps`
applies y = J(x) v (unfused, a10) and y = b - J(x) v (fused, a6/a8) with CUDA
events on the launching stream, for the cell-record kernel (PMNS_JREC=1) and
the per-row-table kernel (PMNS_JREC=0).  The working set (x, v, y, b: 4 x 8N
bytes plus index data) is far larger than the 126 MB L2 at config 4, so no
flush is needed.  Bytes = SURVEY 8(d) B_J = 8(2N + n_f) (+8N fused).  The state
is a seeded N(0,1) field scaled to 0.05 m/s (bandwidth depends on the data only
through the upwind pattern).  Prints one JSON line.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.geometry import load_config, make_image  # noqa: E402
from synth.vectors import seeded_normal  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = load_config(name)
for k, v in (("p_in", 1000.0), ("dt", 0.0), ("ws_merge_h", 0.5), ("ws_min_cells", 50)):
    if cfg.get(k) is None:
        cfg[k] = v
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1)
    cfg[k] = float(v)
img = make_image(cfg)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
out = {"config": name, "reps": reps}
for flag in ("1", "0"):
    os.environ["PMNS_JREC"] = flag
    from paper_2510_22077_b200 import Solver
    s = Solver(cfg, img, device=0)
    q = s.query()
    N, nf = q["N"], q["n_f"]
    x = torch.tensor(seeded_normal(N, 3) * 0.05, dtype=torch.float64, device="cuda")
    v = torch.tensor(seeded_normal(N, 7), dtype=torch.float64, device="cuda")
    y = torch.empty_like(v)
    b = torch.tensor(seeded_normal(N, 9), dtype=torch.float64, device="cuda")
    res = {}
    for fused in (False, True):
        for _ in range(3):
            s.apply_jacobian(x, v, y, b=b if fused else None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            s.apply_jacobian(x, v, y, b=b if fused else None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        by = 8 * (2 * N + nf) + (8 * N if fused else 0)
        res["fused" if fused else "plain"] = {"ms": ms, "GBps": by / ms / 1e6, "frac": by / ms / 1e6 / peak,
                                              "bytes": by}
    out["jrec" if flag == "1" else "table"] = res
    out["N"] = N
    out["n_f"] = nf
    s.close()
out["peak_GBps"] = peak
print(json.dumps(out))
