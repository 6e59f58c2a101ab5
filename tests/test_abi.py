"""The C-ABI library loads (no GPU needed) and exports every entry point that
include/pmns.h declares; host-only contexts report errors through the ABI."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pmns.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmns_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    from paper_2510_22077_b200 import LIB_PATH
    lib = ctypes.CDLL(LIB_PATH)
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2510_22077_b200._lib import EXPORTED
    assert set(_declared()) <= set(EXPORTED)


def test_host_only_context_and_errors():
    from paper_2510_22077_b200 import Solver, PmnsError
    from synth.geometry import slit_2d
    cfg = dict(dim=2, periodic=[False, False], h=1e-5, rho=1e3, mu=1e-3, body_force=[0, 0, 0], p_in=1.0,
               p_out=0.0, dt=0.0, ws_merge_h=1.0, ws_min_cells=3, dual_layers=1, mask_band=2)
    s = Solver(cfg, slit_2d(8, 3), device=-1)
    assert s.query()["n_p"] == 1
    with pytest.raises(PmnsError) as e:       # device calls on a host-only context
        s.build_preconditioner(None)
    assert e.value.status == 9
    s.close()
    img = np.ones((1, 5, 5), dtype=np.uint8)   # no percolating void
    img[0, 2, 2] = 0
    with pytest.raises(PmnsError) as e:
        Solver(cfg, img, device=-1)
    assert e.value.status == 2


def test_no_library_kernels_linked():
    """The hot path and the build run in the library's own kernels: the shared
    object links neither cuBLAS nor cuSOLVER (NEEDED entries of the ELF)."""
    from paper_2510_22077_b200 import LIB_PATH
    import subprocess
    out = subprocess.run(["readelf", "-d", LIB_PATH], capture_output=True, text=True).stdout
    needed = re.findall(r"\(NEEDED\)\s+Shared library: \[([^\]]+)\]", out)
    assert needed, out
    assert not [n for n in needed if "cublas" in n or "cusolver" in n or "cusparse" in n], needed
