"""Multi-rank Krylov phase on ONE GPU: `world` virtual ranks,
each a context driven by its own host thread, joined by the library's
in-process loopback transport (host-synchronised device copies for the halo
exchanges and allreduces; no kernel waits on another).  The distributed solve
(slab-owned unknowns, halo-exchanged J, distributed CGS2, reverse-halo M_d,
coarse-RHS allreduce with a replicated coarse solve) must reproduce the
one-rank solve: same Newton counts, FGMRES counts within +-1 per Newton step,
fields <= 1e-10 (SURVEY 8(e) "parity across GPU counts").  Marked gpu."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.geometry import load_config, make_image, random_blobs  # noqa: E402


def _cfg(dim, per, hm, nmin, p_in=300.0, bf=(0.0, 0.0, 0.0), dt=0.0):
    return dict(dim=dim, periodic=list(per), h=1e-5, rho=1000.0, mu=1e-3, body_force=list(bf),
                p_in=p_in, p_out=0.0, dt=dt, ws_merge_h=hm, ws_min_cells=nmin, dual_layers=1, mask_band=2)


CASES = {
    "blob3d_per": lambda: (_cfg(3, (True, True), 0.5, 10, p_in=150.0), random_blobs(24, 20, 20, 0.45, 2.5, 9)),
    "cfg2": lambda: (load_config("cfg2"), make_image(load_config("cfg2"))),
}


def _canon(s, x):
    out = torch.empty_like(x)
    s.permute(x, out, to_canonical=True)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _run(name, world, how="steady"):
    from paper_2510_22077_b200 import Solver
    from paper_2510_22077_b200._lib import loopback_create, loopback_destroy
    cfg, img = CASES[name]()
    group = loopback_create(world)
    res = [None] * world

    def worker(r):
        s = None
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                s = Solver(cfg, img, device=0)
                s.set_comm_loopback(r, world, group)
                x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
                if how == "steady":
                    code, rep = s.solve_steady(x)
                else:
                    code, rep = s.solve_continuation(x, 2)
                st.synchronize()
                res[r] = (code, rep, _canon(s, x), s.query())
        except Exception as e:   # noqa: BLE001
            res[r] = e
        finally:
            if s is not None:
                s.close()         # before the group is destroyed

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    loopback_destroy(group)
    for r in res:
        if isinstance(r, Exception):
            raise r
    return res, cfg, img


def _one_rank(cfg, img, how="steady"):
    from paper_2510_22077_b200 import Solver
    s = Solver(cfg, img, device=0)
    x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
    code, rep = s.solve_steady(x) if how == "steady" else s.solve_continuation(x, 2)
    out = (code, rep, _canon(s, x), s.query())
    s.close()
    return out


def _compare(res, ref):
    code1, rep1, x1, q1 = ref
    nf = q1["n_f"]
    assert code1 == 0
    k1 = rep1["krylov_iters"][:rep1["newton_iters"]]
    for code, rep, x, q in res:
        assert code == 0 and rep["converged"]
        assert rep["newton_iters"] == rep1["newton_iters"]
        k = rep["krylov_iters"][:rep["newton_iters"]]
        assert all(abs(a - b) <= 1 for a, b in zip(k, k1)), (k, k1)
        for blk in (slice(0, nf), slice(nf, None)):
            err = np.linalg.norm(x[blk] - x1[blk]) / np.linalg.norm(x1[blk])
            assert err <= 1e-10, err


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", list(CASES))
def test_loopback_steady_matches_one_rank(name, world):
    res, cfg, img = _run(name, world)
    owned = sorted(q["own_lo"] for _, _, _, q in res)
    assert len(set(owned)) == world            # disjoint primary slabs
    _compare(res, _one_rank(cfg, img))


def test_loopback_continuation_matches_one_rank():
    res, cfg, img = _run("blob3d_per", 2, how="continuation")
    _compare(res, _one_rank(cfg, img, how="continuation"))
