"""N > 1 host logic on CPU with world_size-2 gloo process groups."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_22077_b200.dist import max_over_ranks
    t = max_over_ranks(10.0 + rank)
    q.put((rank, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    """bench.py's device time is the max over ranks."""
    pytest.importorskip("torch")
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(t == 11.0 for _, t in res)


def _worker_partition(rank, world, port, q):
    """Each rank builds the host-only context of the same image, takes its
    primary range from pmns_set_comm (partition only) and the ranks compare
    their ranges over gloo."""
    import sys
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from synth.geometry import load_config, make_image
    from paper_2510_22077_b200 import Solver
    cfg = load_config("cfg1")
    s = Solver(cfg, make_image(cfg), device=-1)
    s.set_comm(rank, world, None)
    qy = s.query()
    mine = torch.tensor([qy["own_lo"], qy["own_hi"], qy["n_p"], qy["rank"], qy["world"]], dtype=torch.int64)
    allr = [torch.zeros(5, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, mine)
    q.put((rank, [a.numpy() for a in allr]))
    s.close()
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_primary_partition():
    """pmns_set_comm ownership: contiguous, disjoint, covering,
    identical on every rank, balanced by the dense front bytes."""
    pytest.importorskip("torch")
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_partition, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    views = {rank: allr for rank, allr in res}
    assert all(np.array_equal(views[0][r], views[1][r]) for r in range(world))
    ranges = views[0]
    n_p = int(ranges[0][2])
    assert [int(x[3]) for x in ranges] == [0, 1] and all(int(x[4]) == 2 for x in ranges)
    assert int(ranges[0][0]) == 0 and int(ranges[-1][1]) == n_p
    for r in range(world - 1):
        assert int(ranges[r][1]) == int(ranges[r + 1][0])   # contiguous, disjoint
    assert all(int(x[1]) > int(x[0]) for x in ranges)        # every rank owns something


def _worker_halo(rank, world, port, q):
    """Host-only context: this rank's multi-GPU plan (pmns_halo_plan), checked
    against the other ranks' plans over gloo and against the oracle's Jacobian
    sparsity (an independent source of the stencil couplings)."""
    import sys
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from synth.geometry import random_blobs
    from synth.vectors import seeded_normal
    from paper_2510_22077_b200 import Solver
    from oracle.grid import build_grid
    from oracle.mac import Mac
    cfg = dict(dim=3, periodic=[True, True], h=1e-5, rho=1000.0, mu=1e-3, body_force=[0.0, 0.0, 0.0], p_in=150.0,
               p_out=0.0, dt=0.0, ws_merge_h=0.5, ws_min_cells=10, dual_layers=1, mask_band=2)
    img = random_blobs(24, 20, 20, 0.45, 2.5, 9)
    s = Solver(cfg, img, device=-1)
    plan, ranges = s.halo_plan(rank, world)
    perm = s.export_layout()["perm"]       # device slot -> canonical index
    N = s.N
    objs = [None] * world
    dist.all_gather_object(objs, (plan, ranges))
    # oracle Jacobian at a flow state: the couplings of every row (canonical)
    g = build_grid(img, 3, [True, True], 1e-5)
    mac = Mac(g, 1000.0, 1e-3, p_in=150.0)
    J = mac.jacobian(seeded_normal(g.N, 3) * 0.05).tocsr()
    inv = np.empty(N, dtype=np.int64)
    inv[perm] = np.arange(N)
    own = np.zeros(N, dtype=bool)
    for lo, hi in ranges:
        own[lo:hi] = True
    rows = perm[np.nonzero(own)[0]]
    need = np.unique(inv[J[rows].indices])
    need = need[~own[need]]
    q.put((rank, objs, need, N))
    s.close()
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_halo_plan():
    """SURVEY 8(e) halo lists: the ranks' owned unknowns (three contiguous
    device-order ranges each) partition all unknowns; rank p's forward send
    list to q is q's receive list from p (and the same for the reverse dual
    partial sums); every slot is received from its owner; and the forward
    halo covers every non-owned column of the owned rows of the oracle's
    Jacobian."""
    pytest.importorskip("torch")
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_halo, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, objs, need, N = q.get(timeout=240)
        res[rank] = (objs, need, N)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    objs = res[0][0]
    N = res[0][2]
    owner = np.full(N, -1)
    for r, (plan, ranges) in enumerate(objs):
        for lo, hi in ranges:
            assert np.all(owner[lo:hi] == -1)
            owner[lo:hi] = r
    assert np.all(owner >= 0)                        # a partition of all unknowns
    for p in range(world):
        plan_p = objs[p][0]
        for r in range(world):
            if r == p:
                continue
            plan_r = objs[r][0]
            assert np.array_equal(plan_p[(r, "fwd_send")], plan_r[(p, "fwd_recv")])
            assert np.array_equal(plan_p[(r, "rev_send")], plan_r[(p, "rev_recv")])
            assert np.all(owner[plan_p[(r, "fwd_recv")]] == r)
            assert np.all(owner[plan_p[(r, "rev_send")]] == r)
        got = np.concatenate([plan_p[(r, "fwd_recv")] for r in range(world) if r != p])
        need = res[p][1]
        assert np.all(np.isin(need, got)), np.setdiff1d(need, got)[:10]
        assert len(need) > 0                          # the slabs do touch


@pytest.mark.parametrize("world", [2, 3, 8])
def test_slab_partition_is_contiguous_and_balanced(world):
    """pmns_halo_plan's owned primary-row ranges (the partition pmns_set_comm
    uses: primary_cuts) tile the primary rows in rank order, end at the total
    number of primary rows, and leave no rank empty while there are at least
    as many primaries as ranks (config 2: 105 primaries; the round-1
    proportional prefix split could leave a rank empty)."""
    from synth.geometry import load_config, make_image
    from paper_2510_22077_b200 import Solver
    cfg = load_config("cfg2")
    s = Solver(cfg, make_image(cfg), device=-1)
    q = s.query()
    assert q["n_p"] >= world
    lo_expected = 0
    sizes = []
    for r in range(world):
        _, ranges = s.halo_plan(r, world)
        lo, hi = ranges[0]
        assert lo == lo_expected and hi >= lo
        lo_expected = hi
        sizes.append(hi - lo)
    lab = s.export_layout()["label"]
    cells = np.bincount(lab[lab >= 0], minlength=q["n_p"])
    # primary rows = all slots before the interface segments
    assert lo_expected == q["N"] - (q["n_c"] - cells.sum()) - _iface_faces(s, q, cells)
    assert min(sizes) > 0
    s.close()


def _iface_faces(s, q, cells):
    """Face unknowns owned by interfaces = N - primary rows - interface cells,
    recovered from the last rank's plan of a 1-rank partition."""
    _, ranges = s.halo_plan(0, 1)
    prim_rows = ranges[0][1] - ranges[0][0]
    return q["N"] - prim_rows - (q["n_c"] - int(cells.sum()))
