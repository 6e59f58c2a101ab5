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
    from paper_2510_22077_b200.dist import max_over_ranks, slab_owners
    t = max_over_ranks(10.0 + rank)
    rng = np.random.default_rng(3)
    cz = rng.uniform(0, 64, 50)
    work = rng.uniform(1, 10, 50) ** 3
    own = slab_owners(cz, work, 64, world)
    import torch
    allown = [torch.zeros(50, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allown, torch.tensor(own))
    q.put((rank, t, [a.numpy() for a in allown], own))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reduction_and_ownership():
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
    for rank, t, allown, own in res:
        assert t == 11.0                       # max over ranks of the device times
        assert np.array_equal(allown[0], allown[1])   # every rank agrees on ownership
        assert set(np.unique(own)) <= {0, 1}


def test_slab_owners_balance():
    from paper_2510_22077_b200.dist import slab_owners
    rng = np.random.default_rng(0)
    cz = rng.uniform(0, 256, 2000)
    work = rng.uniform(1, 5, 2000) ** 3
    for world in (2, 4, 8):
        own = slab_owners(cz, work, 256, world)
        loads = np.bincount(own, weights=work, minlength=world)
        assert loads.max() <= 1.05 * loads.mean()
        # slabs are contiguous in z
        for r in range(world - 1):
            assert cz[own == r].max() <= cz[own == r + 1].min()


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
    seg = s.export_layout()
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
