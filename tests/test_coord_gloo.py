"""A5 host-side coordination at world size 2 over gloo on CPU: the barrier,
the SUM all-reduce of per-rank dirty/image bytes (== sum of the per-rank
ORACLE values on each rank's own seeded region set) and the MAX of times."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import synth
    from oracle import oracle
    from paper_1808_00117_b200 import coord

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # each rank owns its own region set (different seed / shape per rank)
    S = synth.seed(4) + (rank << 20)
    o = oracle.Oracle()
    mems = []
    for r, (nb, P, mode) in enumerate([(16 * 4096 + 100 * rank, 4096, 0), (3 * 65536, 65536, 1)]):
        m = oracle.aligned_empty(nb)
        synth.fill_region(m, S, r)
        mems.append((m, P))
        o.register(m, P, mode)
    o.checkpoint_gather()
    for r, (m, P) in enumerate(mems):
        pages = synth.choose_dirty(S, 1, r, synth.n_pages(m.nbytes, P), 0.25 + 0.25 * rank)
        synth.apply_writer(m, P, pages, S, 1, r)

    def step():
        st, img, rep = o.checkpoint_gather()
        assert st == 0
        rep["t_total_ms"] = 1.0 + rank
        return rep

    g = coord.coordinated(step)
    out[rank] = (g.local["dirty_bytes"], g.local["image_bytes"], g.local["dirty_pages"], g.dirty_bytes,
                 g.image_bytes, g.dirty_pages, g.max_ms, g.world, coord.max_over_ranks(10.0 * rank))
    dist.destroy_process_group()


def test_coordinated_checkpoint_world2():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    loc = [res[r][:3] for r in range(world)]
    for r in range(world):
        _, _, _, db, ib, dp, mx, w, mo = res[r]
        assert db == sum(l[0] for l in loc)
        assert ib == sum(l[1] for l in loc)
        assert dp == sum(l[2] for l in loc)
        assert mx == 2.0 and w == 2 and mo == 10.0
    assert loc[0] != loc[1]  # the ranks really checkpointed different data


def test_coordinated_single_process_passthrough():
    import sys
    sys.path.insert(0, ROOT)
    from paper_1808_00117_b200 import coord
    g = coord.coordinated(lambda: {"dirty_bytes": 5, "image_bytes": 9, "dirty_pages": 1, "t_total_ms": 2.5})
    assert (g.dirty_bytes, g.image_bytes, g.dirty_pages, g.max_ms, g.world) == (5, 9, 1, 2.5, 1)


def _fail_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1808_00117_b200 import coord

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def bad_step():
        if rank == 1:
            raise RuntimeError("CRUM_E_CAPACITY on rank 1")
        return {"dirty_bytes": 1, "image_bytes": 2, "dirty_pages": 3, "t_total_ms": 1.0}

    try:
        coord.coordinated(bad_step)
        out[rank] = "no error"
    except coord.CoordinatedFailure as e:
        out[rank] = ("failed", e.local_error is not None)
    # the group stays aligned: the next coordinated step completes on both
    g = coord.coordinated(lambda: {"dirty_bytes": 1, "image_bytes": 2, "dirty_pages": 3, "t_total_ms": 1.0})
    out[10 + rank] = (g.dirty_bytes, g.image_bytes, g.dirty_pages)
    dist.destroy_process_group()


def test_coordinated_failure_raises_on_every_rank():
    """A local failure (e.g. CAPACITY) on one rank raises CoordinatedFailure
    on all ranks instead of leaving the others blocked in a collective."""
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_fail_worker, args=(world, port, out), nprocs=world, join=True, )
        res = dict(out)
    assert res[0] == ("failed", False) and res[1] == ("failed", True)
    assert res[10] == res[11] == (2, 4, 6)
