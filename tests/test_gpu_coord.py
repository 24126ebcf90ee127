"""A5 on the CUDA path (SURVEY.md sec. 8(a) row A5, sec. 8(c) "A5 invariant";
PAPER.md:531-534, 965-969): two ranks (gloo, both on cuda:0 -- the pool's
boxes have one GPU) each register their OWN seeded region set with
libcrum.so and checkpoint it under coord.coordinated (barrier, failure flag,
SUM of {dirty bytes, image bytes, dirty pages}, MAX of the time).  Each rank
also runs the CPU oracle on identical inputs.  Checked:
  * every rank's pinned image equals its oracle image byte for byte,
  * the all-reduced sums equal the sum over ranks of the ORACLE values,
  * a CAPACITY failure on one rank raises on both, commits nothing on the
    failing rank, and the next coordinated checkpoint still agrees."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KiB, MiB = 1 << 10, 1 << 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _specs(rank):
    # different shapes per rank (ragged tails, both modes, 4 KiB .. 2 MiB pages)
    return [(64 * MiB + 4096 * rank, 64 * KiB, 0), (3 * 2 * MiB + 777, 2 * MiB, 1),
            (1 * MiB + 100 * rank + 12, 4 * KiB, 1), (40 * 4 * KiB, 4 * KiB, 0)]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch.distributed as dist

    import synth
    from paper_1808_00117_b200 import coord, crum
    from tests.gpu_pair import Pair

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S = synth.seed(4) + (rank << 20)
    p = Pair(_specs(rank), S)
    img = p.g.new_image()
    res = {}
    for epoch, d in ((0, 0.0), (1, 0.1 + 0.2 * rank), (2, 0.0), (3, 0.5)):
        if epoch:
            p.write(epoch, d)
        st, want, rep_o = p.o.checkpoint_gather()
        assert st == 0
        g = coord.coordinated(lambda: p.g.checkpoint_gather(img))
        ok = img.tobytes() == want.tobytes()
        res[epoch] = dict(ok=ok, oracle=(rep_o["dirty_bytes"], rep_o["image_bytes"], rep_o["dirty_pages"]),
                          glob=(g.dirty_bytes, g.image_bytes, g.dirty_pages), world=g.world, max_ms=g.max_ms,
                          local_ms=g.local["t_total_ms"])
    # CAPACITY on rank 1 only: both ranks raise, rank 1 commits nothing
    p.write(4, 0.3)
    small = p.g.new_image(4096 if rank == 1 else img.capacity)
    try:
        coord.coordinated(lambda: p.g.checkpoint_gather(small))
        res["fail"] = "no error"
    except coord.CoordinatedFailure as e:
        res["fail"] = "raised:" + ("local" if e.local_error is not None else "remote")
    # rank 0 committed its epoch-4 checkpoint, rank 1 did not: the oracle of
    # rank 0 follows (its gather succeeded), rank 1's oracle skips it
    if rank == 0:
        p.o.checkpoint_gather()
    p.write(5, 0.2)
    st, want, rep_o = p.o.checkpoint_gather()
    g = coord.coordinated(lambda: p.g.checkpoint_gather(img))
    res[5] = dict(ok=img.tobytes() == want.tobytes(),
                  oracle=(rep_o["dirty_bytes"], rep_o["image_bytes"], rep_o["dirty_pages"]),
                  glob=(g.dirty_bytes, g.image_bytes, g.dirty_pages), world=g.world, max_ms=g.max_ms,
                  local_ms=g.local["t_total_ms"])
    res["regions_equal"] = p.regions_equal() and p.shadows_equal()
    out[rank] = res
    dist.destroy_process_group()


def test_coordinated_checkpoint_on_gpu_matches_oracle_sums():
    assert torch.cuda.is_available()
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for epoch in (0, 1, 2, 3, 5):
        want_sum = tuple(sum(res[r][epoch]["oracle"][i] for r in range(world)) for i in range(3))
        for r in range(world):
            e = res[r][epoch]
            assert e["ok"], (r, epoch)                       # per-rank image == oracle image
            assert e["glob"] == want_sum, (r, epoch)         # all-reduced == sum of oracle values
            assert e["world"] == world
            assert e["max_ms"] == max(res[q][epoch]["local_ms"] for q in range(world))
    assert res[0][1]["oracle"] != res[1][1]["oracle"]       # the ranks checkpointed different data
    assert res[0]["fail"] == "raised:remote" and res[1]["fail"] == "raised:local"
    assert res[0]["regions_equal"] and res[1]["regions_equal"]
