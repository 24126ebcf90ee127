"""A5: coordinated multi-rank checkpoint.

CRUM's coordinated checkpoint quiesces every rank before draining and
finishes with a global view of what was saved.
Here each rank owns one GPU and one crum_ctx; page bytes never cross GPUs, so
the only collectives are:

  1. barrier() before A1 (every rank's application epoch has finished),
  2. all_reduce(MAX) of a failure flag: a rank whose checkpoint raised (e.g.
     CAPACITY, BUSY) makes EVERY rank raise CoordinatedFailure instead of
     leaving the others blocked in the next collective,
  3. all_reduce(SUM) of int64 {dirty bytes, image bytes, dirty pages},
  4. all_reduce(MAX) of the per-rank checkpoint time (device events).

`local_step` is the per-rank checkpoint (e.g. a bound
Context.checkpoint_gather call) returning a crum report dict; keeping it a
callable lets the host-side logic be tested with the gloo backend on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


class CoordinatedFailure(RuntimeError):
    """The coordinated checkpoint failed on at least one rank (raised on all)."""

    def __init__(self, msg: str, local_error: BaseException | None = None):
        super().__init__(msg)
        self.local_error = local_error


@dataclass
class GlobalReport:
    local: dict
    dirty_bytes: int
    image_bytes: int
    dirty_pages: int
    max_ms: float
    world: int


def _device_for(group) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def coordinated(local_step, group=None, time_key: str = "t_total_ms") -> GlobalReport:
    """Run one coordinated checkpoint step across the process group."""
    if not dist.is_available() or not dist.is_initialized():
        rep = local_step()
        return GlobalReport(rep, rep["dirty_bytes"], rep["image_bytes"], rep["dirty_pages"],
                            float(rep.get(time_key, 0.0)), 1)
    dev = _device_for(group)
    dist.barrier(group)
    err = None
    try:
        rep = local_step()
    except Exception as e:  # surfaced on every rank below
        err, rep = e, None
    failed = torch.tensor([1 if err is not None else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(failed, op=dist.ReduceOp.MAX, group=group)
    if int(failed.item()):
        if err is not None:
            raise CoordinatedFailure(f"rank {dist.get_rank(group)}: {err}", err) from err
        raise CoordinatedFailure("coordinated checkpoint failed on another rank")
    sums = torch.tensor([rep["dirty_bytes"], rep["image_bytes"], rep["dirty_pages"]], dtype=torch.int64, device=dev)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    t = torch.tensor([float(rep.get(time_key, 0.0))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    s = sums.tolist()
    return GlobalReport(rep, int(s[0]), int(s[1]), int(s[2]), float(t.item()), dist.get_world_size(group))


def max_over_ranks(x: float, group=None) -> float:
    """Device-timed quantities are reported as the max over ranks."""
    if not dist.is_available() or not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
