"""C1 latency anatomy (profiling aid, GPU): per-call time of a 4 MiB / 4 KiB /
1 % checkpoint into an HBM image, cold (L2 scrubbed between calls) and warm,
with and without the context's timing events, and the kernel durations the
CUDA profiler (CUPTI) sees for the same calls.

    python tools/c1_latency.py
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_00117_b200 import crum  # noqa: E402

MiB, KiB = 1 << 20, 1 << 10


def run(timing, cold, steps=200, warm=20, profile=False, flags=0):
    ctx = crum.Context(0, timing=timing, flags=flags)
    F, P = 4 * MiB, 4 * KiB
    x = torch.randint(0, 255, (F,), dtype=torch.uint8, device="cuda")
    ctx.register_region(x, F, P, crum.MODE_COMPARE)
    cap = ctx.image_required_bytes()
    img = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
    scrub = torch.empty(256 * MiB, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    g = torch.Generator(device="cpu").manual_seed(1)
    N = F // P
    pages = [torch.randperm(N, generator=g)[: N // 100].cuda() * P for _ in range(8)]
    ctx.checkpoint_gather_device(img, cap, stream=s, report=True)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    prof = None
    if profile:
        prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
    with torch.cuda.stream(s):
        for i in range(warm + steps):
            if i == warm and prof is not None:
                prof.__enter__()
            x[pages[i % 8]] += 1  # the application writes ~1 % of the pages
            if cold:
                scrub.fill_(i & 0xff)
            if i >= warm:
                ev0[i - warm].record(s)
            ctx.checkpoint_gather_device(img, cap, stream=s, report=False)
            if i >= warm:
                ev1[i - warm].record(s)
    torch.cuda.synchronize()
    kern = {}
    if prof is not None:
        prof.__exit__(None, None, None)
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA and "crum" in e.name:
                kern.setdefault(e.name.split("(")[0], []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    t = [a.elapsed_time(b) * 1e3 for a, b in zip(ev0, ev1)]
    rep = ctx.last_report()
    ctx.close()
    return {"timing": timing, "cold": cold, "flags": flags, "us_median": round(statistics.median(t), 2),
            "us_mean": round(statistics.mean(t), 2), "us_min": round(min(t), 2),
            "path": rep.get("path"), "dirty_pages": rep.get("dirty_pages"),
            "kernels_us": {k: round(statistics.median(v), 2) for k, v in kern.items()}}


def main():
    out = []
    for timing in (False, True):
        for cold in (True, False):
            out.append(run(timing, cold))
    out.append(run(False, True, profile=True))
    out.append(run(False, True, flags=crum.CFG_NO_GRAPH))
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
