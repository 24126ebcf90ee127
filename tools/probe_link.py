"""Probe: HBM copy, copy-engine D2H/H2D, and SM-driven zero-copy D2H/H2D
bandwidth (kernel stores/loads to mapped pinned host memory), by grid size."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_1808_00117_b200 import crum

out = {}
s = torch.cuda.Stream()
def timeit(fn, reps=10):
    with torch.cuda.stream(s):
        for _ in range(3): fn()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps): fn()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
for n in (107374182 // 16 * 16, 1 << 30):
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t = timeit(lambda: crum.probe_copy(d2, d, n, 0, s)); out[f"d2d_kernel_{n}"] = 2 * n / t / 1e9
    t = timeit(lambda: h.copy_(d, non_blocking=True)); out[f"d2h_ce_{n}"] = n / t / 1e9
    t = timeit(lambda: d.copy_(h, non_blocking=True)); out[f"h2d_ce_{n}"] = n / t / 1e9
    for blocks in (148, 296, 592, 1184, 2368):
        t = timeit(lambda: crum.probe_copy(h, d, n, blocks, s), reps=5); out[f"d2h_zerocopy_{n}_b{blocks}"] = n / t / 1e9
        t = timeit(lambda: crum.probe_copy(d, h, n, blocks, s), reps=5); out[f"h2d_zerocopy_{n}_b{blocks}"] = n / t / 1e9
    # concurrent: zero-copy D2H while an HBM read-heavy kernel runs on another stream
    del d, d2, h
for k, v in out.items(): print(f"{k:40s} {v:9.1f} GB/s")
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_link.json", "w"), indent=1)
