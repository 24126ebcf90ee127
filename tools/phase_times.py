"""Per-phase device times of the C2 compare step (CRUM_CFG_TIMING events)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import synth
from paper_1808_00117_b200 import crum
GiB = 1 << 30
for mode, P in ((crum.MODE_COMPARE, 65536), (crum.MODE_HASH, 65536), (crum.MODE_COMPARE, 4096)):
    ctx = crum.Context(0, timing=True)
    t = torch.empty(GiB, dtype=torch.uint8, device="cuda")
    crum.synth_fill(t, GiB, 1, 0)
    rid = ctx.register_region(t, GiB, P, mode)
    ctx.sync_shadow()
    cap = ctx.image_required_bytes()
    buf = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    n = GiB // P
    reps = []
    for e in range(1, 13):
        pg = torch.from_numpy(synth.choose_dirty(1, e, 0, n, 0.1).astype(np.uint32)).cuda()
        crum.synth_write_pages(t, GiB, P, pg, pg.numel(), 1, e, 0)
        crum.synth_scrub(scrub, scrub.numel())
        ctx.checkpoint_gather_device(buf, cap, report=False)
        reps.append(ctx.last_report())
    keys = ("t_detect_ms", "t_compact_ms", "t_gather_ms", "t_total_ms")
    print(mode, P, {k: round(float(np.median([r[k] for r in reps[4:]])), 4) for k in keys})
