"""Run the pinned-host checkpoint path a few times with the context flag
CRUM_CFG_TRACE (per-range times on stderr; C2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import synth
from paper_1808_00117_b200 import crum
GiB = 1 << 30
P = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
d = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
s = torch.cuda.Stream()
ctx = crum.Context(0, flags=crum.CFG_TRACE)
t = torch.empty(GiB, dtype=torch.uint8, device="cuda")
S = synth.seed(1)
crum.synth_fill(t, GiB, S, 0, stream=s)
ctx.register_region(t, GiB, P, 0)
img = ctx.new_image()
ctx.checkpoint_gather(img, stream=s)
for e in range(1, 4):
    pg = torch.from_numpy(synth.choose_dirty(S, e, 0, GiB // P, d).astype(np.uint32)).cuda()
    crum.synth_write_pages(t, GiB, P, pg, pg.numel(), S, e, 0, stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.checkpoint_gather(img, stream=s)
    print(f"wall {1e3*(time.perf_counter()-t0):.3f} ms  rep t_total {rep['t_total_ms']:.3f} t_copy {rep['t_copy_ms']:.3f}", file=sys.stderr)
