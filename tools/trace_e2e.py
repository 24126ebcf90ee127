"""Run the pinned-host checkpoint path a few times with the context flag
CRUM_CFG_TRACE (per-range / per-chunk times on stderr; C2).

usage: trace_e2e.py [page_size] [dirty] [--compress] [--content random|half|hpgmg]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import synth
import bench
from paper_1808_00117_b200 import crum
GiB = 1 << 30
argv = [a for a in sys.argv[1:] if not a.startswith("--")]
P = int(argv[0]) if len(argv) > 0 else 65536
d = float(argv[1]) if len(argv) > 1 else 0.1
compress = "--compress" in sys.argv
content = sys.argv[sys.argv.index("--content") + 1] if "--content" in sys.argv else "random"
flags = crum.COMPRESS if compress else 0
s = torch.cuda.Stream()
ctx = crum.Context(0, flags=crum.CFG_TRACE)
t = torch.empty(GiB, dtype=torch.uint8, device="cuda")
S = synth.seed(1)
crum.synth_fill(t, GiB, S, 0, stream=s)
torch.cuda.synchronize()
if content == "half":
    t[GiB // 2:].view(torch.float32).fill_(0.25)
elif content == "hpgmg":
    bench.hpgmg_fill_device(t, 0)
torch.cuda.synchronize()
ctx.register_region(t, GiB, P, 0)
img = ctx.new_image()
ctx.checkpoint_gather(img, stream=s, flags=flags)
for e in range(1, 4):
    pg = torch.from_numpy(synth.choose_dirty(S, e, 0, GiB // P, d).astype(np.uint32)).cuda()
    crum.synth_write_pages(t, GiB, P, pg, pg.numel(), S, e, 0, stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.checkpoint_gather(img, stream=s, flags=flags)
    print(f"wall {1e3*(time.perf_counter()-t0):.3f} ms  rep t_total {rep['t_total_ms']:.3f} t_copy {rep['t_copy_ms']:.3f}"
          f"  image {img.length}", file=sys.stderr)
