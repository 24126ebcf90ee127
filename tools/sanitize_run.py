"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel of libcrum.so runs at least once on a
mixed-mode, ragged-tail region set, and the result is checked against the
oracle so a sanitizer-silent run is also a correct one."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import synth
from tests.gpu_pair import Pair
from paper_1808_00117_b200 import crum
KiB, MiB = 1 << 10, 1 << 20
SPECS = [(256 * KiB, 4 * KiB, 0), (3 * 64 * KiB + 1234, 64 * KiB, 1), (5 * 4 * KiB + 17, 4 * KiB, 1),
         (2 * MiB + 100, 2 * MiB, 1), (12 * KiB + 256, 4 * KiB, 0), (2 * 64 * KiB, 64 * KiB, 0)]
p = Pair(SPECS, synth.seed(42), chunk_bytes=64 * KiB)
assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags())
assert p.g.sync_shadow() == p.o.sync_shadow()
img = p.g.new_image()
for e, d in ((1, 0.3), (2, 0.0), (3, 1.0)):
    p.write(e, d)
    st, want, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes(), e
p.write(4, 0.5)
st, want, _ = p.o.checkpoint_gather()
cap = p.g.image_required_bytes()
dimg = torch.zeros(cap + 256, dtype=torch.uint8, device="cuda")
p.g.checkpoint_gather_device(dimg, cap)
assert dimg[:len(want)].cpu().numpy().tobytes() == want.tobytes()
q = crum.Context(0, chunk_bytes=64 * KiB)
zs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for nb, _, _ in SPECS]
for z, (nb, P, m) in zip(zs, SPECS):
    q.register_region(z, nb, P, m)
full = p.g.new_image()
p.g.checkpoint_gather(full, flags=crum.FULL)
q.restore_scatter(full, flags=crum.VERIFY)
q.restore_scatter_device(dimg, len(want), flags=crum.VERIFY)
torch.cuda.synchronize()
assert all(np.array_equal(z.cpu().numpy(), h) for z, h in zip(zs, p.host))
# compressed images: host (ring + copy engine) and device gathers, restore (eager, lazy)
for h, d in zip(p.host, p.dev):
    h[h.nbytes // 2:] = 0
    d.copy_(torch.from_numpy(h))
torch.cuda.synchronize()
p.g.mark_dirty(1, 0, SPECS[0][0])
p.o.mark_dirty(1, 0, SPECS[0][0])
zimg = p.g.new_image()
for e, d in ((5, 0.4), (6, 0.0)):
    p.write(e, d, touch=True)
    st, want, _ = p.o.checkpoint_gather(flags=crum.COMPRESS)
    p.g.checkpoint_gather(zimg, flags=crum.COMPRESS)
    assert zimg.tobytes() == want.tobytes(), e
p.write(7, 0.3, touch=True)
st, want, _ = p.o.checkpoint_gather(flags=crum.COMPRESS)
p.g.checkpoint_gather_device(dimg, cap, flags=crum.COMPRESS)
assert dimg[:len(want)].cpu().numpy().tobytes() == want.tobytes()
fz = p.g.new_image()
p.g.checkpoint_gather(fz, flags=crum.FULL | crum.COMPRESS)
q.restore_scatter(fz, flags=crum.VERIFY)
torch.cuda.synchronize()
assert all(np.array_equal(z.cpu().numpy(), h) for z, h in zip(zs, p.host))
r = crum.Context(0)
zr = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for nb, _, _ in SPECS]
for z, (nb, P, m) in zip(zr, SPECS):
    r.register_region(z, nb, P, m)
sess = r.restore_begin(fz)
for rid, pg in ((1, 3), (1, 4), (2, 0), (4, 0), (6, 1)):
    sess.fetch(rid, pg)
sess.end()
torch.cuda.synchronize()
assert all(np.array_equal(z.cpu().numpy(), h) for z, h in zip(zr, p.host))
# tracked mode: marks from the host and from a writer kernel
t = crum.Context(0)
tb = torch.zeros(64 * 4096, dtype=torch.uint8, device="cuda")
tid = t.register_region(tb, tb.numel(), 4096, crum.MODE_TRACKED)
t.sync_shadow()
pg = torch.tensor([1, 5, 9], dtype=torch.int32, device="cuda")
t.mark_dirty_pages(tid, pg, 3)
crum.synth_write_pages_tracked(tb, tb.numel(), 4096, pg, 3, 7, 1, 0, t.region_tracker(tid))
assert t.sync_shadow() == 3
# persist + load
import tempfile
path = os.path.join(tempfile.mkdtemp(), "img.crum")
fz.persist(path)
fz.persist_wait()
assert r.load_image(path).tobytes() == fz.tobytes()
print("sanitize workload ok; launches", p.g.launch_count + q.launch_count + r.launch_count + t.launch_count)
