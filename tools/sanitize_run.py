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
# round 2 kernels: the one-launch small path (one page size), the single-pass
# kernel (compare-only, two page sizes, small footprint), batch registration,
# and the LZ77 + DEFLATE codec on structured data across two encode chunks
from oracle import oracle
def fresh(specs, seed, structured=False, **kw):
    q2 = Pair(specs, synth.seed(seed), **kw)
    if structured:
        rng = np.random.default_rng(seed)
        for h, d in zip(q2.host, q2.dev):
            f = h[:h.nbytes // 8 * 8].view("<f8")
            for b0 in range(0, f.size, 4096):
                k = int(rng.integers(0, 4))
                f[b0:b0 + 4096] = (np.sin(np.arange(min(4096, f.size - b0)) * 0.01) if k == 0 else
                                   [0.0, 1.0, 1.0 / 6.0][k - 1])
            d.copy_(torch.from_numpy(h))
        torch.cuda.synchronize()
    return q2
for specs, seed in (([(1 * MiB, 4 * KiB, 0), (64 * KiB + 5, 4 * KiB, 2)], 50),
                    ([(1 * MiB, 4 * KiB, 0), (3 * 64 * KiB + 9, 64 * KiB, 0)], 51)):
    q2 = fresh(specs, seed)
    im2 = q2.g.new_image()
    c2 = q2.g.image_required_bytes()
    b2 = torch.zeros(c2 + 256, dtype=torch.uint8, device="cuda")
    for e, d in ((1, 0.2), (2, 0.0), (3, 1.0)):
        q2.write(e, d)
        for r_, (nb, P, m) in enumerate(specs):
            if m == 2:
                pgs = synth.choose_dirty(q2.S, e, r_, synth.n_pages(nb, P), d)
                q2.o.mark_pages(r_ + 1, pgs)
                q2.g.mark_dirty_pages(r_ + 1, torch.from_numpy(pgs.astype(np.uint32)).cuda(), len(pgs))
        st, want, _ = q2.o.checkpoint_gather()
        if e == 2:
            q2.g.checkpoint_gather_device(b2, c2, report=False)
            torch.cuda.synchronize()
            got = b2[:len(want)].cpu().numpy().tobytes()
        else:
            q2.g.checkpoint_gather(im2)
            got = im2.tobytes()
        assert got == want.tobytes(), (seed, e)
bq = crum.Context(0)
bt = [torch.zeros(n, dtype=torch.uint8, device="cuda") for n in (65536, 8192 + 5, 4096 * 3)]
assert bq.register_regions([(x, x.numel(), 4096, 0) for x in bt]) == [1, 2, 3]
zq = fresh([(20 * MiB + 4096 * 3 + 7, 64 * KiB, 0), (2 * MiB, 4 * KiB, 1)], 52, structured=True)
zi = zq.g.new_image()
st, want, _ = zq.o.checkpoint_gather(flags=crum.COMPRESS)
zq.g.checkpoint_gather(zi, flags=crum.COMPRESS)
assert zi.tobytes() == want.tobytes()
zr2 = crum.Context(0)
zz = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for nb, _, _ in zq.specs]
for z, (nb, P, m) in zip(zz, zq.specs):
    zr2.register_region(z, nb, P, m)
zr2.restore_scatter(zi, flags=crum.VERIFY)
torch.cuda.synchronize()
assert all(np.array_equal(z.cpu().numpy(), h) for z, h in zip(zz, zq.host))
# mapped-store pinned gathers (footprints above the small-footprint size): one
# range, halving ranges (mixed modes) and the single pass (compare only), each
# after a gather whose payload selects it
for specs, seed in (([(20 * MiB + 4096 * 3 + 7, 4 * KiB, 0), (8 * MiB, 64 * KiB, 1)], 53),
                    ([(20 * MiB + 4096 * 3 + 7, 4 * KiB, 0), (8 * MiB + 100, 64 * KiB, 0)], 54)):
    mq = fresh(specs, seed)
    mi = mq.g.new_image()
    paths = []
    for e, d in ((1, 0.002), (2, 0.002), (3, 0.15), (4, 0.05), (5, 0.0)):
        mq.write(e, d)
        st, want, _ = mq.o.checkpoint_gather()
        rep = mq.g.checkpoint_gather(mi)
        paths.append(rep["path"])
        assert mi.tobytes() == want.tobytes(), (seed, e)
    assert any(x & crum.PATH_MAPPED for x in paths), paths
print("sanitize workload ok; launches", p.g.launch_count + q.launch_count + r.launch_count + t.launch_count)
