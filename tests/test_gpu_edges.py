"""GPU parity at the edges of the method: no regions, no dirty pages, one-byte
regions, the largest page size with a one-byte tail, exact-capacity images,
many tiny regions, and re-registration — libcrum.so vs the CPU oracle, bit
for bit (image bytes, reports, restored regions, snapshots)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB = 1 << 10, 1 << 20
C, H, T = 0, 1, 2


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    assert torch.cuda.is_available()
    return m


def mkpair(specs, seed_idx, **kw):
    from tests.gpu_pair import Pair
    return Pair(specs, synth.seed(seed_idx), **kw)


def gather_both(p, crum, flags=0, device=False):
    st, want, rep_o = p.o.checkpoint_gather(flags=flags)
    assert st == 0
    if device:
        cap = p.g.image_required_bytes()
        buf = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
        rep = p.g.checkpoint_gather_device(buf, cap, flags=flags)
        got = buf[:rep["image_bytes"]].cpu().numpy().tobytes()
    else:
        img = p.g.new_image()
        rep = p.g.checkpoint_gather(img, flags=flags)
        got = img.tobytes()
    assert got == want.tobytes()
    for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes", "scanned_pages", "scanned_bytes"):
        assert rep[k] == rep_o[k], k
    return want


@pytest.mark.parametrize("device", [False, True])
def test_no_regions(crum, device):
    p = mkpair([], 100)
    assert p.g.sync_shadow() == 0 == p.o.sync_shadow()
    for flags in (0, crum.FULL, crum.COMPRESS):
        want = gather_both(p, crum, flags, device)
        assert len(want) == 4096                      # header + (empty) table, padded
    q = crum.Context(0)
    assert q.restore_scatter(q.import_image(want))["dirty_pages"] == 0
    r = mkpair([(4096, 4096, C)], 101)                # a live region: the table mismatches
    st, _ = r.g.restore_scatter(r.g.import_image(want), raise_on_error=False)
    assert st == crum.E_MISMATCH


@pytest.mark.parametrize("device", [False, True])
def test_no_dirty_pages(crum, device):
    p = mkpair([(3 * 64 * KiB + 5, 64 * KiB, C), (5 * 4 * KiB, 4 * KiB, H), (2 * 4 * KiB, 4 * KiB, T)], 102)
    p.g.sync_shadow()
    p.o.sync_shadow()
    for flags in (0, crum.COMPRESS):
        want = gather_both(p, crum, flags, device)
        assert len(want) == 4096                      # K = 0: no payload, no unit-size table


@pytest.mark.parametrize("mode", [C, H, T])
def test_one_byte_regions(crum, mode):
    specs = [(1, 4096, mode), (1, 2 * MiB, mode), (2 * MiB + 1, 2 * MiB, mode), (4097, 4096, mode)]
    p = mkpair(specs, 103 + mode)
    want0 = gather_both(p, crum)                      # first gather lists everything
    p.write(1, 1.0)
    if mode == T:
        for rid_o, rid_g, (nb, P, _) in zip(p.rid_o, p.rid_g, specs):
            p.o.mark_dirty(rid_o, 0, nb)
            p.g.mark_dirty(rid_g, 0, nb)
    want1 = gather_both(p, crum, device=True)
    gather_both(p, crum, crum.FULL | crum.COMPRESS)
    # restore both images onto zeros: the regions come back byte for byte
    q = crum.Context(0)
    zs = []
    for nb, P, m in specs:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, m)
    q.restore_scatter(q.import_image(want0), flags=crum.VERIFY)
    q.restore_scatter(q.import_image(want1), flags=crum.VERIFY)
    torch.cuda.synchronize()
    for z, h in zip(zs, p.host):
        assert np.array_equal(z.cpu().numpy(), h)


def test_exact_capacity(crum):
    p = mkpair([(9 * 4 * KiB + 3, 4 * KiB, C), (2 * 64 * KiB, 64 * KiB, H)], 107)
    st, want, rep_o = p.o.checkpoint_gather()
    n = len(want)
    small = p.g.new_image(n - 1)
    st, rep = p.g.checkpoint_gather(small, raise_on_error=False)
    assert st == crum.E_CAPACITY and rep["image_bytes"] == n
    exact = p.g.new_image(n)
    p.g.checkpoint_gather(exact)
    assert exact.tobytes() == want.tobytes()
    # device form with exactly the image's size (synchronous: capacity checked on the device)
    p.write(1, 0.5)
    st, want, _ = p.o.checkpoint_gather()
    buf = torch.empty(len(want) + 256, dtype=torch.uint8, device="cuda")
    st, rep = p.g.checkpoint_gather_device(buf, len(want) - 1, raise_on_error=False)
    assert st == crum.E_CAPACITY
    rep = p.g.checkpoint_gather_device(buf, len(want))
    assert buf[:len(want)].cpu().numpy().tobytes() == want.tobytes()


def test_many_tiny_regions_mixed(crum):
    rng = np.random.default_rng(5)
    specs = []
    for i in range(300):
        P = int(rng.choice([4 * KiB, 64 * KiB]))
        nb = int(rng.integers(1, 3 * P))
        specs.append((nb, P, int(rng.integers(0, 2))))
    p = mkpair(specs, 108, chunk_bytes=64 * KiB)
    gather_both(p, crum)
    for epoch, d in ((1, 0.3), (2, 0.0), (3, 1.0)):
        p.write(epoch, d)
        gather_both(p, crum, device=epoch == 2)
        assert p.shadows_equal()


def test_reregistration(crum):
    p = mkpair([(4 * 64 * KiB, 64 * KiB, C), (3 * 4 * KiB, 4 * KiB, H)], 109)
    gather_both(p, crum)
    for rid_o, rid_g in zip(p.rid_o, p.rid_g):
        p.o.unregister(rid_o)
        p.g.unregister_region(rid_g)
    assert p.g.sync_shadow() == 0 == p.o.sync_shadow()
    from oracle import oracle
    h = oracle.aligned_empty(5 * 4 * KiB + 7)
    synth.fill_region(h, synth.seed(110), 0)
    d = torch.from_numpy(h.copy()).cuda()
    ro = p.o.register(h, 4 * KiB, H)
    rg = p.g.register_region(d, h.nbytes, 4 * KiB, H)
    assert ro == rg                                   # ids keep counting in both
    st, want, rep_o = p.o.checkpoint_gather()
    img = p.g.new_image()
    rep = p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes() and rep["dirty_pages"] == 6


def test_batch_registration(crum):
    """crum_register_regions: consecutive ids in descriptor order, the same
    images as one-by-one registration (so the same as the oracle's), and a
    transactional failure (an overlap between two descriptors, a bad page
    size, an overlap with a live region) registers nothing and names the
    offending descriptor."""
    from oracle import oracle
    specs = [(3 * 64 * KiB + 77, 64 * KiB, C), (40 * KiB + 8, 4 * KiB, H), (2 * MiB + 16, 2 * MiB, C),
             (12 * KiB, 4 * KiB, 2)]
    S = synth.seed(131)
    ctx = crum.Context(0)
    o = oracle.Oracle()
    ts, hs = [], []
    for r, (nb, P, mode) in enumerate(specs):
        h = oracle.aligned_empty(nb)
        synth.fill_region(h, S, r)
        hs.append(h)
        ts.append(torch.from_numpy(h.copy()).cuda())
        o.register(h, P, mode)
    ids = ctx.register_regions([(t, nb, P, m) for t, (nb, P, m) in zip(ts, specs)])
    assert ids == [1, 2, 3, 4]
    st, want, _ = o.checkpoint_gather()
    img = ctx.new_image()
    ctx.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()
    # failures register nothing
    extra = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    a = extra.data_ptr()
    st, fail = ctx.try_register_regions([(a, 65536, 4096, C), (a + 32768, 65536, 4096, C)])
    assert st == crum.E_OVERLAP and fail == 1
    st, fail = ctx.try_register_regions([(a, 65536, 4096, C), (a + 131072, 65536, 3000, C)])
    assert st == crum.E_INVAL and fail == 1
    st, fail = ctx.try_register_regions([(a, 65536, 4096, C), (ts[0].data_ptr() + 4096, 8192, 4096, C)])
    assert st == crum.E_OVERLAP and fail == 1
    assert ctx.try_register_regions([]) == ([], None)
    # the registry is unchanged: the next ids continue, the next image lists the same regions
    ids2 = ctx.register_regions([(extra, 65536, 4096, C)])
    assert ids2 == [5]
    ctx.unregister_region(5)
    for r, (nb, P, mode) in enumerate(specs):
        pg = synth.choose_dirty(S, 1, r, synth.n_pages(nb, P), 0.5)
        synth.apply_writer(hs[r], P, pg, S, 1, r)
        ts[r].copy_(torch.from_numpy(hs[r]))
        if mode == 2:
            o.mark_pages(r + 1, pg)
            ctx.mark_dirty_pages(ids[r], torch.from_numpy(pg.astype(np.uint32)).cuda(), len(pg))
    st, want, _ = o.checkpoint_gather()
    ctx.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()
