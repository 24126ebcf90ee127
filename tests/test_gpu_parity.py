"""GPU parity: libcrum.so (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs (bit-exact: flags, ids, hashes, image
bytes, restored regions, snapshots).  Sizes span several tiles and ragged
tails; the C2 (1 GiB) case runs in the launch configuration bench.py times."""
import numpy as np
import pytest
import xxhash

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30
C, H = 0, 1

MIXED = [
    (4 * MiB, 4 * KiB, C),                 # C1 shape
    (3 * 64 * KiB + 1234, 64 * KiB, H),    # ragged tail, hash
    (5 * 4 * KiB + 17, 4 * KiB, H),        # odd page count at 4 KiB (two pages per warp)
    (2 * MiB + 4 * KiB + 100, 2 * MiB, C),  # 2 MiB pages, tiny tail page
    (2 * MiB * 2 + 300, 2 * MiB, H),
    (12 * KiB + 256, 4 * KiB, C),          # HPGMG-like small box region
    (64 * KiB * 7, 64 * KiB, C),
]


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


def test_synth_device_matches_numpy(crum):
    for nb in (8, 13, 4096, 65536 + 5):
        d = torch.empty(nb, dtype=torch.uint8, device="cuda")
        crum.synth_fill(d, nb, synth.seed(1), 3)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), synth.region_content(synth.seed(1), 3, nb))


@pytest.mark.parametrize("misalign", [0, 16])
def test_detect_parity_mixed(crum, misalign):
    p = mkpair(MIXED, 10, misalign=misalign)
    assert p.g.debug_detect(p.N).tolist() == [1] * p.N       # all force-dirty at register
    assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags())
    assert p.g.sync_shadow() == p.o.sync_shadow() == p.N
    assert p.shadows_equal()
    assert p.g.sync_shadow() == 0 and p.o.sync_shadow() == 0
    for epoch, d in ((1, 0.1), (2, 0.5), (3, 1.0), (4, 0.0)):
        p.write(epoch, d)
        assert p.regions_equal()
        want = p.oracle_flags()
        assert np.array_equal(p.g.debug_detect(p.N), want), epoch
        assert p.g.sync_shadow() == p.o.sync_shadow() == int(want.sum())
        assert p.shadows_equal()
    p.write(5, 0.3, touch=True)                               # one word per page
    assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags())


def test_synth_batched_matches_single(crum):
    """crum_synth_fill_regions / crum_synth_write_regions (one launch for many
    regions, bench.py's C4 setup and writer) give every region exactly what
    the per-region calls give it: ragged sizes (one below a word), empty
    page lists, both writer forms."""
    sizes = [4 * 4096 + 13, 5, 64 * KiB, 3 * 4096, 9 * 4096 + 8]
    P = 4096
    S = synth.seed(9)
    a = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for nb in sizes]
    b = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for nb in sizes]
    crum.synth_fill_regions([(t, nb, r + 3) for r, (t, nb) in enumerate(zip(a, sizes))], S)
    for r, (t, nb) in enumerate(zip(b, sizes)):
        crum.synth_fill(t, nb, S, r + 3)
    torch.cuda.synchronize()
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    for touch in (False, True):
        pages = [torch.tensor(sorted({0, synth.n_pages(nb, P) - 1}) if r != 1 else [], dtype=torch.int32,
                              device="cuda") for r, nb in enumerate(sizes)]
        crum.synth_write_regions([(t, nb, P, r + 3, pg, pg.numel()) for r, (t, nb, pg) in enumerate(zip(a, sizes, pages))],
                                 S, 7, touch)
        for r, (t, nb, pg) in enumerate(zip(b, sizes, pages)):
            crum.synth_write_pages(t, nb, P, pg, pg.numel(), S, 7, r + 3, touch)
        torch.cuda.synchronize()
        assert all(torch.equal(x, y) for x, y in zip(a, b)), touch


def test_exhaustive_single_byte_flips(crum):
    for mode in (C, H):
        p = mkpair([(2 * 4096, 4096, mode)], 11)
        p.g.sync_shadow()
        d = p.dev[0]
        step = 1 if mode == C else 5
        for pos in range(0, 8192, step):
            d[pos] ^= 1
            f = p.g.debug_detect(2)
            assert f.tolist() == [int(pos < 4096), int(pos >= 4096)], (mode, pos)
            d[pos] ^= 1


def test_hash_table_matches_library(crum):
    specs = [(3 * 64 * KiB + 999, 64 * KiB, H), (2 * MiB + 5, 2 * MiB, H), (9 * 4096 + 1, 4096, H)]
    p = mkpair(specs, 12)
    p.g.sync_shadow()
    for (nb, P, _), rg, h in zip(specs, p.rid_g, p.host):
        got = p.g.debug_export(rg, crum.EXPORT_HASHES, synth.n_pages(nb, P))
        for i in range(len(got)):
            seg = h[i * P:(i + 1) * P].tobytes()
            assert int(got[i]) == xxhash.xxh3_64_intdigest(seg + b"\0" * (P - len(seg))), (P, i)


@pytest.mark.parametrize("chunk", [0, 64 * KiB])
def test_gather_image_bit_exact(crum, chunk):
    p = mkpair(MIXED, 13, chunk_bytes=chunk)
    img = p.g.new_image()
    for epoch, d, flags in ((0, 0, 0), (1, 0.1, 0), (2, 0.5, 0), (3, 0.0, 0), (4, 0.2, 1), (5, 1.0, 0)):
        if epoch:
            p.write(epoch, d)
        st, want, rep_o = p.o.checkpoint_gather(flags=flags)
        assert st == 0
        rep = p.g.checkpoint_gather(img, flags=flags)
        assert img.length == len(want)
        assert img.tobytes() == want.tobytes(), epoch
        for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes", "scanned_pages", "scanned_bytes"):
            assert rep[k] == rep_o[k], (epoch, k)
        assert p.shadows_equal()


def test_gather_device_image_bit_exact(crum):
    p = mkpair(MIXED, 14)
    cap = p.g.image_required_bytes()
    buf = torch.empty(cap + 4096, dtype=torch.uint8, device="cuda")
    for epoch, d in ((0, 0), (1, 0.25), (2, 0.0)):
        if epoch:
            p.write(epoch, d)
        st, want, _ = p.o.checkpoint_gather()
        rep = p.g.checkpoint_gather_device(buf, cap)
        assert rep["image_bytes"] == len(want)
        assert buf[:len(want)].cpu().numpy().tobytes() == want.tobytes()
    # asynchronous form (no report) then a synchronous read of the header
    p.write(3, 0.4)
    st, want, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather_device(buf, cap, report=False)
    torch.cuda.synchronize()
    assert buf[:len(want)].cpu().numpy().tobytes() == want.tobytes()


def test_capacity_error_commits_nothing(crum):
    p = mkpair(MIXED[:3], 15)
    small = p.g.new_image(4096)
    st, rep = p.g.checkpoint_gather(small, raise_on_error=False)
    assert st == crum.E_CAPACITY and rep["image_bytes"] > 4096
    assert p.g.debug_detect(p.N).tolist() == [1] * p.N       # force bits untouched
    buf = torch.empty(8192, dtype=torch.uint8, device="cuda")
    st, rep = p.g.checkpoint_gather_device(buf, 8192, raise_on_error=False)
    assert st == crum.E_CAPACITY
    assert p.g.debug_detect(p.N).tolist() == [1] * p.N
    st, _ = p.g.checkpoint_gather_device(buf, 8192, report=False, raise_on_error=False)
    assert st == crum.E_CAPACITY                               # async form: checked on the host


def test_restore_chain_parity(crum):
    p = mkpair(MIXED, 16)
    imgs, states = [], []
    for epoch in range(4):
        if epoch:
            p.write(epoch, 0.3)
        img = p.g.new_image()
        p.g.checkpoint_gather(img)
        imgs.append(img)
        states.append([h.copy() for h in p.host])
    # restart: fresh context, zeroed regions; replay the chain (VERIFY on odd steps)
    q = crum.Context(0, chunk_bytes=128 * KiB)
    zs = []
    for nb, P, mode in MIXED:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, mode)
    for k, img in enumerate(imgs):
        rep = q.restore_scatter(img, flags=crum.VERIFY if k % 2 else 0)
        assert rep["dirty_pages"] == (sum(synth.n_pages(nb, P) for nb, P, _ in MIXED) if k == 0 else rep["dirty_pages"])
        torch.cuda.synchronize()
        for z, want in zip(zs, states[k]):
            assert np.array_equal(z.cpu().numpy(), want), k
    assert q.sync_shadow() == 0


def test_restore_device_and_errors(crum):
    specs = [(3 * 4096, 4096, C), (2 * 4096 + 7, 4096, H)]
    p = mkpair(specs, 17)
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    raw = img.view().copy()
    from tests import imgfmt
    q = crum.Context(0)
    zs = []
    for nb, P, mode in specs:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, mode)
    # every single-byte corruption of the header + metadata is rejected, nothing written
    for pos in imgfmt.meta_positions(raw):
        bad = raw.copy()
        bad[pos] ^= 0x10
        st, _ = q.restore_scatter(q.import_image(bad), raise_on_error=False)
        assert st == crum.E_CORRUPT, pos
    st, _ = q.restore_scatter(q.import_image(raw[:-1]), raise_on_error=False)
    assert st == crum.E_CORRUPT
    assert all(int(z.sum()) == 0 for z in zs)
    # VERIFY catches a tampered hash-mode slot
    bad = raw.copy()
    bad[imgfmt.parse_image(raw)["ids_off"] - 1] ^= 0xFF   # last byte of the last (hash-mode) slot
    st, _ = q.restore_scatter(q.import_image(bad), flags=crum.VERIFY, raise_on_error=False)
    assert st == crum.E_CORRUPT
    st, _ = q.restore_scatter(q.import_image(bad), raise_on_error=False)
    assert st == crum.OK                      # only VERIFY looks at payload bytes
    q.restore_scatter(q.import_image(raw))
    # table != live set
    r = crum.Context(0)
    z = torch.zeros(4 * 4096, dtype=torch.uint8, device="cuda")
    r.register_region(z, 4 * 4096, 4096, C)
    st, _ = r.restore_scatter(r.import_image(raw), raise_on_error=False)
    assert st == crum.E_MISMATCH
    # device-resident image restore
    dimg = torch.from_numpy(raw).cuda()
    dbuf = torch.empty(len(raw) + 256, dtype=torch.uint8, device="cuda")
    dbuf[:len(raw)].copy_(dimg)
    q.restore_scatter_device(dbuf, len(raw), flags=crum.VERIFY)
    torch.cuda.synchronize()
    for z, h in zip(zs, p.host):
        assert np.array_equal(z.cpu().numpy(), h)
    # oracle agrees on the same images
    o2 = p.o  # regions match the image's table
    assert o2.restore_scatter(raw)[0] == 0


def test_mark_dirty_parity(crum):
    p = mkpair([(8 * 4096, 4096, C), (4 * 64 * KiB, 64 * KiB, H)], 18)
    p.g.sync_shadow()
    p.o.sync_shadow()
    for (rid_o, rid_g), (off, ln) in zip([(p.rid_o[0], p.rid_g[0])] * 3 + [(p.rid_o[1], p.rid_g[1])],
                                         [(4095, 2), (5 * 4096, 0), (7 * 4096, 4096), (65536 * 2 + 1, 1)]):
        assert p.g.mark_dirty(rid_g, off, ln) == p.o.mark_dirty(rid_o, off, ln) == 0
    assert p.g.mark_dirty(p.rid_g[0], 8 * 4096, 1) == crum.E_RANGE
    assert p.g.mark_dirty(999, 0, 1) == crum.E_NOREGION
    assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags())
    st, want, _ = p.o.checkpoint_gather()
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()


def test_register_errors(crum):
    g = crum.Context(0)
    t = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    a = t.data_ptr()
    assert g.try_register(0, 4096, 4096) == crum.E_INVAL
    assert g.try_register(a, 0, 4096) == crum.E_INVAL
    assert g.try_register(a, 4096, 2048) == crum.E_INVAL
    assert g.try_register(a, 4096, 12288) == crum.E_INVAL
    assert g.try_register(a + 8, 4096, 4096) == crum.E_INVAL
    assert g.try_register(a, 4096, 4096, 5) == crum.E_INVAL
    h = np.zeros(8192, dtype=np.uint8)
    assert g.try_register(h.ctypes.data // 16 * 16 + 16, 4096, 4096) == crum.E_DEVICE
    assert g.try_register(a, 65536, 4096) == 0
    assert g.try_register(a + 4096, 4096, 4096) == crum.E_OVERLAP
    assert g.try_register(a + 65536, 4096, 4096) == 0
    g.unregister_region(1)
    with pytest.raises(crum.CrumError):
        g.unregister_region(1)


def test_unregister_keeps_other_state(crum):
    specs = [(4 * 4096, 4096, C), (4 * 4096, 4096, H), (4 * 4096, 4096, C)]
    p = mkpair(specs, 19)
    p.g.sync_shadow()
    p.o.sync_shadow()
    p.write(1, 0.5)
    p.g.unregister_region(p.rid_g[1])
    p.o.unregister(p.rid_o[1])
    del p.specs[1], p.host[1], p.dev[1], p.rid_o[1], p.rid_g[1]
    assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags())
    st, want, _ = p.o.checkpoint_gather()
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()


@pytest.mark.parametrize("mode", [C, H])
@pytest.mark.parametrize("P", [64 * KiB, 2 * MiB])
def test_c2_full_size_parity(crum, mode, P):
    """Config 2 (1 GiB region) in the bench launch configuration, d = 10%:
    the whole image (ids, hashes, payload) compared with the oracle."""
    p = mkpair([(GiB, P, mode)], 2)
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    p.o.checkpoint_gather()
    p.write(1, 0.1)
    st, want, rep_o = p.o.checkpoint_gather()
    rep = p.g.checkpoint_gather(img)
    assert rep["dirty_pages"] == rep_o["dirty_pages"] == synth.dirty_count(0.1, GiB // P)
    assert img.length == len(want)
    assert np.array_equal(img.view(), want)


def test_c3_multi_region_sampled(crum):
    """Config 3 shape (Rodinia-style region mix), 2 replicas, 64 KiB pages:
    full checkpoint, 10% incremental, restore onto zeros, compared exactly."""
    sizes = synth.c3_region_sizes(replicas=2)
    specs = [(s, 64 * KiB, C if i % 3 else H) for i, s in enumerate(sizes)]
    p = mkpair(specs, 3)
    img0 = p.g.new_image()
    p.g.checkpoint_gather(img0)
    st, want0, _ = p.o.checkpoint_gather()
    assert np.array_equal(img0.view(), want0)
    p.write(1, 0.1)
    img1 = p.g.new_image()
    p.g.checkpoint_gather(img1)
    st, want1, _ = p.o.checkpoint_gather()
    assert np.array_equal(img1.view(), want1)
    q = crum.Context(0)
    zs = []
    for nb, P, mode in specs:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, mode)
    q.restore_scatter(img0)
    q.restore_scatter(img1, flags=crum.VERIFY)
    torch.cuda.synchronize()
    for z, h in zip(zs, p.host):
        assert np.array_equal(z.cpu().numpy(), h)


def test_tracked_mode_parity(crum):
    """CRUM_MODE_TRACKED (Alg. 1 write rule): pages marked in-kernel by the
    writer (crum_mark_write of include/crum_device.h), marked by the
    stream-ordered batch call, and an unmarked change -- images bit-exact with
    the oracle given the same marks."""
    T = 2
    specs = [(6 * 4096 + 10, 4096, T), (5 * 65536, 65536, T), (3 * 4096, 4096, C), (2 * 65536, 65536, H)]
    p = mkpair(specs, 21)
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    st, want, _ = p.o.checkpoint_gather()
    assert img.tobytes() == want.tobytes()
    # epoch 1: the writer marks what it writes in regions 0 and 1
    for r in (0, 1):
        nb, P, _ = specs[r]
        pages = synth.choose_dirty(p.S, 1, r, synth.n_pages(nb, P), 0.4)
        synth.apply_writer(p.host[r], P, pages, p.S, 1, r)
        p.o.mark_pages(p.rid_o[r], pages)
        dp = torch.from_numpy(pages.astype(np.uint32)).cuda()
        crum.synth_write_pages_tracked(p.dev[r], nb, P, dp, len(pages), p.S, 1, r, p.g.region_tracker(p.rid_g[r]))
    # an unmarked change (not captured by definition) and a batch mark of an unchanged page
    p.host[0][4096 * 5 + 7] ^= 1
    p.dev[0][4096 * 5 + 7] ^= 1
    marks = np.array([3], dtype=np.uint32)
    p.o.mark_pages(p.rid_o[1], marks)
    assert p.g.mark_dirty_pages(p.rid_g[1], torch.from_numpy(marks).cuda(), 1) == 0
    torch.cuda.synchronize()
    assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags())
    st, want, _ = p.o.checkpoint_gather()
    rep = p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()
    assert p.g.sync_shadow() == p.o.sync_shadow() == 0
    # restore of both images onto zeroed tracked regions reproduces the marked state
    q = crum.Context(0)
    zs = []
    for nb, P, mode in specs:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, mode)
    st, full_want, _ = p.o.checkpoint_gather(flags=crum.FULL)
    full = p.g.new_image()
    p.g.checkpoint_gather(full, flags=crum.FULL)
    assert full.tobytes() == full_want.tobytes()
    q.restore_scatter(full)
    torch.cuda.synchronize()
    for z, h in zip(zs, p.host):
        assert np.array_equal(z.cpu().numpy(), h)


def test_async_device_gather_graph_replays(crum):
    """The asynchronous device gather is captured once as a CUDA graph and
    replayed: replays, a second image buffer (recapture) and a registration
    in between (invalidation) all stay bit-exact with the oracle."""
    p = mkpair(MIXED[:5], 18)
    cap = p.g.image_required_bytes()
    bufs = [torch.empty(cap + 256, dtype=torch.uint8, device="cuda") for _ in range(2)]
    st, want, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather_device(bufs[0], cap)                 # epoch 0 (with report)
    for epoch in range(1, 9):
        p.write(epoch, 0.2 if epoch % 3 else 0.0)
        st, want, _ = p.o.checkpoint_gather()
        b = bufs[(epoch // 3) % 2]
        n0 = p.g.launch_count
        p.g.checkpoint_gather_device(b, cap, report=False)     # graph replay (or capture)
        torch.cuda.synchronize()
        assert p.g.launch_count > n0                           # replays count their kernels
        assert b[:len(want)].cpu().numpy().tobytes() == want.tobytes(), epoch
        assert p.shadows_equal(), epoch
    # a new region invalidates the captured graph
    from oracle import oracle
    nb, P = 3 * 4096 + 5, 4096
    h = oracle.aligned_empty(nb)
    synth.fill_region(h, synth.seed(19), 9)
    d = torch.from_numpy(h.copy()).cuda()
    p.o.register(h, P, C)
    p.g.register_region(d, nb, P, C)
    cap = p.g.image_required_bytes()
    big = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
    for epoch in (20, 21):
        p.write(epoch, 0.3)
        st, want, _ = p.o.checkpoint_gather()
        p.g.checkpoint_gather_device(big, cap, report=False)
        torch.cuda.synchronize()
        assert big[:len(want)].cpu().numpy().tobytes() == want.tobytes(), epoch


def test_numa_bound_image_bit_exact(crum):
    """A pinned image placed by mmap + mbind + cudaHostRegister (forced with
    crum_config.numa_node = 0, since a single-node box would otherwise take
    cudaHostAlloc) holds the same bytes as the oracle's image and restores as
    one."""
    p = mkpair(MIXED[:4], 27, numa_node=0)
    img = p.g.new_image()
    assert img.numa_node in (0, -1)          # -1: the sandbox refused mbind (memory still mmap'ed + registered)
    assert crum.device_numa_node(0) >= -1
    for epoch, d in ((0, 0), (1, 0.3)):
        if epoch:
            p.write(epoch, d)
        st, want, _ = p.o.checkpoint_gather()
        p.g.checkpoint_gather(img)
        assert img.tobytes() == want.tobytes(), epoch
    # restore the delta onto the previous state of a fresh pair
    q = mkpair(MIXED[:4], 27)
    q.g.sync_shadow()
    q.o.sync_shadow()
    q.g.restore_scatter(img)
    torch.cuda.synchronize()
    assert all(np.array_equal(d.cpu().numpy(), h) for d, h in zip(q.dev, p.host))
    img.destroy()
    ctx = crum.Context(0, numa_node=crum.NUMA_DEFAULT)
    assert ctx.new_image(4096).numa_node == -1


@pytest.mark.parametrize("P", [64 * KiB, 2 * MiB])
def test_hash_detect_repeatable_under_load(crum, P):
    """Stress of the TMA-fed hash kernel's shared-memory ring (DESIGN.md,
    "TMA ring rule"): after a sync, every re-detect of an unchanged 1 GiB
    region must flag nothing -- a stage overwritten while its reads were in
    flight shows up as a spurious dirty page -- and the committed hashes must
    equal the library's XXH3 on sampled pages."""
    nb = GiB
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    crum.synth_fill(d, nb, synth.seed(31), 0)
    ctx = crum.Context(0)
    rid = ctx.register_region(d, nb, P, H)
    n = nb // P
    assert ctx.sync_shadow() == n
    for _ in range(24):
        assert int(ctx.debug_detect(n).sum()) == 0
    table = ctx.debug_export(rid, crum.EXPORT_HASHES, n)
    rng = np.random.default_rng(5)
    for i in sorted(rng.choice(n, 8, replace=False)):
        page = d[i * P:(i + 1) * P].cpu().numpy().tobytes()
        assert int(table[i]) == xxhash.xxh3_64_intdigest(page), i


def test_hash_page_groups_straddle_regions(crum):
    """The page-group hash kernel hashes big-page indices 2t, 2t+1 together:
    with 5 pages of 64 KiB (ragged tail) before 2 pages of 2 MiB (ragged) and
    3 pages of 64 KiB, the groups (4, 5) and (6, 7) pair pages of different
    sizes from different regions.  Flags, hashes and images stay bit-exact."""
    specs = [(4 * 64 * KiB + 100, 64 * KiB, H), (2 * MiB + 5000, 2 * MiB, H), (3 * 64 * KiB, 64 * KiB, H),
             (7 * 4 * KiB + 9, 4 * KiB, H)]
    p = mkpair(specs, 41)
    img = p.g.new_image()
    for epoch, d in ((0, 0), (1, 0.5), (2, 1.0), (3, 0.3)):
        if epoch:
            p.write(epoch, d)
            assert np.array_equal(p.g.debug_detect(p.N), p.oracle_flags()), epoch
        st, want, _ = p.o.checkpoint_gather()
        p.g.checkpoint_gather(img)
        assert img.tobytes() == want.tobytes(), epoch
        assert p.shadows_equal()


def test_deferred_commit_streaming_gather(crum):
    """A pinned image smaller than the worst case (the bench's C4 setting): the
    gather still streams range by range, copying without committing, and
    commits after the final range shows the image fits.  Image bytes and
    shadows equal the oracle's every epoch; an image that overflows part-way
    through the ranges returns CAPACITY with the exact required size and
    commits nothing (crum.h error convention)."""
    specs = [(40 * MiB + 4096 * 3 + 5, 4 * KiB, C), (72 * MiB, 64 * KiB, H), (24 * MiB, 64 * KiB, C),
             (8 * MiB + 300, 2 * MiB, H)]
    p = mkpair(specs, 19, chunk_bytes=1 * MiB)
    p.g.sync_shadow()
    p.o.sync_shadow()
    worst = p.g.image_required_bytes()
    for epoch, d in [(1, 0.1), (2, 0.02), (3, 0.3), (4, 0.0)]:
        p.write(epoch, d)
        flags_before = p.oracle_flags().tolist()     # the dirty set before either side commits
        st, want, rep_o = p.o.checkpoint_gather()
        assert st == 0
        assert len(want) < worst
        # overflow: the first ranges fit, a later one does not
        short = p.g.new_image(len(want) * 2 // 3 if len(want) > 3 * 65536 else 4096)
        st, rep = p.g.checkpoint_gather(short, raise_on_error=False)
        if len(want) > short.capacity:
            assert st == crum.E_CAPACITY and rep["image_bytes"] == len(want)
            assert p.g.debug_detect(p.N).tolist() == flags_before   # nothing committed
        short.destroy()
        img = p.g.new_image(len(want))     # exactly the image: deferred commit path
        rep = p.g.checkpoint_gather(img)
        assert img.tobytes() == want.tobytes(), epoch
        assert rep["dirty_pages"] == rep_o["dirty_pages"] and rep["image_bytes"] == len(want)
        assert p.shadows_equal(), epoch
        img.destroy()


def test_small_path_tracked_and_compare(crum):
    """The one-launch small path (k_small_ckpt, C1-sized footprints with one
    page size): tracked and compare regions together, device (async graph
    replay and synchronous) and pinned images, byte for byte with the oracle
    every epoch, shadows equal."""
    from oracle import oracle
    specs = [(4 * MiB, 4 * KiB, C), (256 * KiB + 100, 4 * KiB, 2), (64 * KiB, 4 * KiB, C)]
    S = synth.seed(77)
    o = oracle.Oracle()
    ctx = crum.Context(0)
    hs, ds = [], []
    for r, (nb, P, mode) in enumerate(specs):
        h = oracle.aligned_empty(nb)
        synth.fill_region(h, S, r)
        hs.append(h)
        ds.append(torch.from_numpy(h.copy()).cuda())
        o.register(h, P, mode)
        ctx.register_region(ds[-1], nb, P, mode)
    cap = ctx.image_required_bytes()
    buf = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
    img = ctx.new_image()
    for epoch in range(8):
        if epoch:
            for r, (nb, P, mode) in enumerate(specs):
                pg = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), [0.01, 0.3, 0.0, 1.0][epoch % 4])
                synth.apply_writer(hs[r], P, pg, S, epoch, r)
                ds[r].copy_(torch.from_numpy(hs[r]))
                if mode == 2:
                    o.mark_pages(r + 1, pg)
                    ctx.mark_dirty_pages(r + 1, torch.from_numpy(pg.astype(np.uint32)).cuda(), len(pg))
        st, want, rep_o = o.checkpoint_gather()
        assert st == 0
        how = epoch % 3
        if how == 0:
            rep = ctx.checkpoint_gather(img)
            got = img.tobytes()
        else:
            rep = ctx.checkpoint_gather_device(buf, cap, report=(how == 2))
            rep = rep or ctx.last_report()
            torch.cuda.synchronize()
            got = buf[:len(want)].cpu().numpy().tobytes()
        assert got == want.tobytes(), epoch
        assert rep["path"] & crum.PATH_FUSED, epoch
        for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes"):
            assert rep[k] == rep_o[k], (epoch, k)
    for r, (nb, P, mode) in enumerate(specs):
        if mode == C:
            assert np.array_equal(ctx.debug_export(r + 1, crum.EXPORT_MIRROR, nb), o.mirror(r + 1))
        assert np.array_equal(ctx.debug_export(r + 1, crum.EXPORT_FORCE, synth.n_pages(nb, P)), o.force_bits(r + 1))


@pytest.mark.parametrize("kind", ["mixed", "compare", "tracked"])
@pytest.mark.parametrize("no_mapped", [False, True])
def test_mapped_store_gather(crum, kind, no_mapped):
    """Pinned gathers above the small-footprint size whose previous payload
    was small store straight into the pinned image through its mapped address
    (CRUM_PATH_MAPPED, previous payload <= 16 MiB -- 32 MiB in compare-only
    contexts: the single-pass kernel above 2 MiB when every region is COMPARE
    with pages <= 64 KiB, else the
    detect -> compact -> gather sequence in halving ranges above 1 MiB, in
    one range below); a larger
    previous payload, the first gather after registration, or
    CRUM_CFG_NO_MAPPED take the ring + D2H pipeline.  Image bytes, reports
    and shadows equal the oracle's every epoch, on every path, with ragged
    tails (and hash regions in the mixed set)."""
    T = 2
    if kind == "mixed":
        specs = [(40 * MiB + 4096 * 3 + 5, 4 * KiB, C), (72 * MiB, 64 * KiB, H), (24 * MiB, 64 * KiB, C),
                 (8 * MiB + 300, 2 * MiB, H)]
        limit = 16 * MiB
    elif kind == "tracked":  # TRACKED regions: the writer marks what it writes
        specs = [(24 * MiB + 4096 + 9, 4 * KiB, T), (16 * MiB, 64 * KiB, C), (8 * MiB, 64 * KiB, T)]
        limit = 16 * MiB
    else:  # compare-only: the single pass takes payloads up to 32 MiB
        specs = [(40 * MiB + 4096 * 3 + 5, 4 * KiB, C), (72 * MiB, 64 * KiB, C), (8 * MiB + 300, 64 * KiB, C)]
        limit = 32 * MiB
    p = mkpair(specs, 23, flags=crum.CFG_NO_MAPPED if no_mapped else 0)
    img = p.g.new_image()
    assert img.capacity == p.g.image_required_bytes()
    prev_payload = None
    for epoch, d in [(0, 0.0), (1, 0.01), (2, 0.0), (3, 0.3), (4, 0.02), (5, 0.005), (6, 0.1), (7, 0.0)]:
        if epoch:
            p.write(epoch, d)
            for r, (nb, P, mode) in enumerate(specs):
                if mode == T:
                    pages = synth.choose_dirty(p.S, epoch, r, synth.n_pages(nb, P), d)
                    p.o.mark_pages(p.rid_o[r], pages)
                    p.g.mark_dirty_pages(p.rid_g[r], torch.from_numpy(pages.astype(np.uint32)).cuda(), len(pages))
            torch.cuda.synchronize()
        st, want, rep_o = p.o.checkpoint_gather()
        assert st == 0
        rep = p.g.checkpoint_gather(img)
        assert img.length == len(want)
        assert img.tobytes() == want.tobytes(), epoch
        for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes"):
            assert rep[k] == rep_o[k], (epoch, k)
        assert p.shadows_equal(), epoch
        mapped = bool(rep["path"] & crum.PATH_MAPPED)
        # epoch 0: the first gather after registration (every page force-dirty)
        expect = not no_mapped and prev_payload is not None and prev_payload <= limit
        assert mapped == expect, (epoch, prev_payload)
        if mapped:  # the single pass above 2 MiB; below it, halving ranges above 1 MiB, else one range
            assert bool(rep["path"] & crum.PATH_FUSED) == (kind == "compare" and prev_payload > 2 * MiB)
        prev_payload = int.from_bytes(want.tobytes()[32:40], "little")


@pytest.mark.parametrize("where", ["pool", "numa"])
def test_mapped_store_pool_and_numa_images(crum, where):
    """The mapped-store paths write through the image's device-mapped
    address: images carved from the context's pinned pool
    (crum_config.pinned_pool_bytes) and NUMA-bound images (mmap + mbind +
    registration) take them too, bit-exact with the oracle."""
    specs = [(40 * MiB + 4096 * 3 + 5, 4 * KiB, C), (24 * MiB, 64 * KiB, C)]
    kw = {"pinned_pool_bytes": 256 * MiB} if where == "pool" else {"numa_node": 0}
    p = mkpair(specs, 29, **kw)
    img = p.g.new_image()
    paths = []
    for epoch, d in [(0, 0.0), (1, 0.005), (2, 0.0), (3, 0.1), (4, 0.001)]:
        if epoch:
            p.write(epoch, d)
        st, want, _ = p.o.checkpoint_gather()
        assert st == 0
        rep = p.g.checkpoint_gather(img)
        assert img.tobytes() == want.tobytes(), epoch
        assert p.shadows_equal(), epoch
        paths.append(rep["path"])
    assert sum(bool(x & crum.PATH_MAPPED) for x in paths) >= 3, paths
    assert any(x & crum.PATH_FUSED for x in paths), paths   # epoch 4: after the 10 % epoch
