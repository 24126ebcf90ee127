"""GPU parity at BASELINE.json's full sizes (C3 16 GiB, C4 64 GiB, C5 240 GiB
oversubscribed UVM), in the launch configuration bench.py times.  The oracle
cannot hold these footprints, so the checks are (a) properties that hold at
any size -- K and the id list equal the written set exactly, both CRC-32s
verify (zlib), restoring the image onto its own state changes nothing and a
sync afterwards finds 0 dirty pages -- and (b) sampled slots the oracle
computes one by one: slot bytes from the seeded recipe, and for hash-mode
slots the listed hash vs the oracle's XXH3 of the expected slot."""
import struct
import zlib

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    return m


def expected_page(S, r, nbytes, P, i, writes):
    """Page i of region r after the epochs in `writes` ({epoch: set(pages)})."""
    lo = i * P
    ln = min(P, nbytes - lo)
    b = synth.region_content(S, r, ln, word_offset=lo // 8)
    full = ln // 8 * 8
    for e in sorted(writes):
        if i in writes[e]:
            m = synth.page_mask(S, e, r, np.array([i]))[0]
            b[:full].view(np.uint64)[:] ^= np.uint64(m)
            if ln > full:
                b[full:ln] ^= np.frombuffer(np.uint64(m).tobytes(), dtype=np.uint8)[:ln - full]
    return b


def check_image(img_head, img_tail, fetch_slot, specs, rids, S, writes_by_region, epoch, rng, nsample=64):
    """img_head: bytes [0, 64+48R); img_tail: bytes [ids_off, image_bytes);
    fetch_slot(offset, n) -> bytes of the image at payload offset."""
    from oracle import oracle
    from tests import imgfmt
    hdr = imgfmt.HDR.unpack_from(img_head, 0)
    magic, ver, flags, R, K, poff, paylen, ids_off, total, mcrc, hcrc = hdr
    assert magic == b"CRUM" and ver == 1 and R == len(specs)
    assert zlib.crc32(img_head[:60]) == hcrc
    table = img_head[64:64 + 48 * R]
    assert zlib.crc32(table + img_tail) == mcrc
    # ids == the pages written in `epoch`, exactly
    ids = list(struct.unpack_from(f"<{K}I", img_tail, 0)) if K else []
    hashes = list(struct.unpack_from(f"<{K}Q", img_tail, (4 * K + 7) // 8 * 8)) if (flags & 2) and K else []
    want_total = 0
    entries = [imgfmt.ENTRY.unpack_from(table, 48 * k) for k in range(R)]
    slot_of = []
    pay = 0
    for r, ((nb, P, mode), e, rid) in enumerate(zip(specs, entries, rids)):
        want = sorted(writes_by_region[r].get(epoch, set()))
        eid, emode, ebytes, eps, enp, nd, first = e
        assert (eid, emode, ebytes, eps, enp) == (rid, mode, nb, P, synth.n_pages(nb, P))
        assert nd == len(want) and first == want_total
        assert ids[first:first + nd] == want
        for j, i in enumerate(want):
            slot_of.append((r, i, pay + j * P, first + j))
        pay += nd * P
        want_total += nd
    assert K == want_total and paylen == pay and ids_off == poff + pay
    # sampled slots: bytes and (hash mode) the listed hash vs the oracle's XXH3
    if slot_of:
        picks = set(rng.choice(len(slot_of), size=min(nsample, len(slot_of)), replace=False).tolist())
        picks |= {0, len(slot_of) - 1}
        for p in sorted(picks):
            r, i, off, k = slot_of[p]
            nb, P, mode = specs[r]
            exp = expected_page(S, r, nb, P, i, writes_by_region[r])
            got = fetch_slot(off, P)
            slot = np.zeros(P, dtype=np.uint8)
            slot[:len(exp)] = exp
            assert np.array_equal(np.frombuffer(got, dtype=np.uint8), slot), (r, i)
            if flags & 2:
                want_h = oracle.xxh3_64(slot) if mode == 1 else 0
                assert hashes[k] == want_h, (r, i)


def make_regions(crum, specs, S, managed=None):
    g = crum.Context(0)
    regs, rids = [], []
    for r, (nb, P, mode) in enumerate(specs):
        if managed is not None:
            t = managed[r]
        else:
            t = torch.empty(nb, dtype=torch.uint8, device="cuda")
        crum.synth_fill(t, nb, S, r)
        regs.append(t)
    torch.cuda.synchronize()
    for r, (nb, P, mode) in enumerate(specs):
        rids.append(g.register_region(regs[r], nb, P, mode))
    return g, regs, rids


def write_epoch(crum, regs, specs, S, epoch, d, writes):
    for r, (nb, P, _) in enumerate(specs):
        pages = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), d)
        writes[r][epoch] = set(pages.tolist())
        if len(pages):
            dp = torch.from_numpy(pages.astype(np.uint32)).cuda()
            crum.synth_write_pages(regs[r], nb, P, dp, len(pages), S, epoch, r)
    torch.cuda.synchronize()


def run_incremental(crum, specs, S, managed=None, d=0.1, host_image=True, nsample=64):
    g, regs, rids = make_regions(crum, specs, S, managed)
    N = sum(synth.n_pages(nb, P) for nb, P, _ in specs)
    assert g.sync_shadow() == N          # epoch 0: commit everything (all force-dirty)
    writes = [dict() for _ in specs]
    write_epoch(crum, regs, specs, S, 1, d, writes)
    rng = np.random.default_rng(S)
    R = len(specs)
    if host_image:
        img = g.new_image(g.image_required_bytes(sum(synth.dirty_count(d, synth.n_pages(nb, P))
                                                     for nb, P, _ in specs)))
        rep = g.checkpoint_gather(img)
        v = img.view()
        head = v[:64 + 48 * R].tobytes()
        ids_off = struct.unpack_from("<Q", head, 40)[0]
        tail = v[ids_off:img.length].tobytes()
        poff = struct.unpack_from("<Q", head, 24)[0]
        fetch = lambda off, n: v[poff + off:poff + off + n].tobytes()
    else:
        raise NotImplementedError
    check_image(head, tail, fetch, specs, rids, S, writes, 1, rng, nsample)
    assert rep["dirty_pages"] == sum(len(w[1]) for w in writes)
    # restoring the image onto its own state changes nothing; nothing is dirty after
    g.restore_scatter(img)
    assert g.sync_shadow() == 0
    return g, regs, img


@pytest.fixture(autouse=True)
def _release_memory():
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    yield
    gc.collect()
    torch.cuda.empty_cache()


def test_c3_fullsize_sampled(crum):
    sizes = synth.c3_region_sizes(20)
    specs = [(s, 64 * KiB, 0 if i % 3 else 1) for i, s in enumerate(sizes)]
    g, regs, img = run_incremental(crum, specs, synth.seed(3))
    img.destroy()
    g.close()


def _full_oracle_run(crum, specs, S, d, full=False, touch=False):
    """Register the full footprint, commit it, copy the committed content to
    the host, rewrite a d-fraction of pages (device writer) and gather into a
    pinned image; then check EVERY byte of that image against the oracle
    region by region (tests/fullparity.py)."""
    from tests import fullparity
    g, regs, rids = make_regions(crum, specs, S)
    N = sum(synth.n_pages(nb, P) for nb, P, _ in specs)
    assert g.sync_shadow() == N
    host = [r.cpu().numpy() for r in regs]          # committed state (epoch 0)
    writes = [dict() for _ in specs]
    if not full:
        write_epoch(crum, regs, specs, S, 1, d, writes)
    kmax = N if full else sum(synth.dirty_count(d, synth.n_pages(nb, P)) for nb, P, _ in specs)
    img = g.new_image(g.image_required_bytes(kmax))
    rep = g.checkpoint_gather(img, flags=crum.FULL if full else 0)
    res = fullparity.regionwise_check(img.view(), specs, rids, lambda r: host[r], S, 1, d, touch=touch, full=full)
    assert res["ok"] and res["image_bytes"] == rep["image_bytes"] == img.length, res
    assert res["dirty_pages"] == rep["dirty_pages"]
    return g, regs, img, host


def test_c3_full_image_bit_exact_incremental(crum):
    """C3 (15.96 GiB, 220 Rodinia-shaped regions, both modes), 10% rewritten:
    every byte of the 1.7 GB incremental image equals the oracle's."""
    sizes = synth.c3_region_sizes(20)
    specs = [(s, 64 * KiB, 0 if i % 3 else 1) for i, s in enumerate(sizes)]
    g, regs, img, host = _full_oracle_run(crum, specs, synth.seed(3), 0.1)
    img.destroy()
    g.close()


def test_c3_full_checkpoint_and_full_restore(crum):
    """C3 (a): FULL checkpoint (17.1 GB image, every byte checked against the
    oracle), then a full restore onto zeroed regions of a fresh context
    reproduces every region byte for byte."""
    sizes = synth.c3_region_sizes(20)
    specs = [(s, 64 * KiB, 0 if i % 3 else 1) for i, s in enumerate(sizes)]
    g, regs, img, host = _full_oracle_run(crum, specs, synth.seed(3), 0.0, full=True)
    g.close()
    del regs
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    q = crum.Context(0)
    zs = []
    for nb, P, mode in specs:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, mode)
    rep = q.restore_scatter(img, flags=crum.VERIFY)
    assert rep["dirty_pages"] == sum(synth.n_pages(nb, P) for nb, P, _ in specs)
    torch.cuda.synchronize()
    for z, h in zip(zs, host):
        assert np.array_equal(z.cpu().numpy(), h)
    assert q.sync_shadow() == 0
    img.destroy()
    q.close()


def test_c4_full_image_bit_exact(crum):
    """C4 (64.2 GiB per GPU: 56 multigrid vectors at 64 KiB pages + 4096 box
    regions at 4 KiB pages), 10% rewritten, compare mode -- the bench's
    headline configuration: every byte of the 6.9 GB image equals the
    oracle's (checked region by region)."""
    big, small = synth.c4_region_sizes(synth.seed(4))
    specs = [(s, 64 * KiB, 0) for s in big] + [(s, 4 * KiB, 0) for s in small]
    g, regs, img, host = _full_oracle_run(crum, specs, synth.seed(4), 0.1)
    img.destroy()
    g.close()


def test_c4_hash_full_image_bit_exact(crum):
    """C4 in hash mode (the page-group TMA kernel at 64 KiB pages over 64 GiB):
    every byte of the image, hashes included, equals the oracle's."""
    big, small = synth.c4_region_sizes(synth.seed(4))
    specs = [(s, 64 * KiB, 1) for s in big] + [(s, 4 * KiB, 1) for s in small]
    g, regs, img, host = _full_oracle_run(crum, specs, synth.seed(4) + 7, 0.1)
    img.destroy()
    g.close()


def test_c4_fullsize_sampled(crum):
    big, small = synth.c4_region_sizes(synth.seed(4))
    specs = [(s, 64 * KiB, 0) for s in big] + [(s, 4 * KiB, 0) for s in small]
    assert abs(sum(s for s, _, _ in specs) / GiB - 64.19) < 0.05
    g, regs, img = run_incremental(crum, specs, synth.seed(4), nsample=96)
    img.destroy()
    g.close()


def test_c5_managed_host_resident_sampled(crum):
    """UVM (managed) regions with host-resident pages, C5 shape at the scale
    the GPU box's sandbox allows (it caps cudaMallocManaged at ~56 GiB in
    total): 2 x 24 GiB managed, 37.5% of each host-preferred
    + accessed-by (read over the host link, as 90 of C5's 240 GiB), hash mode,
    2 MiB pages, 10% rewritten."""
    region = 24 * GiB
    bufs = [crum.ManagedBuffer(region, 0, 15 * GiB) for _ in range(2)]
    specs = [(region, 2 * MiB, 1), (region, 2 * MiB, 1)]
    try:
        g, regs, img = run_incremental(crum, specs, synth.seed(5), managed=bufs, nsample=24)
        img.destroy()
        g.close()
    finally:
        for b in bufs:
            b.free()


def test_c5_oversubscribed_hostmapped_sampled(crum):
    """A footprint larger than HBM (192 GiB > 178 GiB): 160 GiB of device
    regions plus 32 GiB of pinned host memory mapped into the GPU's address
    space (host-resident pages read over the host link), hash mode, 2 MiB
    pages, 10% rewritten."""
    import os
    if os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") < 96 * GiB:
        pytest.skip("host RAM too small")
    host = [torch.empty(16 * GiB, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    dev = [80 * GiB, 80 * GiB]
    bufs = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in dev] + host
    specs = [(b.numel(), 2 * MiB, 1) for b in bufs]
    g, regs, img = run_incremental(crum, specs, synth.seed(5), managed=bufs, nsample=24)
    img.destroy()
    g.close()
    del bufs, host, regs
