"""GPU parity of every kernel path the library ships, selected per context by
crum_config (include/crum.h): the captured-graph replay vs direct launches
(CRUM_CFG_NO_GRAPH) and the single-pass detect+compact+gather kernel
(CRUM_CFG_FUSED) vs the multi-kernel path, the mapped-store pinned gathers vs
the ring + D2H pipeline (CRUM_CFG_NO_MAPPED), each bit-exact with the oracle on
the same seeded inputs; the pinned pool (crum_config.pinned_pool_bytes) and
the transactional register / unregister (a failed rebuild changes nothing)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30
C, H = 0, 1

# all COMPARE with P <= 64 KiB: eligible for the single-pass kernel
FUSABLE = [
    (4 * MiB, 4 * KiB, C),
    (3 * 64 * KiB + 1234, 64 * KiB, C),     # ragged tail page
    (5 * 4 * KiB + 17, 4 * KiB, C),
    (32 * MiB + 4096, 64 * KiB, C),         # several tiles, partial last page
    (12 * KiB + 256, 4 * KiB, C),
]
# one page size, compare only, 5.1 MiB: the one-launch small path (k_small_ckpt)
SMALL = [(4 * MiB, 4 * KiB, C), (12 * KiB + 256, 4 * KiB, C), (1 * MiB + 4096 * 3 + 5, 4 * KiB, C)]
# the same kind, above the default single-pass threshold (64 MiB): the
# multi-kernel path unless CRUM_CFG_FUSED asks for the single pass
FUSABLE_BIG = FUSABLE + [(40 * MiB + 12288, 64 * KiB, C)]
MIXED = [
    (4 * MiB, 4 * KiB, C),
    (3 * 64 * KiB + 1234, 64 * KiB, H),
    (5 * 4 * KiB + 17, 4 * KiB, H),
    (2 * MiB + 4 * KiB + 100, 2 * MiB, C),
    (12 * KiB + 256, 4 * KiB, C),
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


def variants():
    from paper_1808_00117_b200 import crum as m
    return [("default", 0), ("no_graph", m.CFG_NO_GRAPH), ("fused", m.CFG_FUSED),
            ("fused_no_graph", m.CFG_FUSED | m.CFG_NO_GRAPH), ("no_mapped", m.CFG_NO_MAPPED)]


@pytest.mark.parametrize("specs_name", ["small", "fusable", "fusable_big", "mixed"])
@pytest.mark.parametrize("variant", [v[0] for v in variants()])
def test_every_path_bit_exact(crum, variant, specs_name):
    """Device image (asynchronous: graph replay unless NO_GRAPH; synchronous
    with a report), host image and sync, epoch by epoch, every dirty ratio and
    FULL: image bytes, reports and snapshots equal the oracle's."""
    flags = dict(variants())[variant]
    specs = {"small": SMALL, "fusable": FUSABLE, "fusable_big": FUSABLE_BIG, "mixed": MIXED}[specs_name]
    small = sum(nb for nb, _, _ in specs) <= 64 * MiB
    p = mkpair(specs, 40, flags=flags)
    cap = p.g.image_required_bytes()
    dbuf = torch.empty(cap + 4096, dtype=torch.uint8, device="cuda")
    img = p.g.new_image()
    seq = [(0, 0.0, 0, "dev_async"), (1, 0.1, 0, "dev_async"), (2, 0.5, 0, "dev_sync"), (3, 0.0, 0, "dev_async"),
           (4, 1.0, 0, "host"), (5, 0.2, crum.FULL, "dev_async"), (6, 0.3, 0, "sync"), (7, 0.05, 0, "dev_async"),
           (8, 0.7, 0, "host"), (9, 0.0, 0, "dev_sync")]
    prev_frac = 0.0  # dirty fraction of the previous call (the adaptive single-pass rule)
    prev_payload = None  # payload of the previous gather (the mapped-store rule)
    host_gathers = 0
    for epoch, d, gflags, how in seq:
        if epoch:
            p.write(epoch, d)
        if how == "sync":
            n = p.g.sync_shadow()
            assert n == p.o.sync_shadow()
            assert p.shadows_equal()
            prev_frac = n / p.N
            continue
        st, want, rep_o = p.o.checkpoint_gather(flags=gflags)
        assert st == 0
        if how == "host":
            rep = p.g.checkpoint_gather(img, flags=gflags)
            got = img.tobytes()
        else:
            rep = p.g.checkpoint_gather_device(dbuf, cap, flags=gflags, report=(how == "dev_sync"))
            if rep is None:
                rep = p.g.last_report()
            torch.cuda.synchronize()
            got = dbuf[:len(want)].cpu().numpy().tobytes()
        assert rep["image_bytes"] == len(want), (epoch, how)
        assert got == want.tobytes(), (variant, epoch, how)
        for k in ("dirty_pages", "dirty_bytes", "image_bytes"):
            assert rep[k] == rep_o[k], (epoch, k)
        # single pass: compare-only, incremental, device image (the pinned
        # path of these footprints is the range pipeline), and either asked
        # for or a footprint <= 64 MiB (the default)
        # (a pinned image of the small footprint takes the small path too)
        # Above 64 MiB the single pass also runs when the previous call listed
        # >= 25 % of the pages (adaptive rule)
        fused_eligible = (specs_name != "mixed" and not gflags and
                          (how != "host" or specs_name == "small") and
                          (variant.startswith("fused") or small or prev_frac >= 0.25))
        # a pinned gather above the small-footprint size (worst case > 16 MiB:
        # FUSABLE, FUSABLE_BIG) whose previous payload was <= 32 MiB (not the
        # first since registration) stores through the image's mapped address;
        # the single pass there above 2 MiB (these sets are compare-only)
        mapped = (how == "host" and specs_name in ("fusable", "fusable_big") and not gflags and host_gathers > 0 and
                  variant != "no_mapped" and prev_payload is not None and prev_payload <= 32 * MiB)
        assert bool(rep["path"] & crum.PATH_MAPPED) == mapped, (variant, epoch, how, rep["path"])
        if mapped:
            fused_eligible = prev_payload > 2 * MiB
        prev_frac = rep_o["dirty_pages"] / p.N
        prev_payload = int.from_bytes(want.tobytes()[32:40], "little")
        host_gathers += how == "host"
        assert bool(rep["path"] & crum.PATH_FUSED) == fused_eligible, (variant, epoch, how, rep["path"])
        # the one-launch kernel: one page size, compare-only, <= 16384 pages
        assert bool(rep["path"] & crum.PATH_SMALL) == (fused_eligible and specs_name == "small"), \
            (variant, epoch, how, rep["path"])
        assert p.shadows_equal(), (variant, epoch)


@pytest.mark.parametrize("flags_name", ["fused", "default"])
def test_back_to_back_async_gathers(crum, flags_name):
    """Many stream-asynchronous device gathers in a row on one stream, each
    checked: the single-pass kernel's ticket / done scratch is reset
    stream-ordered before every launch (a late warp must never restart the
    tile sequence), and the look-back tags wrap after 255 launches."""
    flags = crum.CFG_FUSED if flags_name == "fused" else 0
    specs = [(256 * MiB, 64 * KiB, C), (8 * MiB + 4096, 4 * KiB, C)]
    p = mkpair(specs, 41, flags=flags)
    cap = p.g.image_required_bytes()
    bufs = [torch.empty(cap + 4096, dtype=torch.uint8, device="cuda") for _ in range(2)]
    p.g.sync_shadow()
    p.o.sync_shadow()
    rng = np.random.default_rng(41)
    for epoch in range(1, 41):
        d = float(rng.choice([0.0, 0.01, 0.1, 0.3]))
        p.write(epoch, d)
        buf = bufs[epoch % 2]
        p.g.checkpoint_gather_device(buf, cap, report=False)
        st, want, _ = p.o.checkpoint_gather()
        torch.cuda.synchronize()
        assert buf[:len(want)].cpu().numpy().tobytes() == want.tobytes(), epoch
    # tag wrap: 260 more empty checkpoints, then one with changes
    for _ in range(260):
        p.g.checkpoint_gather_device(bufs[0], cap, report=False)
    p.o.checkpoint_gather()
    p.write(100, 0.2)
    st, want, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather_device(bufs[1], cap, report=False)
    torch.cuda.synchronize()
    assert bufs[1][:len(want)].cpu().numpy().tobytes() == want.tobytes()


def test_pinned_pool(crum):
    """Images carved from the context's pinned pool: first fit, freed ranges
    coalesce, an image that does not fit gets its own allocation, and a pooled
    image's bytes equal the oracle's."""
    pool = 64 * MiB
    p = mkpair(MIXED, 42, pinned_pool_bytes=pool)
    info = p.g.pool_info()
    assert info == {"bytes": pool, "in_use": 0, "largest_free": pool, "images": 0}
    a = p.g.new_image(10 * MiB + 1)
    b = p.g.new_image(20 * MiB)
    c = p.g.new_image(8 * MiB)
    info = p.g.pool_info()
    assert info["images"] == 3 and info["in_use"] == 10 * MiB + 4096 + 28 * MiB
    big = p.g.new_image(40 * MiB)          # does not fit: its own allocation
    assert p.g.pool_info()["images"] == 3
    b.destroy()                            # b's extent is not adjacent to the tail (c in between)
    assert p.g.pool_info()["largest_free"] == pool - (38 * MiB + 4096)
    a.destroy()                            # a + b coalesce
    assert p.g.pool_info()["largest_free"] == 30 * MiB + 4096
    c.destroy()
    info = p.g.pool_info()
    assert info == {"bytes": pool, "in_use": 0, "largest_free": pool, "images": 0}   # fully coalesced
    img = p.g.new_image()
    assert p.g.pool_info()["images"] == 1
    for epoch, d in ((0, 0), (1, 0.3)):
        if epoch:
            p.write(epoch, d)
        st, want, _ = p.o.checkpoint_gather()
        p.g.checkpoint_gather(img)
        assert img.tobytes() == want.tobytes(), epoch
    img.destroy()
    big.destroy()
    assert p.g.pool_info()["images"] == 0


def test_register_rollback_on_nomem(crum):
    """A register whose rebuild runs out of device memory returns NOMEM and
    changes nothing: the old registry keeps working, bit-exact."""
    p = mkpair([(8 * MiB, 64 * KiB, C), (3 * 4096 + 5, 4096, H)], 43)
    p.g.sync_shadow()
    p.o.sync_shadow()
    nb = 4 * GiB                       # hash mode at 4 KiB pages: 1 Mi pages, 8 MiB table
    region = torch.empty(nb, dtype=torch.uint8, device="cuda")
    free, _ = torch.cuda.mem_get_info()
    # leave room for the 8 MiB table (+ force bits) but not the ~40 B/page arrays
    hog = torch.empty(max(0, free - 24 * MiB), dtype=torch.uint8, device="cuda")
    st = p.g.try_register(region.data_ptr(), nb, 4096, H)
    del hog
    torch.cuda.empty_cache()
    assert st == crum.E_NOMEM, st
    assert p.g.image_required_bytes() == p.o.required_bytes()
    p.write(1, 0.4)
    st, want, _ = p.o.checkpoint_gather()
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()
    # and a later register succeeds
    rid = p.g.register_region(region, nb, 4096, H)
    assert rid == 3
    p.g.unregister_region(rid)


@pytest.mark.parametrize("specs_name", ["small", "fusable_big"])
def test_phase_times_reported(crum, specs_name):
    """CRUM_CFG_TIMING: the small kernel times itself (t_detect = t_total =
    its own duration, no events around it); the multi-kernel path reports its
    phases from events.  Without the flag an asynchronous device-image call
    reports no times (a pinned-image gather and a synchronous report always
    time their call).  Images stay bit-exact
    either way."""
    specs = {"small": SMALL, "fusable_big": FUSABLE_BIG}[specs_name]
    for timing in (True, False):
        p = mkpair(specs, 41, timing=timing)
        img = p.g.new_image()
        for epoch, d in ((0, 0.0), (1, 0.1), (2, 0.02)):
            if epoch:
                p.write(epoch, d)
            st, want, _ = p.o.checkpoint_gather()
            rep = p.g.checkpoint_gather(img)
            assert img.tobytes() == want.tobytes()
            if not timing:  # (a pinned-image gather times itself regardless)
                continue
            assert 0 < rep["t_detect_ms"] <= rep["t_total_ms"] < 1e3, rep
            if specs_name == "small":
                assert rep["path"] & crum.PATH_SMALL
                assert rep["t_detect_ms"] == rep["t_total_ms"] and rep["t_compact_ms"] == 0
            else:
                assert not rep["path"] & crum.PATH_SMALL
        # the device image path: asynchronous (timed only under the flag; a
        # synchronous report always times its call)
        dbuf = torch.empty(p.g.image_required_bytes() + 256, dtype=torch.uint8, device="cuda")
        p.write(3, 0.05)
        st, want, _ = p.o.checkpoint_gather()
        assert p.g.checkpoint_gather_device(dbuf, p.g.image_required_bytes(), report=False) is None
        rep = p.g.last_report()
        assert dbuf[:len(want)].cpu().numpy().tobytes() == want.tobytes()
        assert (rep["t_total_ms"] > 0) == timing, rep
        assert bool(rep["path"] & crum.PATH_SMALL) == (specs_name == "small")
