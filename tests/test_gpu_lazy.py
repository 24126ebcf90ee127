"""GPU parity of the lazy restore (sec. 4.2 read-fault heuristic applied to
restart): libcrum.so's crum_restore_begin / fetch / end vs
the CPU oracle's, bit-exact after every fault (region bytes, counts) and at
the end (regions, mirrors, hash tables, force bits, report)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB = 1 << 10, 1 << 20
C, H = 0, 1
SPECS = [
    (3 * MiB + 777, 4 * KiB, C),       # 769 pages
    (40 * 64 * KiB, 64 * KiB, H),      # 40 pages
    (5 * 4 * KiB + 9, 4 * KiB, H),     # small (6 pages): read whole
    (2 * MiB * 4 + 100, 2 * MiB, C),   # 5 pages, 2 MiB, tiny tail
    (300 * 4 * KiB, 4 * KiB, H),
]


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    assert torch.cuda.is_available()
    return m


def restart_pair(crum, specs):
    """Fresh oracle + fresh device context over zeroed regions."""
    from oracle import oracle
    o = oracle.Oracle()
    g = crum.Context(0)
    hz, dz, ro, rg = [], [], [], []
    for nb, P, mode in specs:
        h = oracle.aligned_empty(nb)
        h[:] = 0
        d = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        hz.append(h)
        dz.append(d)
        ro.append(o.register(h, P, mode))
        rg.append(g.register_region(d, nb, P, mode))
    return o, g, hz, dz, ro, rg


def source_image(crum, seed_idx, d=0.35):
    from tests.gpu_pair import Pair
    p = Pair(SPECS, synth.seed(seed_idx))
    img = p.g.new_image()
    p.o.checkpoint_gather()
    p.g.checkpoint_gather(img)
    p.write(1, d)
    st, want, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather(img)
    assert img.tobytes() == want.tobytes()
    return p, want


@pytest.mark.parametrize("verify", [0, 1])
def test_lazy_restore_parity_random_faults(crum, verify):
    p, raw = source_image(crum, 70)
    o, g, hz, dz, ro, rg = restart_pair(crum, SPECS)
    gimg = g.import_image(raw)
    flags = crum.VERIFY if verify else 0
    assert o.restore_begin(raw, flags) == 0
    sess = g.restore_begin(gimg, flags=flags)
    rng = np.random.default_rng(9 + verify)
    for step in range(120):
        r = int(rng.integers(0, len(SPECS)))
        n = synth.n_pages(*SPECS[r][:2])
        i = int(rng.integers(0, n)) if rng.random() < 0.5 else min(n - 1, step % n)
        st, cov, res = o.restore_fetch(ro[r], i)
        assert st == 0
        assert sess.fetch(rg[r], i) == (cov, res), (step, r, i)
        if step % 10 == 0 or cov:
            torch.cuda.synchronize()
            assert np.array_equal(dz[r].cpu().numpy(), hz[r]), (step, r)
    st, rep_o = o.restore_end()
    rep = sess.end()
    assert st == 0
    for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes", "scanned_pages", "scanned_bytes"):
        assert rep[k] == rep_o[k], k
    torch.cuda.synchronize()
    for r, (nb, P, mode) in enumerate(SPECS):
        n = synth.n_pages(nb, P)
        assert np.array_equal(dz[r].cpu().numpy(), hz[r]), r
        assert np.array_equal(g.debug_export(rg[r], crum.EXPORT_FORCE, n), o.force_bits(ro[r]))
        if mode == H:
            assert np.array_equal(g.debug_export(rg[r], crum.EXPORT_HASHES, n), o.hashes(ro[r]))
        else:
            assert np.array_equal(g.debug_export(rg[r], crum.EXPORT_MIRROR, nb), o.mirror(ro[r]))
    assert g.sync_shadow() == o.sync_shadow()


def test_lazy_sequential_fault_count(crum):
    p, raw = source_image(crum, 71, d=1.0)
    o, g, hz, dz, ro, rg = restart_pair(crum, SPECS)
    gimg = g.import_image(raw)
    with g.restore_begin(gimg) as sess:
        for r, (nb, P, _) in enumerate(SPECS):
            n = synth.n_pages(nb, P)
            faults = [c for c in (sess.fetch(rg[r], i)[0] for i in range(n)) if c]
            want = 1 if n <= 8 else int(np.ceil(np.log2(n + 1)))
            assert len(faults) == want and sum(faults) == n, r
        torch.cuda.synchronize()
        for d, h in zip(dz, p.host):
            assert np.array_equal(d.cpu().numpy(), h)


def test_lazy_exclusion_and_errors(crum):
    p, raw = source_image(crum, 72)
    o, g, hz, dz, ro, rg = restart_pair(crum, SPECS)
    gimg = g.import_image(raw)
    other = g.new_image()
    sess = g.restore_begin(gimg)
    with pytest.raises(crum.CrumError) as e:
        g.restore_begin(gimg)
    assert e.value.status == crum.E_BUSY
    with pytest.raises(crum.CrumError) as e:
        g.sync_shadow()
    assert e.value.status == crum.E_BUSY
    st, _ = g.checkpoint_gather(other, raise_on_error=False)
    assert st == crum.E_BUSY
    with pytest.raises(crum.CrumError) as e:
        gimg.destroy()
    assert e.value.status == crum.E_BUSY
    with pytest.raises(crum.CrumError) as e:
        sess.fetch(rg[0], 1 << 40)
    assert e.value.status == crum.E_RANGE
    with pytest.raises(crum.CrumError) as e:
        sess.fetch(999, 0)
    assert e.value.status == crum.E_NOREGION
    torch.cuda.synchronize()
    assert all(int(d.count_nonzero()) == 0 for d in dz)            # begin wrote nothing
    sess.end()
    g.checkpoint_gather(other)                                     # free again
    gimg.destroy()
    # a corrupted hash slot is caught by begin(VERIFY) before anything is written
    o2, g2, _, dz2, _, _ = restart_pair(crum, SPECS)
    from tests import imgfmt
    info = imgfmt.parse_image(raw)
    k_hash = next(k for k, e in enumerate(info["table"]) if e[1] == H and e[5] > 0)
    first = info["table"][k_hash][6]
    off = info["poff"] + sum(e[5] * e[3] for e in info["table"][:k_hash])
    bad = raw.copy()
    bad[off + 5] ^= 0x40
    assert first >= 0
    with pytest.raises(crum.CrumError) as e:
        g2.restore_begin(g2.import_image(bad), flags=crum.VERIFY)
    assert e.value.status == crum.E_CORRUPT
    torch.cuda.synchronize()
    assert all(int(d.count_nonzero()) == 0 for d in dz2)
