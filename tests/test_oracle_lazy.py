"""Oracle lazy restore (the sec. 4.2 read-fault heuristic, PAPER.md:783-793,
applied to restart) pinned to things other than itself:
  * the fault count of a sequential read of an n-page region is the closed
    form ceil(log2(n + 1)) and the windows are 1, 2, 4, ... (SPEC.md:363
    "Fault-count bound"; clamped at the region end);
  * small regions (<= 8 pages) are read in whole on their first fault;
  * after each fault exactly the window's listed pages hold the image's bytes
    (image from the independent builder in tests/imgfmt.py), everything else
    is untouched;
  * begin + any fetch sequence + end == the (already pinned) one-shot restore;
  * error and exclusion rules."""
import math

import numpy as np
import pytest

import synth
from tests import imgfmt

KiB = 1 << 10


def zero_ctx(oracle_mod, specs):
    o = oracle_mod.Oracle()
    zs, rids = [], []
    for nb, P, mode in specs:
        z = oracle_mod.aligned_empty(nb)
        z[:] = 0
        zs.append(z)
        rids.append(o.register(z, P, mode))
    return o, zs, rids


def state_and_image(specs, S, listed, rids):
    """Seeded region contents and an independently built image listing `listed`."""
    cur = []
    for r, (nb, P, _) in enumerate(specs):
        m = np.zeros(nb, dtype=np.uint8)
        synth.fill_region(m, S, r)
        cur.append(m)
    regions = [dict(id=rid, mode=md, cur=m, page_size=P) for rid, m, (_, P, md) in zip(rids, cur, specs)]
    full = all(len(l) == synth.n_pages(nb, P) for l, (nb, P, _) in zip(listed, specs))
    return cur, np.frombuffer(imgfmt.build_image(regions, listed, full=full), dtype=np.uint8).copy()


@pytest.mark.parametrize("n", [9, 16, 17, 31, 32, 100, 1000])
def test_sequential_read_fault_count(oracle_mod, n):
    specs = [(n * 4 * KiB, 4 * KiB, 0)]
    o, zs, rids = zero_ctx(oracle_mod, specs)
    cur, img = state_and_image(specs, synth.seed(60), [list(range(n))], rids)
    assert o.restore_begin(img) == 0
    windows = []
    for i in range(n):
        st, cov, res = o.restore_fetch(rids[0], i)
        assert st == 0 and cov == res
        if cov:
            windows.append(cov)
    assert len(windows) == math.ceil(math.log2(n + 1))
    assert windows[:-1] == [1 << j for j in range(len(windows) - 1)]
    assert sum(windows) == n                        # the last window is clamped at the region end
    assert np.array_equal(zs[0], cur[0])
    assert o.restore_end()[0] == 0


@pytest.mark.parametrize("n", [1, 3, 8])
def test_small_region_read_whole(oracle_mod, n):
    specs = [(n * 4 * KiB - 100, 4 * KiB, 1)]
    o, zs, rids = zero_ctx(oracle_mod, specs)
    listed = [list(range(0, n, 2))]
    cur, img = state_and_image(specs, synth.seed(61), listed, rids)
    assert o.restore_begin(img) == 0
    st, cov, res = o.restore_fetch(rids[0], n - 1)
    assert (st, cov, res) == (0, n, len(listed[0]))
    for i in range(n):
        assert o.restore_fetch(rids[0], i)[1:] == (0, 0)
    P = 4 * KiB
    for i in range(n):
        want = cur[0][i * P:(i + 1) * P] if i in listed[0] else 0
        assert np.all(zs[0][i * P:(i + 1) * P] == want)
    o.restore_end()


def test_windows_hold_image_bytes_only(oracle_mod):
    P = 4 * KiB
    specs = [(40 * P + 123, P, 0), (20 * P, P, 1), (5 * P, P, 0)]
    S = synth.seed(62)
    o, zs, rids = zero_ctx(oracle_mod, specs)
    listed = [sorted(set(range(0, 41, 3)) | {40}), list(range(1, 20, 2)), [0, 4]]
    cur, img = state_and_image(specs, S, listed, rids)
    assert o.restore_begin(img) == 0
    present = [np.zeros(synth.n_pages(nb, P), bool) for nb, _, _ in specs]
    window = [1, 1, 1]
    rng = np.random.default_rng(7)
    for _ in range(40):
        r = int(rng.integers(0, 3))
        n = len(present[r])
        i = int(rng.integers(0, n))
        st, cov, res = o.restore_fetch(rids[r], i)
        assert st == 0
        # the heuristic, restated from PAPER.md:783-793
        if present[r][i]:
            want = []
        elif n <= 8:
            want = [j for j in range(n) if not present[r][j]]
        else:
            want = [j for j in range(i, min(n, i + window[r])) if not present[r][j]]
            window[r] *= 2
        assert cov == len(want)
        assert res == len([j for j in want if j in listed[r]])
        present[r][want] = True
        for rr, (nb, _, _) in enumerate(specs):
            exp = np.zeros(nb, dtype=np.uint8)
            for j in listed[rr]:
                if present[rr][j]:
                    exp[j * P:(j + 1) * P] = cur[rr][j * P:(j + 1) * P]
            assert np.array_equal(zs[rr], exp)
    st, rep = o.restore_end()
    assert st == 0 and rep["dirty_pages"] == sum(len(x) for x in listed)


def test_lazy_equals_eager(oracle_mod):
    specs = [(37 * 4 * KiB + 5, 4 * KiB, 0), (9 * 64 * KiB, 64 * KiB, 1), (3 * 4 * KiB, 4 * KiB, 1)]
    S = synth.seed(63)
    src = oracle_mod.Oracle()
    mems = []
    for r, (nb, P, mode) in enumerate(specs):
        m = oracle_mod.aligned_empty(nb)
        synth.fill_region(m, S, r)
        mems.append(m)
        src.register(m, P, mode)
    src.checkpoint_gather()
    for r, (nb, P, _) in enumerate(specs):
        synth.apply_writer(mems[r], P, synth.choose_dirty(S, 1, r, synth.n_pages(nb, P), 0.4), S, 1, r)
    st, img, _ = src.checkpoint_gather()
    a, za, ra = zero_ctx(oracle_mod, specs)
    b, zb, rb = zero_ctx(oracle_mod, specs)
    st_a, rep_a = a.restore_scatter(img)
    assert st_a == 0
    assert b.restore_begin(img) == 0
    rng = np.random.default_rng(8)
    for _ in range(25):
        r = int(rng.integers(0, 3))
        b.restore_fetch(rb[r], int(rng.integers(0, synth.n_pages(*specs[r][:2]))))
    st_b, rep_b = b.restore_end()
    assert st_b == 0 and rep_a == rep_b
    for r, (nb, P, mode) in enumerate(specs):
        assert np.array_equal(za[r], zb[r])
        assert np.array_equal(a.force_bits(ra[r]), b.force_bits(rb[r]))
        if mode == 1:
            assert np.array_equal(a.hashes(ra[r]), b.hashes(rb[r]))
        else:
            assert np.array_equal(a.mirror(ra[r]), b.mirror(rb[r]))


def test_session_errors_and_exclusion(oracle_mod):
    specs = [(20 * 4 * KiB, 4 * KiB, 0)]
    o, zs, rids = zero_ctx(oracle_mod, specs)
    cur, img = state_and_image(specs, synth.seed(64), [[1, 2, 3]], rids)
    assert o.restore_fetch(rids[0], 0)[0] == oracle_mod.E_INVAL       # no session
    bad = img.copy()
    bad[img.size - 1] ^= 1
    assert o.restore_begin(bad) == oracle_mod.E_CORRUPT
    assert o.restore_fetch(rids[0], 0)[0] == oracle_mod.E_INVAL       # failed begin opens nothing
    assert o.restore_begin(img) == 0
    assert o.restore_begin(img) == oracle_mod.E_BUSY
    assert o.restore_fetch(rids[0], 20)[0] == oracle_mod.E_RANGE
    assert o.restore_fetch(rids[0] + 7, 0)[0] == oracle_mod.E_NOREGION
    assert o.restore_scatter(img)[0] == oracle_mod.E_BUSY
    assert o.checkpoint_gather()[0] == oracle_mod.E_BUSY
    assert zs[0].sum() == 0                                             # nothing written yet
    st, rep = o.restore_end()
    assert st == 0 and rep["dirty_pages"] == 3
    assert o.restore_end()[0] == oracle_mod.E_INVAL
    assert np.array_equal(zs[0][4 * KiB:16 * KiB], cur[0][4 * KiB:16 * KiB])
