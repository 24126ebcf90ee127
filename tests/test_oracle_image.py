"""Oracle gather/restore pinned to: the independent format builder in
tests/imgfmt.py (zlib + xxhash + struct), the round-trip invariants
restore(state_{k-1}, ckpt_k) == state_k,
corruption detection and the SPEC run-coalescing example
(SPEC.md:378)."""
import os

import numpy as np
import pytest

import synth
from tests import imgfmt

HERE = os.path.dirname(os.path.abspath(__file__))


def make_ctx(oracle_mod, specs, S):
    """specs: list of (nbytes, page_size, mode)."""
    o = oracle_mod.Oracle()
    mems, rids = [], []
    for r, (nb, P, mode) in enumerate(specs):
        m = oracle_mod.aligned_empty(nb)
        synth.fill_region(m, S, r)
        mems.append(m)
        rids.append(o.register(m, P, mode))
    return o, mems, rids


SPECS = [(5 * 4096 + 333, 4096, 0), (3 * 65536, 65536, 1), (4096 * 7, 4096, 1), (8192, 4096, 0)]


def dirty_epoch(mems, specs, S, epoch, d):
    listed = []
    for r, (m, (nb, P, _)) in enumerate(zip(mems, specs)):
        pages = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), d)
        synth.apply_writer(m, P, pages, S, epoch, r)
        listed.append(pages.tolist())
    return listed


@pytest.mark.parametrize("full", [False, True])
def test_image_bytes_match_independent_builder(oracle_mod, full):
    S = synth.seed(3)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    st, img0, rep0 = o.checkpoint_gather()
    assert st == 0
    regions = [dict(id=rid, mode=md, cur=m, page_size=P) for rid, m, (_, P, md) in zip(rids, mems, SPECS)]
    every = [list(range(synth.n_pages(nb, P))) for nb, P, _ in SPECS]
    assert bytes(img0) == imgfmt.build_image(regions, every, full=False)  # first gather is full (Q3)
    assert rep0["dirty_pages"] == sum(len(x) for x in every)
    listed = dirty_epoch(mems, SPECS, S, 1, 0.4)
    st, img, rep = o.checkpoint_gather(flags=oracle_mod.FULL if full else 0)
    assert st == 0
    want = imgfmt.build_image(regions, every if full else listed, full=full)
    assert bytes(img) == want
    assert rep["image_bytes"] == len(want)
    assert rep["dirty_pages"] == sum(len(x) for x in (every if full else listed))


def test_restore_chain_and_full_restore(oracle_mod):
    S = synth.seed(4)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    st, img0, _ = o.checkpoint_gather()
    states = [[m.copy() for m in mems]]
    imgs = [img0]
    for epoch in range(1, 6):
        dirty_epoch(mems, SPECS, S, epoch, 0.3)
        st, img, _ = o.checkpoint_gather()
        assert st == 0
        imgs.append(img)
        states.append([m.copy() for m in mems])
    # restart: fresh context over zeroed regions, replay the chain of 6 images
    o2 = oracle_mod.Oracle()
    zm = []
    for nb, P, mode in SPECS:
        z = oracle_mod.aligned_empty(nb)
        z[:] = 0
        zm.append(z)
        o2.register(z, P, mode)
    for k, img in enumerate(imgs):
        st, rep = o2.restore_scatter(img, oracle_mod.VERIFY)
        assert st == 0
        for z, want in zip(zm, states[k]):
            assert np.array_equal(z, want), k
    assert o2.sync_shadow() == 0     # restore commits what it writes
    # full image onto zeros == x
    o3 = oracle_mod.Oracle()
    zz = []
    for nb, P, mode in SPECS:
        z = oracle_mod.aligned_empty(nb)
        z[:] = 0
        zz.append(z)
        o3.register(z, P, mode)
    st, full_img, _ = o.checkpoint_gather(flags=oracle_mod.FULL)
    assert o3.restore_scatter(full_img)[0] == 0
    for z, m in zip(zz, mems):
        assert np.array_equal(z, m)


def test_capacity_error_changes_nothing(oracle_mod):
    S = synth.seed(5)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    need = o.required_bytes()
    st, img, rep = o.checkpoint_gather(capacity=need - 1 - 4096 * 3)
    assert st == oracle_mod.E_CAPACITY and img is None
    assert rep["image_bytes"] > need - 1 - 4096 * 3
    assert all(o.force_bits(r).all() for r in rids)   # nothing committed
    st, img, rep2 = o.checkpoint_gather(capacity=rep["image_bytes"])
    assert st == 0 and len(img) == rep["image_bytes"]


def test_zero_dirty_image(oracle_mod):
    """Reading Q18: zero dirty pages still gives a header + table image."""
    S = synth.seed(6)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    o.sync_shadow()
    st, img, rep = o.checkpoint_gather()
    assert st == 0 and rep["dirty_pages"] == 0 and rep["dirty_bytes"] == 0
    p = imgfmt.parse_image(img)
    assert p["K"] == 0 and p["payload_bytes"] == 0 and len(img) == p["poff"] == 4096


def test_corruption_and_truncation_detected(oracle_mod):
    S = synth.seed(7)
    o, mems, rids = make_ctx(oracle_mod, [(3 * 4096, 4096, 0), (2 * 4096, 4096, 1)], S)
    st, img, _ = o.checkpoint_gather()
    before = [m.copy() for m in mems]
    for pos in imgfmt.meta_positions(img):
        bad = img.copy()
        bad[pos] ^= 0x04
        assert o.restore_scatter(bad)[0] == oracle_mod.E_CORRUPT, pos
    assert o.restore_scatter(img[:-1])[0] == oracle_mod.E_CORRUPT
    assert o.restore_scatter(img[:63])[0] == oracle_mod.E_CORRUPT
    for m, b in zip(mems, before):
        assert np.array_equal(m, b)
    # payload of a hash-mode slot tampered: only VERIFY notices
    bad = img.copy()
    bad[imgfmt.parse_image(img)["ids_off"] - 1] ^= 0xFF   # last byte of the last (hash-mode) slot
    assert o.restore_scatter(bad, oracle_mod.VERIFY)[0] == oracle_mod.E_CORRUPT
    assert o.restore_scatter(bad)[0] == 0


def test_mismatch_leaves_state(oracle_mod):
    S = synth.seed(8)
    o, mems, rids = make_ctx(oracle_mod, [(3 * 4096, 4096, 0)], S)
    st, img, _ = o.checkpoint_gather()
    o2, mems2, _ = make_ctx(oracle_mod, [(4 * 4096, 4096, 0)], S)
    before = mems2[0].copy()
    assert o2.restore_scatter(img)[0] == oracle_mod.E_MISMATCH
    assert np.array_equal(mems2[0], before)
    o3, _, _ = make_ctx(oracle_mod, [(3 * 4096, 4096, 1)], S)          # mode differs
    assert o3.restore_scatter(img)[0] == oracle_mod.E_MISMATCH


def test_spec_run_example(oracle_mod):
    """pages {3,4,5,9} dirty -> runs [3..5] and [9] (2 runs)."""
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(16 * P)
    synth.fill_region(mem, synth.seed(0), 0)
    rid = o.register(mem, P, 0)
    o.sync_shadow()
    for i in (3, 4, 5, 9):
        mem[i * P + 100] ^= 1
    st, img, rep = o.checkpoint_gather()
    assert rep["dirty_pages"] == 4 and rep["dirty_runs"] == 2
    assert imgfmt.parse_image(img)["ids"] == [3, 4, 5, 9]


def test_golden_fixture(oracle_mod):
    """tests/golden/spec_examples.txt: the SPEC/paper behavioural examples."""
    path = os.path.join(HERE, "golden", "spec_examples.txt")
    rows = [l.split("|") for l in open(path) if l.strip() and not l.startswith("#")]
    for name, pages, dirty, want_k, want_runs, _cite in rows:
        P = 4096
        n = int(pages)
        o = oracle_mod.Oracle()
        mem = oracle_mod.aligned_empty(n * P)
        synth.fill_region(mem, synth.seed(0), 0)
        o.register(mem, P, 0)
        if dirty.strip() != "ALL":
            o.sync_shadow()
            for i in [int(x) for x in dirty.split()] if dirty.strip() else []:
                mem[i * P] ^= 1
        st, img, rep = o.checkpoint_gather()
        assert st == 0
        assert rep["dirty_pages"] == int(want_k), name
        assert rep["dirty_runs"] == int(want_runs), name


def test_deterministic_image(oracle_mod):
    """fixed seed -> identical image bytes."""
    imgs = []
    for _ in range(2):
        S = synth.seed(9)
        o, mems, rids = make_ctx(oracle_mod, SPECS, S)
        o.checkpoint_gather()
        dirty_epoch(mems, SPECS, S, 1, 0.5)
        imgs.append(o.checkpoint_gather()[1].tobytes())
    assert imgs[0] == imgs[1]


def test_tracked_mode_image_and_restore(oracle_mod):
    """Images of TRACKED regions list the marked pages with the bytes they hold
    at gather time; hash entries are 0; restore replays them."""
    S = synth.seed(11)
    specs = [(6 * 4096 + 10, 4096, 2), (2 * 65536, 65536, 1), (3 * 4096, 4096, 0)]
    o, mems, rids = make_ctx(oracle_mod, specs, S)
    st, img0, _ = o.checkpoint_gather()
    regions = [dict(id=rid, mode=md, cur=m, page_size=P) for rid, m, (_, P, md) in zip(rids, mems, specs)]
    mems[0][2 * 4096] ^= 1
    mems[0][5 * 4096 + 3] ^= 1
    o.mark_pages(rids[0], [2, 6])                          # page 5 changed but unmarked; 6 marked, unchanged
    mems[2][4096] ^= 1                                      # compare region: found by content
    st, img, rep = o.checkpoint_gather()
    assert bytes(img) == imgfmt.build_image(regions, [[2, 6], [], [1]])
    z = [oracle_mod.aligned_empty(nb) for nb, _, _ in specs]
    o2 = oracle_mod.Oracle()
    for zz, (nb, P, md) in zip(z, specs):
        zz[:] = 0
        o2.register(zz, P, md)
    assert o2.restore_scatter(img0)[0] == 0 and o2.restore_scatter(img)[0] == 0
    want0 = mems[0].copy()
    assert np.array_equal(z[1], mems[1]) and np.array_equal(z[2], mems[2])
    # page 5's unmarked change is (by definition) not in the images
    assert not np.array_equal(z[0], want0)
    assert np.array_equal(z[0][:5 * 4096], want0[:5 * 4096]) and np.array_equal(z[0][6 * 4096:], want0[6 * 4096:])
