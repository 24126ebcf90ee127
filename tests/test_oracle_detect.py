"""Oracle detect / sync / register pinned to brute force (Python bytes
equality per page) and to the paper's stated rules:
 - a new region starts with all pages dirty,
 - dirty pages are flushed then cleared at each CUDA call,
 - reading Q1: same-value writes are not dirty unless force-marked."""
import numpy as np
import pytest
import xxhash

import synth

MODES = [0, 1]


def brute_dirty(cur: np.ndarray, snap: np.ndarray, P: int) -> np.ndarray:
    n = -(-cur.nbytes // P)
    return np.array([cur[i * P:(i + 1) * P].tobytes() != snap[i * P:(i + 1) * P].tobytes()
                     for i in range(n)], dtype=np.uint8)


@pytest.mark.parametrize("mode", MODES)
def test_register_all_dirty_then_clean(oracle_mod, mode):
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(16 * P)
    synth.fill_region(mem, synth.seed(0), 0)
    rid = o.register(mem, P, mode)
    # SPEC.md:354 "create 16-page region -> 16 dirty bits"
    assert o.detect(rid).tolist() == [1] * 16
    assert o.force_bits(rid).tolist() == [1] * 16
    assert o.sync_shadow() == 16            # first sync returns N (reading Q3)
    assert o.sync_shadow() == 0             # idempotence
    assert o.detect(rid).sum() == 0


@pytest.mark.parametrize("mode", MODES)
def test_exhaustive_single_byte_flips(oracle_mod, mode):
    """Every single-byte flip of a 2 x 4 KiB region flags exactly its page."""
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(2 * P)
    synth.fill_region(mem, synth.seed(0), 1)
    rid = o.register(mem, P, mode)
    o.sync_shadow()
    step = 1 if mode == 0 else 7   # hash mode is slower per call; still covers every stripe/lane
    for pos in range(0, 2 * P, step):
        mem[pos] ^= 0x01
        f = o.detect(rid)
        assert f.tolist() == [int(pos < P), int(pos >= P)], pos
        mem[pos] ^= 0x01
    assert o.detect(rid).sum() == 0


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("P,nbytes", [(4096, 64 * 4096), (65536, 3 * 65536 + 1234), (4096, 4096 * 5 + 17)])
def test_random_writes_vs_brute_force(oracle_mod, mode, P, nbytes):
    rng = np.random.default_rng(P + nbytes + mode)
    o = oracle_mod.Oracle()
    mem = oracle_mod.aligned_empty(nbytes)
    synth.fill_region(mem, synth.seed(1), 2)
    rid = o.register(mem, P, mode)
    o.sync_shadow()
    for _ in range(5):
        snap = mem.copy()
        for _ in range(rng.integers(0, 12)):
            pos = int(rng.integers(0, nbytes))
            mem[pos] = rng.integers(0, 256)          # may be a same-value write
        want = brute_dirty(mem, snap, P)
        assert np.array_equal(o.detect(rid), want)
        assert o.sync_shadow() == int(want.sum())
        assert o.detect(rid).sum() == 0


def test_same_value_write_not_dirty_unless_marked(oracle_mod):
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(8 * P)
    mem[:] = 3
    rid = o.register(mem, P, 0)
    o.sync_shadow()
    mem[5 * P + 9] = 3                       # same value: not dirty (reading Q1)
    assert o.detect(rid).sum() == 0
    assert o.mark_dirty(rid, 5 * P + 9, 1) == 0
    assert o.detect(rid).tolist() == [0, 0, 0, 0, 0, 1, 0, 0]
    assert o.mark_dirty(rid, P - 1, 2) == 0  # straddles pages 0 and 1
    assert o.detect(rid).tolist() == [1, 1, 0, 0, 0, 1, 0, 0]
    assert o.mark_dirty(rid, 0, 0) == 0      # empty range: no page
    assert o.mark_dirty(rid, 8 * P, 1) == oracle_mod.E_RANGE
    assert o.mark_dirty(rid, 8 * P + 1, 0) == oracle_mod.E_RANGE
    assert o.mark_dirty(999, 0, 1) == oracle_mod.E_NOREGION
    assert o.sync_shadow() == 3


@pytest.mark.parametrize("d", [0.0, 0.1, 0.5, 1.0])
def test_dirty_set_equals_written_set_and_modes_agree(oracle_mod, d):
    P, n = 4096, 200
    S = synth.seed(1)
    sets = []
    for mode in MODES:
        o = oracle_mod.Oracle()
        mem = oracle_mod.aligned_empty(n * P - 100)   # partial last page
        synth.fill_region(mem, S, 0)
        rid = o.register(mem, P, mode)
        o.sync_shadow()
        pages = synth.choose_dirty(S, 1, 0, n, d)
        assert len(pages) == synth.dirty_count(d, n)
        synth.apply_writer(mem, P, pages, S, 1, 0)
        got = np.flatnonzero(o.detect(rid))
        assert np.array_equal(got, pages)
        sets.append(got)
        # touch writer: one word per page changes
        o.sync_shadow()
        pages2 = synth.choose_dirty(S, 2, 0, n, d)
        synth.apply_writer(mem, P, pages2, S, 2, 0, touch=True)
        assert np.array_equal(np.flatnonzero(o.detect(rid)), pages2)
    assert np.array_equal(sets[0], sets[1])


def test_hash_table_commit_matches_library(oracle_mod):
    """After sync, the hash-mode table holds XXH3 of each zero-padded slot."""
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(3 * P + 100)
    synth.fill_region(mem, synth.seed(2), 0)
    rid = o.register(mem, P, 1)
    o.sync_shadow()
    h = o.hashes(rid)
    for i in range(4):
        seg = mem[i * P:(i + 1) * P].tobytes()
        assert int(h[i]) == xxhash.xxh3_64_intdigest(seg + b"\0" * (P - len(seg)))
        assert o.page_hash(rid, i) == int(h[i])


def test_compare_mirror_commit(oracle_mod):
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(4 * P)
    synth.fill_region(mem, synth.seed(2), 1)
    rid = o.register(mem, P, 0)
    assert o.mirror(rid).sum() == 0          # initial snapshot is zeros (irrelevant under force)
    o.sync_shadow()
    assert np.array_equal(o.mirror(rid), mem)


def test_register_validation(oracle_mod):
    o = oracle_mod.Oracle()
    mem = oracle_mod.aligned_empty(1 << 20)
    p = mem.ctypes.data
    E = oracle_mod
    assert o.try_register(0, 4096, 4096) == E.E_INVAL               # null
    assert o.try_register(p, 0, 4096) == E.E_INVAL                  # bytes == 0
    assert o.try_register(p, 4096, 2048) == E.E_INVAL               # page < 4 KiB
    assert o.try_register(p, 4096, 4 << 20) == E.E_INVAL            # page > 2 MiB
    assert o.try_register(p, 4096, 12288) == E.E_INVAL              # not a power of two
    assert o.try_register(p + 8, 4096, 4096) == E.E_INVAL           # misaligned
    assert o.try_register(p, 4096, 4096, mode=7) == E.E_INVAL       # bad mode
    assert o.try_register(p, 65536, 4096) == 0
    assert o.try_register(p + 4096, 4096, 4096) == E.E_OVERLAP
    assert o.try_register(p + 65536, 4096, 4096) == 0               # adjacent is fine
    assert o.try_register(p + 65536 - 16, 32, 4096) == E.E_OVERLAP


def test_region_ids_monotonic_never_reused(oracle_mod):
    o = oracle_mod.Oracle()
    a = oracle_mod.aligned_empty(8192)
    b = oracle_mod.aligned_empty(8192)
    r1 = o.register(a, 4096)
    r2 = o.register(b, 4096)
    assert (r1, r2) == (1, 2)
    o.unregister(r1)
    assert o.register(a, 4096) == 3


def test_tracked_mode_dirty_is_exactly_the_marked_set(oracle_mod):
    """CRUM_MODE_TRACKED follows Alg. 1's write rule:
    a page is dirty iff marked since its last commit -- content changes that
    were not marked are NOT listed, marked pages are listed even if unchanged."""
    o = oracle_mod.Oracle()
    P = 4096
    mem = oracle_mod.aligned_empty(10 * P + 100)
    synth.fill_region(mem, synth.seed(3), 0)
    rid = o.register(mem, P, oracle_mod.MODE_TRACKED)
    assert o.detect(rid).tolist() == [1] * 11            # all pages start dirty
    assert o.sync_shadow() == 11 and o.sync_shadow() == 0
    mem[3 * P + 5] ^= 0xFF                                 # unmarked change: not dirty
    assert o.detect(rid).sum() == 0
    assert o.mark_pages(rid, [1, 7, 10]) == 0              # marked (7 and 10 unchanged, 10 partial)
    assert np.flatnonzero(o.detect(rid)).tolist() == [1, 7, 10]
    assert o.mark_pages(rid, [11]) == oracle_mod.E_RANGE
    assert o.mark_pages(999, [0]) == oracle_mod.E_NOREGION
    assert o.sync_shadow() == 3 and o.detect(rid).sum() == 0
    assert o.try_register(mem.ctypes.data, 4096, 4096, mode=3) == oracle_mod.E_INVAL
