"""CPU checks of tests/fullparity.py (the region-by-region whole-image checker
used at full footprints): on an image built by ONE multi-region oracle
context it passes and covers every byte; any single flipped byte (header,
table, payload, ids, hashes, padding) or a wrong region id fails it."""
import numpy as np
import pytest

import synth
from tests import fullparity

KiB = 1 << 10
SPECS = [(3 * 64 * KiB + 1234, 64 * KiB, 1), (5 * 4 * KiB + 17, 4 * KiB, 0), (40 * 4 * KiB, 4 * KiB, 1),
         (2 * 64 * KiB, 64 * KiB, 0)]


def _image(oracle_mod, S, d, full=False):
    o = oracle_mod.Oracle()
    mems, committed = [], []
    for r, (nb, P, mode) in enumerate(SPECS):
        m = oracle_mod.aligned_empty(nb)
        synth.fill_region(m, S, r)
        mems.append(m)
        o.register(m, P, mode)
    o.sync_shadow()
    committed = [m.copy() for m in mems]
    if not full:
        for r, (nb, P, mode) in enumerate(SPECS):
            synth.apply_writer(mems[r], P, synth.choose_dirty(S, 1, r, synth.n_pages(nb, P), d), S, 1, r)
    st, img, rep = o.checkpoint_gather(flags=1 if full else 0)
    assert st == 0
    return img, committed, rep


@pytest.mark.parametrize("d,full", [(0.3, False), (0.0, False), (1.0, False), (0.0, True)])
def test_regionwise_check_passes_and_covers_every_byte(oracle_mod, d, full):
    S = synth.seed(60)
    img, committed, rep = _image(oracle_mod, S, d, full)
    res = fullparity.regionwise_check(img, SPECS, [1, 2, 3, 4], lambda r: committed[r].copy(), S, 1, d, full=full,
                                      threads=3)
    assert res["ok"] and res["checked_bytes"] == img.nbytes == rep["image_bytes"]


def test_regionwise_check_catches_any_flipped_byte(oracle_mod):
    S = synth.seed(61)
    img, committed, _ = _image(oracle_mod, S, 0.4)
    rng = np.random.default_rng(0)
    positions = sorted(set(rng.choice(img.nbytes, 60, replace=False).tolist()) | {0, 20, 64, 100, img.nbytes - 1})
    for pos in positions:
        bad = img.copy()
        bad[pos] ^= 0x01
        with pytest.raises(AssertionError):
            fullparity.regionwise_check(bad, SPECS, [1, 2, 3, 4], lambda r: committed[r].copy(), S, 1, 0.4, threads=2)
    with pytest.raises(AssertionError):
        fullparity.regionwise_check(img, SPECS, [1, 2, 3, 5], lambda r: committed[r].copy(), S, 1, 0.4)
