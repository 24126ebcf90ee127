"""Oracle primitives pinned to library routines (not to themselves):
XXH3-64 -> python-xxhash (reading Q8), CRC-32 -> zlib (image format)."""
import zlib

import numpy as np
import pytest
import xxhash

LENGTHS = [241, 255, 256, 1023, 1024, 1025, 1088, 2047, 4095, 4096, 4097, 8192, 65536,
           65536 + 64, 131072, 2 << 20]


@pytest.mark.parametrize("n", LENGTHS)
def test_xxh3_random(oracle_mod, n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 256, n, dtype=np.uint8)
    assert oracle_mod.xxh3_64(a) == xxhash.xxh3_64_intdigest(a.tobytes())


@pytest.mark.parametrize("n", [4096, 65536, 2 << 20])
@pytest.mark.parametrize("fill", [0x00, 0xFF, 0x5A])
def test_xxh3_constant(oracle_mod, n, fill):
    a = np.full(n, fill, dtype=np.uint8)
    assert oracle_mod.xxh3_64(a) == xxhash.xxh3_64_intdigest(a.tobytes())


def test_xxh3_partial_tail_slots(oracle_mod):
    """Zero-padded slots of partial last pages (reading Q7)."""
    rng = np.random.default_rng(7)
    for P in (4096, 65536):
        for ln in (1, 17, 1000, P - 1):
            slot = np.zeros(P, dtype=np.uint8)
            slot[:ln] = rng.integers(0, 256, ln, dtype=np.uint8)
            assert oracle_mod.xxh3_64(slot) == xxhash.xxh3_64_intdigest(slot.tobytes())


def test_xxh3_every_stripe_position_matters(oracle_mod):
    """A flip in each 64-byte stripe (incl. the last stripe, secret offset 121,
    and the stripe before it) changes the hash and still matches the library."""
    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, 4096, dtype=np.uint8)
    h0 = oracle_mod.xxh3_64(a)
    for pos in range(0, 4096, 61):
        b = a.copy()
        b[pos] ^= 0x80
        h = oracle_mod.xxh3_64(b)
        assert h != h0
        assert h == xxhash.xxh3_64_intdigest(b.tobytes())


@pytest.mark.parametrize("n", [0, 1, 7, 60, 1000, 4096, 100003])
def test_crc32(oracle_mod, n):
    rng = np.random.default_rng(n + 11)
    a = rng.integers(0, 256, n, dtype=np.uint8)
    assert oracle_mod.crc32(a) == zlib.crc32(a.tobytes())
