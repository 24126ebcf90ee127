"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NONE of the method's arithmetic (no detection,
hashing, compaction or image logic): it only says which bytes a region holds
and which pages an "application epoch" rewrites.

Recipe (SURVEY.md sec. 8(d) "Common input rules"):

* seed           S = 0x18080117 + config_index
* content        u64 word j of region r = splitmix64(S ^ (r << 40) ^ j)
                 (uniform random words, standing in for the paper's random
                 FP32 payload); a trailing partial word takes
                 the low bytes of its word (little-endian).
* dirty choice   exactly K_r = floor(d * n_r + 0.5) pages of region r: those
                 with the smallest key splitmix64((S+1) ^ (epoch << 56) ^ (r << 40) ^ i)
                 (ties broken by page index).
* writer         every u64 word of a chosen page (logical bytes only) is XORed
                 with mask = splitmix64((S+2) ^ (epoch << 56) ^ (r << 40) ^ i) | 1;
                 the mask is odd, so every word -- and the page's first byte of
                 every word -- changes: the dirty set equals the written set.
                 The "touch" writer XORs only the page's last word.

The CUDA path has its own implementation of the same counter-based generator
(paper_1808_00117_b200/csrc/synth.cu); tests check the two agree.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0x18080117
M64 = (1 << 64) - 1


def seed(config_index: int) -> int:
    return SEED_BASE + config_index


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser over a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def region_content(S: int, r: int, nbytes: int, word_offset: int = 0) -> np.ndarray:
    """Bytes of region r (or of the slice starting at u64 word `word_offset`)."""
    nw = (nbytes + 7) // 8
    j = np.arange(word_offset, word_offset + nw, dtype=np.uint64)
    w = splitmix64_np(np.uint64(S) ^ (np.uint64(r) << np.uint64(40)) ^ j)
    return w.view(np.uint8)[:nbytes].copy()


def fill_region(buf: np.ndarray, S: int, r: int) -> None:
    buf[:] = region_content(S, r, buf.nbytes)


def n_pages(nbytes: int, page_size: int) -> int:
    return -(-nbytes // page_size)


def dirty_count(d: float, n: int) -> int:
    return int(np.floor(d * n + 0.5))


def choose_dirty(S: int, epoch: int, r: int, n: int, d: float) -> np.ndarray:
    """Ascending page indices of the K_r pages rewritten at `epoch`."""
    k = dirty_count(d, n)
    if k <= 0:
        return np.zeros(0, dtype=np.int64)
    i = np.arange(n, dtype=np.uint64)
    key = splitmix64_np(np.uint64(S + 1) ^ (np.uint64(epoch) << np.uint64(56)) ^ (np.uint64(r) << np.uint64(40)) ^ i)
    order = np.lexsort((np.arange(n), key))
    return np.sort(order[:k]).astype(np.int64)


def page_mask(S: int, epoch: int, r: int, i: np.ndarray) -> np.ndarray:
    i = np.asarray(i, dtype=np.uint64)
    return splitmix64_np(np.uint64(S + 2) ^ (np.uint64(epoch) << np.uint64(56)) ^ (np.uint64(r) << np.uint64(40)) ^ i) | np.uint64(1)


def apply_writer(buf: np.ndarray, page_size: int, pages: np.ndarray, S: int, epoch: int, r: int,
                 touch: bool = False) -> None:
    """XOR every u64 word (or only the last word, touch=True) of each chosen
    page's logical bytes with that page's odd mask, in place."""
    nbytes = buf.nbytes
    masks = page_mask(S, epoch, r, pages)
    for i, m in zip(np.asarray(pages).tolist(), masks.tolist()):
        lo = i * page_size
        hi = min(lo + page_size, nbytes)
        mb = np.frombuffer(np.uint64(m).tobytes(), dtype=np.uint8)
        if touch:
            # last (possibly partial) word of the page
            wlo = lo + ((hi - lo - 1) // 8) * 8
            seg = buf[wlo:hi]
            seg ^= mb[:hi - wlo]
            continue
        seg = buf[lo:hi]
        full = (hi - lo) // 8 * 8
        if full:
            seg[:full].view(np.uint64)[:] ^= np.uint64(m)
        if hi - lo > full:
            seg[full:] ^= mb[:hi - lo - full]


# --------------------------------------------------------------------------
# Workload shapes (BASELINE.json configs)
# --------------------------------------------------------------------------
KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30


def c3_region_sizes(replicas: int = 20):
    """Rodinia-UVM-style footprint (Table 1 shapes):
    LUD 2048^2 fp32; Hotspot3D 512x512x8 fp32 x3; Gaussian 8192^2 fp32 x2 +
    8192-float b; LavaMD-like 100 MiB x2, 25 MiB, 40 MiB."""
    one = [16 * MiB, 8 * MiB, 8 * MiB, 8 * MiB, 256 * MiB, 256 * MiB, 32 * KiB,
           100 * MiB, 100 * MiB, 25 * MiB, 40 * MiB]
    # 11 regions per replica, 817.03 MiB; x20 replicas = 15.96 GiB.
    return one * replicas


def c4_region_sizes(S: int, n_box: int = 4096, levels: int = 7):
    """HPGMG-FV-style: 7 levels x 8 vectors (7 GiB / 8^l) + n_box regions
    log-uniform in [12 KiB, 128 KiB] rounded up to 256 B."""
    big = []
    for lvl in range(levels):
        big += [(7 * GiB) >> (3 * lvl)] * 8
    u = splitmix64_np(np.uint64(S + 3) ^ np.arange(n_box, dtype=np.uint64)).astype(np.float64) / 2.0**64
    lo, hi = np.log(12 * KiB), np.log(128 * KiB)
    small = np.exp(lo + u * (hi - lo))
    small = (np.ceil(small / 256) * 256).astype(np.int64).tolist()
    return big, small


# --------------------------------------------------------------------------
# Structured content (bench --content hpgmg; compressed-image measurements)
HPGMG_KINDS = ("smooth u", "smooth f", "alpha", "beta_x", "beta_y", "beta_z", "Dinv", "temporary")


def hpgmg_box_kinds(nbox: int, r: int) -> np.ndarray:
    """Kind (index into HPGMG_KINDS) of every 32 KiB box of fp64 values of
    region r: HPGMG-FV keeps 8 vectors per level -- two smooth fields, four
    constant coefficients, the constant diagonal inverse, one cleared
    temporary (PAPER.md:704-751 describes the application; the kinds are a
    proposal, the paper prints no data).  Box b of region r has kind
    (b + r) % 8, so every region holds every kind."""
    return ((np.arange(nbox) + r) % 8).astype(np.int64)


def hpgmg_fill(buf: np.ndarray, r: int) -> None:
    """Host version of bench.hpgmg_fill_device (values agree up to the last
    bits of sin(); used for the CPU baseline's sample only)."""
    n = buf.nbytes // 8
    nbox = n // 4096
    if nbox == 0:
        return
    F = buf[:nbox * 4096 * 8].view(np.float64).reshape(nbox, 4096)
    kinds = hpgmg_box_kinds(nbox, r)
    x = np.arange(4096, dtype=np.float64)
    for b in range(nbox):
        k = kinds[b]
        if k <= 1:
            F[b] = np.sin(x * (0.001 + 0.0005 * (b % 7)) + b) * (1 + (b % 3))
        else:
            F[b] = {2: 1.0, 3: 1.0, 4: 1.0, 5: 1.0, 6: 1.0 / 6.0, 7: 0.0}[int(k)]
        F[b, :256] = 0
        F[b, -256:] = 0
