"""Oracle unit codec and compressed images (DESIGN.md
readings Z1-Z2) pinned to: hand-written encodings of small patterns, closed-
form sizes (zero / constant fp32 / constant fp64 / ramp / random / the paper's
"50% random" vector), round trips, an independent numpy
restatement in tests/imgfmt.py (byte-identical images), and restore of a
compressed image == restore of the plain one."""
import struct

import numpy as np
import pytest

import synth
from tests import imgfmt

U = 4096


def words(ws):
    return np.asarray(ws, dtype="<u4").tobytes()


def test_zero_unit_encodes_to_nothing(oracle_mod):
    assert oracle_mod.z_encode(bytes(U)) == b""
    assert oracle_mod.z_decode(b"") == bytes(U)


def test_hand_encoding(oracle_mod):
    w = [0] * 1024
    w[1] = 7            # literal (pred 0)
    w[3] = 7            # predicted by w[1]
    w[5] = 7
    w[10] = 0xDEADBEEF  # literal
    w[12] = 5           # literal (pred w[10])
    enc = oracle_mod.z_encode(words(w))
    # by hand: odd class 0,7,7,7,0,... -> literals at 1 and 7 (w[7] = 0 != w[5] = 7);
    # even class ..., 0, 0xDEADBEEF, 5, 0, ... -> literals at 10, 12 and 14 (0 != 5)
    lits = [1, 7, 10, 12, 14]
    bitmap = bytearray(128)
    for j in lits:
        bitmap[j // 8] |= 1 << (j % 8)
    want = bytes(bitmap) + words([w[j] for j in lits])
    assert enc == want and len(enc) == 128 + 4 * 5
    assert oracle_mod.z_decode(enc) == words(w)


@pytest.mark.parametrize("kind,size", [
    ("const_f32", 128 + 8), ("const_f64", 128 + 8), ("ramp", U), ("random", U),
    ("half_random", 128 + 4 * (512 + 2)), ("sparse", 128 + 4 * 128)])
def test_closed_form_sizes(oracle_mod, kind, size):
    rng = np.random.default_rng(1)
    if kind == "const_f32":
        u = np.full(1024, 1.5, dtype="<f4").tobytes()
    elif kind == "const_f64":
        u = np.full(512, 3.141592653589793, dtype="<f8").tobytes()
    elif kind == "ramp":
        u = np.arange(1024, dtype="<u4").tobytes()            # w0 = 0 predicted, the rest literal
    elif kind == "random":
        u = rng.integers(1, 2**32, 1024, dtype=np.uint64).astype("<u4").tobytes()
    elif kind == "half_random":                               # PAPER.md:907-912 "only half ... randomly"
        r = rng.random(512, dtype=np.float32) + 1
        u = np.concatenate([r, np.full(512, 0.25, np.float32)]).astype("<f4").tobytes()
    else:   # 64 scattered nonzero words in zeros: each is a literal, and so is the 0 two words later
        w = np.zeros(1024, dtype="<u4")
        w[np.arange(0, 1024, 16)] = rng.integers(1, 2**32, 64, dtype=np.uint64).astype(np.uint32)
        u = w.tobytes()
    enc = oracle_mod.z_encode(u)
    assert len(enc) == size
    assert enc == imgfmt.z_encode_unit(u)
    assert oracle_mod.z_decode(enc) == u


def test_raw_threshold(oracle_mod):
    """128 + 4n < 4096 <=> n <= 991: n = 991 encodes, n = 992 goes raw."""
    for n, size in ((991, 128 + 4 * 991), (992, U)):
        w = np.zeros(1024, dtype="<u4")
        w[:n - 2] = np.arange(1, n - 1)   # n-2 distinct nonzero literals, then 2 mispredicted zeros
        enc = oracle_mod.z_encode(w.tobytes())
        assert len(enc) == size
        assert oracle_mod.z_decode(enc) == w.tobytes()


def test_round_trip_structured(oracle_mod):
    rng = np.random.default_rng(2)
    for t in range(200):
        w = np.zeros(1024, dtype=np.uint32)
        for _ in range(int(rng.integers(0, 6))):              # runs of constants / randoms / ramps
            a = int(rng.integers(0, 1024))
            b = int(rng.integers(a, 1025))
            k = int(rng.integers(0, 3))
            w[a:b] = [int(rng.integers(0, 2**32)), 0, 0][k] if k == 0 else (
                rng.integers(0, 2**32, b - a, dtype=np.uint64).astype(np.uint32) if k == 1 else np.arange(a, b))
        u = w.astype("<u4").tobytes()
        enc = oracle_mod.z_encode(u)
        assert enc == imgfmt.z_encode_unit(u), t
        assert oracle_mod.z_decode(enc) == u, t


def test_decode_rejects_inconsistent(oracle_mod):
    enc = bytearray(oracle_mod.z_encode(words([0, 9] * 512)))   # 1 literal (w[1]): 132 bytes
    assert len(enc) == 132
    bad = bytearray(enc)
    bad[0] |= 4                                               # a second bitmap bit, no second literal
    assert oracle_mod.z_decode(bytes(bad)) is None
    assert oracle_mod.z_decode(bytes(enc[:130])) is None      # size not 0 / 4096 / 128+4n
    assert oracle_mod.z_decode(bytes(128)) is None            # 128 = 128 + 4*0 is not a valid size


SPECS = [(5 * 4096 + 333, 4096, 0), (3 * 65536, 65536, 1), (4096 * 7, 4096, 1), (8192, 4096, 0)]


def make_ctx(oracle_mod, specs, S, half_const=True):
    o = oracle_mod.Oracle()
    mems, rids = [], []
    for r, (nb, P, mode) in enumerate(specs):
        m = oracle_mod.aligned_empty(nb)
        synth.fill_region(m, S, r)
        if half_const:                                        # the paper's 50%-random shape
            m[nb // 2:] = 0
        mems.append(m)
        rids.append(o.register(m, P, mode))
    return o, mems, rids


@pytest.mark.parametrize("full", [False, True])
def test_compressed_image_matches_builder(oracle_mod, full):
    S = synth.seed(80)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    regions = [dict(id=rid, mode=md, cur=m, page_size=P) for rid, m, (_, P, md) in zip(rids, mems, SPECS)]
    every = [list(range(synth.n_pages(nb, P))) for nb, P, _ in SPECS]
    st, img0, rep0 = o.checkpoint_gather(flags=oracle_mod.COMPRESS)
    assert st == 0
    assert bytes(img0) == imgfmt.build_image(regions, every, compress=True)
    plain = imgfmt.build_image(regions, every)
    assert len(img0) < len(plain)
    for r, (nb, P, _) in enumerate(SPECS):
        synth.apply_writer(mems[r], P, synth.choose_dirty(S, 1, r, synth.n_pages(nb, P), 0.5), S, 1, r)
    listed = [sorted(set(synth.choose_dirty(S, 1, r, synth.n_pages(nb, P), 0.5).tolist()))
              for r, (nb, P, _) in enumerate(SPECS)]
    flags = oracle_mod.COMPRESS | (oracle_mod.FULL if full else 0)
    st, img, rep = o.checkpoint_gather(flags=flags)
    assert st == 0
    assert bytes(img) == imgfmt.build_image(regions, every if full else listed, full=full, compress=True)
    p = imgfmt.parse_image(img)
    assert p["flags"] & 4 and sum(p["zsizes"]) <= p["payload_bytes"] < sum(p["zsizes"]) + 4096


def test_compressed_restore_equals_plain(oracle_mod):
    S = synth.seed(81)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    imgs, states = [], []
    for epoch in range(4):
        if epoch:
            for r, (nb, P, _) in enumerate(SPECS):
                synth.apply_writer(mems[r], P, synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), 0.3),
                                   S, epoch, r)
        st, img, _ = o.checkpoint_gather(flags=oracle_mod.COMPRESS if epoch % 2 == 0 else 0)
        assert st == 0
        imgs.append(img)
        states.append([m.copy() for m in mems])
    o2 = oracle_mod.Oracle()
    zs = []
    for nb, P, mode in SPECS:
        z = oracle_mod.aligned_empty(nb)
        z[:] = 0
        zs.append(z)
        o2.register(z, P, mode)
    for k, img in enumerate(imgs):
        st, rep = o2.restore_scatter(img, oracle_mod.VERIFY)
        assert st == 0, k
        for z, want in zip(zs, states[k]):
            assert np.array_equal(z, want), k
    assert o2.sync_shadow() == 0
    # lazy restore of a compressed image
    o3 = oracle_mod.Oracle()
    z3 = []
    for nb, P, mode in SPECS:
        z = oracle_mod.aligned_empty(nb)
        z[:] = 0
        z3.append(z)
        o3.register(z, P, mode)
    assert o3.restore_begin(imgs[0]) == 0
    assert o3.restore_fetch(2, 1)[0] == 0
    assert np.array_equal(z3[1][65536:131072], states[0][1][65536:131072])
    assert o3.restore_end()[0] == 0
    for z, want in zip(z3, states[0]):
        assert np.array_equal(z, want)


def test_compressed_corruption(oracle_mod):
    S = synth.seed(82)
    o, mems, rids = make_ctx(oracle_mod, SPECS, S)
    st, img, _ = o.checkpoint_gather(flags=oracle_mod.COMPRESS)
    p = imgfmt.parse_image(img)
    zoff = p["ids_off"] + imgfmt.round_up(4 * p["K"], 8) + 8 * p["K"]

    def fresh():
        o2 = oracle_mod.Oracle()
        for nb, P, mode in SPECS:
            z = oracle_mod.aligned_empty(nb)
            z[:] = 0
            o2.register(z, P, mode)
        return o2

    def refresh_crcs(b):
        b = bytearray(b)
        tab = bytes(b[64:64 + 48 * p["R"]])
        tail = bytes(b[p["ids_off"]:p["image_bytes"]])
        import zlib
        struct.pack_into("<I", b, 56, zlib.crc32(tab + tail))
        struct.pack_into("<I", b, 60, zlib.crc32(bytes(b[:60])))
        return np.frombuffer(bytes(b), dtype=np.uint8)

    assert fresh().restore_scatter(img)[0] == 0
    bad = img.copy()
    bad[zoff] ^= 1                                            # CRC catches a changed size
    assert fresh().restore_scatter(bad)[0] == oracle_mod.E_CORRUPT
    # a size that is not 0 / 4096 / 128+4n, with CRCs recomputed
    u = next(i for i, cs in enumerate(p["zsizes"]) if 132 <= cs < 4096)
    b2 = bytearray(img.tobytes())
    struct.pack_into("<H", b2, zoff + 2 * u, p["zsizes"][u] + 2)
    assert fresh().restore_scatter(refresh_crcs(b2))[0] == oracle_mod.E_CORRUPT
    # sizes consistent in total but a bitmap that disagrees with its size
    poff = p["poff"]
    coff = poff + sum(p["zsizes"][:u])
    b3 = bytearray(img.tobytes())
    bm = np.frombuffer(bytes(b3[coff:coff + 128]), dtype=np.uint8)
    j = int(np.flatnonzero(np.unpackbits(bm, bitorder="little") == 0)[0])
    b3[coff + j // 8] |= 1 << (j % 8)
    assert fresh().restore_scatter(np.frombuffer(bytes(b3), dtype=np.uint8))[0] == oracle_mod.E_CORRUPT
