"""Oracle unit codec and compressed images (DESIGN.md
readings Z2-Z3: per 4 KiB unit, greedy LZ77 + one fixed-Huffman DEFLATE block,
RFC 1951) pinned to:
  * zlib's own inflater (raw DEFLATE, wbits = -15): every non-raw encoding
    inflates to exactly its unit and ends exactly at its last byte;
  * closed-form sizes worked out by hand from RFC 1951's code lengths
    (constant fp64 / fp32 vectors, zero, random, the literal-only bound and
    the one-match boundary at 4095 / 4096 bytes);
  * an independent plain-Python restatement (tests/imgfmt.py) byte-identical
    on structured units, whole images byte-identical to its builder;
  * every malformed-stream class rejected; restore of a compressed image ==
    restore of the plain one."""
import struct
import zlib

import numpy as np
import pytest

import synth
from tests import imgfmt

U = 4096


def inflate(enc: bytes) -> bytes:
    d = zlib.decompressobj(-15)
    out = d.decompress(enc)
    assert d.eof and d.unused_data == b"", "stream must end exactly at its last byte"
    return out


def structured_units(n, seed):
    """Units shaped like checkpoint data: fp64 / fp32 fields (constant, smooth,
    random), zero spans, small-integer arrays, byte ramps."""
    rng = np.random.default_rng(seed)
    out = []
    for t in range(n):
        kind = t % 7
        if kind == 0:
            u = np.sin(np.arange(512) * rng.uniform(0.001, 0.1)).astype("<f8")
        elif kind == 1:
            u = np.full(1024, rng.uniform(-9, 9), dtype="<f4")
        elif kind == 2:
            u = np.round(np.cumsum(rng.normal(size=512)), 2).astype("<f8")
        elif kind == 3:
            u = rng.integers(0, 8, 1024).astype("<u4")
        elif kind == 4:
            u = np.zeros(4096, np.uint8)
            for _ in range(int(rng.integers(1, 6))):      # constant byte spans in zeros
                a = int(rng.integers(0, 4096))
                u[a:a + int(rng.integers(1, 600))] = int(rng.integers(1, 256))
        elif kind == 5:
            u = (np.arange(4096) * int(rng.integers(1, 7)) % 251).astype(np.uint8)
        else:
            u = np.concatenate([rng.random(512, dtype=np.float32), np.full(512, 0.25, np.float32)]).astype("<f4")
        out.append(np.asarray(u).view(np.uint8).tobytes()[:U].ljust(U, b"\0"))
    return out


def test_zero_unit_encodes_to_nothing(oracle_mod):
    assert oracle_mod.z_encode(bytes(U)) == b""
    assert oracle_mod.z_decode(b"") == bytes(U)


def test_constant_fp64_closed_form(oracle_mod):
    """pi as fp64 (8 distinct bytes 18 2D 44 54 FB 21 09 40): 8 literals (one of
    them, 0xFB, a 9-bit code), then matches at distance 8 (code 5 + 1 extra
    bit): 15 x 258 (code 285, 8 bits) and one 218 (code 283, 8 bits + 5 extra).
    Bits: 3 + (7*8 + 9) + 15*(8 + 6) + (13 + 6) + 7 (end of block) = 304 = 38 bytes."""
    u = np.full(512, np.pi, dtype="<f8").tobytes()
    enc = oracle_mod.z_encode(u)
    assert len(enc) == 38
    assert imgfmt.z_tokens(u)[:9] == [("lit", b) for b in u[:8]] + [("match", 258, 8)]
    assert inflate(enc) == u and oracle_mod.z_decode(enc) == u


def test_constant_fp32_closed_form(oracle_mod):
    """1.5f = 00 00 C0 3F: 4 literals (0xC0 a 9-bit code), 15 x 258 at distance 4
    (code 3, no extra bits) and one 222 (code 283): 3 + 33 + 15*13 + 18 + 7 = 256
    bits = 32 bytes."""
    u = np.full(1024, 1.5, dtype="<f4").tobytes()
    enc = oracle_mod.z_encode(u)
    assert len(enc) == 32
    assert inflate(enc) == u and oracle_mod.z_decode(enc) == u


def test_random_unit_stays_raw(oracle_mod):
    u = np.random.default_rng(3).integers(0, 256, U, dtype=np.uint8).tobytes()
    assert oracle_mod.z_encode(u) == u


def test_raw_boundary(oracle_mod):
    """Bytes < 144 (8-bit literal codes) with no repeated 4-byte window: 3 + 4096*8
    + 7 = 32778 bits -> 4098 bytes -> raw.  Plant one 4-byte repeat at distance
    <= 4 (length code 258: 7 bits, distance code 5 bits, no extra): 4092
    literals -> 3 + 32736 + 12 + 7 = 32758 bits = 4095 bytes, encoded.  At a
    distance in 2049..4096 (10 extra bits): 32768 bits = 4096 bytes -> raw."""
    for seed in range(11, 60):
        rng = np.random.default_rng(seed)
        b = rng.integers(0, 144, U, dtype=np.uint8)
        if not all(t[0] == "lit" for t in imgfmt.z_tokens(b.tobytes())):
            continue
        planted = []
        for d in (3, 3000):
            c = b.copy()
            for i in range(4):                       # byte by byte: the copy may overlap (d < 4)
                c[3500 + i] = c[3500 + i - d]
            planted.append(c)
        if all([t for t in imgfmt.z_tokens(c.tobytes()) if t[0] == "match"] == [("match", 4, d)]
               for c, d in zip(planted, (3, 3000))):
            break
    else:
        pytest.fail("no seed gives the premise")
    assert oracle_mod.z_encode(b.tobytes()) == b.tobytes()
    for c, size in zip(planted, (4095, 4096)):
        enc = oracle_mod.z_encode(c.tobytes())
        assert len(enc) == size
        if size < U:
            assert inflate(enc) == c.tobytes()


def test_restatement_and_zlib_round_trip(oracle_mod):
    for t, u in enumerate(structured_units(140, 5)):
        enc = oracle_mod.z_encode(u)
        assert enc == imgfmt.z_encode_unit(u), t
        assert oracle_mod.z_decode(enc) == u, t
        if 0 < len(enc) < U:
            assert inflate(enc) == u, t


def test_decode_rejects_malformed(oracle_mod):
    u = np.full(512, np.pi, dtype="<f8").tobytes()
    enc = bytearray(oracle_mod.z_encode(u))
    assert oracle_mod.z_decode(bytes(enc)) == u
    assert oracle_mod.z_decode(bytes(enc[:-1])) is None            # truncated
    assert oracle_mod.z_decode(bytes(enc) + b"\0") is None         # a byte after the end of block
    b = bytearray(enc)
    b[0] ^= 1                                                       # BFINAL = 0
    assert oracle_mod.z_decode(bytes(b)) is None
    b = bytearray(enc)
    b[0] ^= 6                                                       # BTYPE = 10 (dynamic): not this codec
    assert oracle_mod.z_decode(bytes(b)) is None
    # 304 bits: the last byte holds 0 padding bits... use a stream with padding
    u2 = np.full(1024, 1.5, dtype="<f4").tobytes()[:-1] + b"\x07"
    e2 = bytearray(oracle_mod.z_encode(u2))
    nbits = None
    for pad in range(1, 8):                                         # find a set-able padding bit
        b = bytearray(e2)
        b[-1] |= 0x80 >> (pad - 1)
        if b != e2 and zlib.decompressobj(-15).decompress(bytes(b)) == u2:
            nbits = pad
            assert oracle_mod.z_decode(bytes(b)) is None            # nonzero padding
            break
    assert nbits is not None
    # hand-built streams: a match before any output; an early end of block;
    # one literal too many
    def stream(bits):
        bits = bits + [0] * (-len(bits) % 8)
        return bytes(sum(v << i for i, v in enumerate(bits[k:k + 8])) for k in range(0, len(bits), 8))
    hdr = [1, 1, 0]
    eob = [0] * 7
    match3_d1 = [0, 0, 0, 0, 0, 0, 1] + [0, 0, 0, 0, 0]            # length code 257 (3), distance code 0 (1)
    assert oracle_mod.z_decode(stream(hdr + match3_d1 + eob)) is None
    lit0 = [0, 0, 1, 1, 0, 0, 0, 0]                                  # literal 0: code 00110000
    assert oracle_mod.z_decode(stream(hdr + lit0 + eob)) is None    # 1 byte, not 4096
    body = lit0 + ([1, 1, 0, 0, 0, 1, 0, 1] + [0, 0, 0, 0, 0]) * 15 + [1, 1, 0, 0, 0, 0, 1, 1] + [0, 1, 1, 1, 1] + [0] * 5
    # lit 0 + 15 x 258 + a 225-length match (code 283: base 195, extra 30 = 11110b, LSB first) at
    # distance 1 = 4096 bytes
    ok = stream(hdr + body + eob)
    assert inflate(ok) == bytes(U) and oracle_mod.z_decode(ok) == bytes(U)
    assert oracle_mod.z_decode(stream(hdr + body + lit0 + eob)) is None   # 4097 bytes


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
    # a size larger than 4096, with CRCs recomputed
    u = next(i for i, cs in enumerate(p["zsizes"]) if 0 < cs < 4096)
    b2 = bytearray(img.tobytes())
    struct.pack_into("<H", b2, zoff + 2 * u, 4097)
    assert fresh().restore_scatter(refresh_crcs(b2))[0] == oracle_mod.E_CORRUPT
    # sizes consistent, CRCs fine, but a unit's stream damaged (the CRCs cover
    # only the metadata): flip BFINAL of its first byte
    coff = p["poff"] + sum(p["zsizes"][:u])
    b3 = bytearray(img.tobytes())
    b3[coff] ^= 1
    assert fresh().restore_scatter(np.frombuffer(bytes(b3), dtype=np.uint8))[0] == oracle_mod.E_CORRUPT
