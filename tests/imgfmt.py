"""Independent image-format v1 builder/parser for tests,
written with library routines only: struct, zlib.crc32 and
xxhash.xxh3_64_intdigest.  It pins the oracle's image assembly and is reused by
the GPU parity tests to decode images.  Imports neither oracle/ nor the
product package.

Layout: header(64) | table(48R) | zero pad to payload_offset | payload |
        ids (u32, padded to 8 B) | hashes (u64, if any hash-mode region)
"""
from __future__ import annotations

import struct
import zlib

import numpy as np
import xxhash

HDR = struct.Struct("<4sIIIQQQQQII")  # 64 bytes
ENTRY = struct.Struct("<IIQQQQQ")      # 48 bytes
assert HDR.size == 64 and ENTRY.size == 48


def round_up(x, a):
    return (x + a - 1) // a * a


def slot_bytes(cur: np.ndarray, page_size: int, i: int) -> bytes:
    seg = cur[i * page_size:(i + 1) * page_size].tobytes()
    return seg + b"\0" * (page_size - len(seg))


# --- unit codec, reading Z3, restated in plain Python ----------
# RFC 1951 sec. 3.2.5 length / distance code tables, derived here from their
# ranges instead of copied: lengths 3..258 -> codes 257..285; distances
# 1..32768 -> codes 0..29.
def _len_codes():
    out, base, code = {}, 3, 257
    for extra, n in [(0, 8), (1, 4), (2, 4), (3, 4), (4, 4), (5, 4)]:
        for _ in range(n):
            for L in range(base, base + (1 << extra)):
                out[L] = (code, extra, L - base)
            base += 1 << extra
            code += 1
    out[258] = (285, 0, 0)          # 258 has its own code (RFC 1951: 284 covers 227-257)
    return out


def _dist_codes():
    out, base = {}, 1
    for code in range(30):
        extra = max(0, code // 2 - 1)
        for d in range(base, base + (1 << extra)):
            out[d] = (code, extra, d - base)
        base += 1 << extra
    return out


_LEN, _DIST = _len_codes(), _dist_codes()


def _litlen_code(s):
    """(code, nbits) of the fixed literal/length code (RFC 1951 sec. 3.2.6)."""
    if s <= 143:
        return 0b00110000 + s, 8
    if s <= 255:
        return 0b110010000 + s - 144, 9
    if s <= 279:
        return s - 256, 7
    return 0b11000000 + s - 280, 8


def z_tokens(unit: bytes):
    """The greedy parse of reading Z3: list of ("lit", byte) / ("match", len, dist)."""
    u = bytes(unit)
    head = {}
    cand = []
    for p in range(4096):
        if p + 4 <= 4096:
            h = ((int.from_bytes(u[p:p + 4], "little") * 2654435761) & 0xFFFFFFFF) >> 20
            cand.append(head.get(h))
            head[h] = p
        else:
            cand.append(None)
    toks, p = [], 0
    while p < 4096:
        L = 0
        q = cand[p]
        if q is not None:
            while L < min(258, 4096 - p) and u[q + L] == u[p + L]:
                L += 1
        if L >= 4:
            toks.append(("match", L, p - q))
            p += L
        else:
            toks.append(("lit", u[p]))
            p += 1
    return toks


def z_encode_unit(unit: bytes) -> bytes:
    """Reading Z3: b"" for a zero unit; else the fixed-Huffman DEFLATE stream
    of z_tokens() if shorter than 4096 bytes; else the raw unit."""
    u = bytes(unit)
    if not any(u):
        return b""
    bits = [1, 1, 0]                          # BFINAL = 1, BTYPE = 01 (LSB first)

    def code(c, n):                           # Huffman codes: most significant bit first
        bits.extend((c >> (n - 1 - i)) & 1 for i in range(n))

    def extra(v, n):                          # extra bits: least significant bit first
        bits.extend((v >> i) & 1 for i in range(n))

    for t in z_tokens(u):
        if t[0] == "lit":
            code(*_litlen_code(t[1]))
        else:
            lc, le, lv = _LEN[t[1]]
            code(*_litlen_code(lc))
            extra(lv, le)
            dc, de, dv = _DIST[t[2]]
            code(dc, 5)
            extra(dv, de)
    code(*_litlen_code(256))
    nbytes = (len(bits) + 7) // 8
    if nbytes >= 4096:
        return u
    bits += [0] * (8 * nbytes - len(bits))
    return bytes(sum(b << i for i, b in enumerate(bits[8 * k:8 * k + 8])) for k in range(nbytes))


def z_decode_unit(enc: bytes) -> bytes:
    """Inverse for tests: zlib's own inflater (raw DEFLATE, wbits = -15); the
    stream must end exactly at its last byte."""
    if len(enc) == 0:
        return bytes(4096)
    if len(enc) == 4096:
        return bytes(enc)
    d = zlib.decompressobj(-15)
    out = d.decompress(bytes(enc))
    assert d.eof and d.unused_data == b"" and len(out) == 4096
    return out


def build_image(regions, listed, full=False, compress=False) -> bytes:
    """regions: list of dicts {id, mode, cur (np.uint8 array), page_size};
    listed: list (same order) of ascending page-index lists."""
    R = len(regions)
    K = sum(len(l) for l in listed)
    has_hashes = any(r["mode"] == 1 for r in regions)
    poff = round_up(64 + 48 * R, 4096)
    table, ids, hashes, payload = b"", b"", b"", []
    first = 0
    for r, l in zip(regions, listed):
        cur, P = r["cur"], r["page_size"]
        n = -(-cur.nbytes // P)
        table += ENTRY.pack(r["id"], r["mode"], cur.nbytes, P, n, len(l), first)
        first += len(l)
        for i in l:
            s = slot_bytes(cur, P, i)
            ids += struct.pack("<I", i)
            if has_hashes:
                hashes += struct.pack("<Q", xxhash.xxh3_64_intdigest(s) if r["mode"] == 1 else 0)
            payload.append(s)
    ids += b"\0" * (round_up(4 * K, 8) - 4 * K)
    pay = b"".join(payload)
    tail = ids + hashes
    if compress:
        units = [z_encode_unit(pay[u:u + 4096]) for u in range(0, len(pay), 4096)]
        zs = b"".join(struct.pack("<H", len(e)) for e in units)
        tail += zs + b"\0" * (round_up(len(zs), 8) - len(zs))
        pay = b"".join(units)
        pay += b"\0" * (round_up(len(pay), 4096) - len(pay))
    ids_off = poff + len(pay)
    total = ids_off + len(tail)
    flags = (1 if full else 0) | (2 if has_hashes else 0) | (4 if compress else 0)
    hdr0 = struct.pack("<4sIIIQQQQQI", b"CRUM", 1, flags, R, K, poff, len(pay), ids_off, total,
                       zlib.crc32(table + tail))
    hdr = hdr0 + struct.pack("<I", zlib.crc32(hdr0))
    out = hdr + table + b"\0" * (poff - 64 - len(table)) + pay + tail
    assert len(out) == total
    return out


def parse_image(img: bytes):
    img = bytes(img)
    magic, ver, flags, R, K, poff, paylen, ids_off, total, mcrc, hcrc = HDR.unpack_from(img, 0)
    table = [ENTRY.unpack_from(img, 64 + 48 * k) for k in range(R)]
    ids = list(struct.unpack_from(f"<{K}I", img, ids_off)) if K else []
    hashes = []
    if flags & 2 and K:
        hashes = list(struct.unpack_from(f"<{K}Q", img, ids_off + round_up(4 * K, 8)))
    zsizes = []
    if flags & 4:
        U = sum(e[5] * e[3] for e in table) // 4096
        zoff = ids_off + round_up(4 * K, 8) + (8 * K if flags & 2 else 0)
        zsizes = list(struct.unpack_from(f"<{U}H", img, zoff)) if U else []
    return dict(magic=magic, version=ver, flags=flags, R=R, K=K, poff=poff, payload_bytes=paylen,
                ids_off=ids_off, image_bytes=total, meta_crc=mcrc, header_crc=hcrc, table=table, ids=ids,
                hashes=hashes, zsizes=zsizes)


def meta_positions(img: bytes):
    """Byte positions covered by the two CRCs (header, table, ids, hashes)."""
    p = parse_image(img)
    return list(range(0, 64 + 48 * p["R"])) + list(range(p["ids_off"], p["image_bytes"]))
