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


def z_encode_unit(unit: bytes) -> bytes:
    """DESIGN.md readings Z1-Z2, restated with numpy: 1024 LE u32 words, word j
    predicted by word j-2 (0 for j < 2); literals = mispredicted words;
    0 literals -> b""; 128 + 4n < 4096 -> LSB-first bitmap + literals; else raw."""
    w = np.frombuffer(unit, dtype="<u4")
    pred = np.concatenate([np.zeros(2, dtype="<u4"), w[:-2]])
    lit = w != pred
    n = int(lit.sum())
    if n == 0:
        return b""
    if 128 + 4 * n >= 4096:
        return bytes(unit)
    return np.packbits(lit, bitorder="little").tobytes() + w[lit].astype("<u4").tobytes()


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
