"""ctypes wrapper over oracle/crum_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It never touches the CUDA
path (paper_1808_00117_b200/) and the CUDA path never touches it.

Region memory is a caller-owned numpy uint8 array (the oracle's stand-in for
the registered UVM region); the oracle keeps a pointer to it,
so this wrapper pins the array for the lifetime of the registration.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "crum_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_crum.so")
_lock = threading.Lock()
_lib = None

OK, E_INVAL, E_OVERLAP, E_NOREGION, E_RANGE, E_NOMEM, E_CAPACITY, E_CORRUPT, E_MISMATCH, E_BUSY = (
    0, -1, -2, -3, -4, -5, -6, -7, -8, -9)
MODE_COMPARE, MODE_HASH, MODE_TRACKED = 0, 1, 2
FULL, VERIFY, COMPRESS = 1, 2, 4


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what} -> status {status}")
        self.status = status


class Report(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "scanned_pages", "scanned_bytes", "dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no intrinsics, -O2)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
                                   "-o", tmp, _SRC])
            os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        u8p, u64p, u32p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
        L.orc_create.restype = C.c_void_p
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_register_region.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, u32p]
        L.orc_unregister_region.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_mark_dirty.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64]
        L.orc_mark_pages.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]
        L.orc_detect.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.orc_sync_shadow.argtypes = [C.c_void_p, u64p]
        L.orc_image_required_bytes.argtypes = [C.c_void_p, C.c_uint64, u64p]
        L.orc_checkpoint_gather.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.POINTER(Report)]
        L.orc_restore_scatter.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(Report)]
        L.orc_xxh3_64.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_xxh3_64.restype = C.c_uint64
        L.orc_crc32.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_crc32.restype = C.c_uint32
        L.orc_get_force.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.orc_get_hashes.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.orc_get_mirror.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.orc_page_hash.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p]
        L.orc_z_encode.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_z_encode.restype = C.c_uint64
        L.orc_z_decode.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.orc_z_decode.restype = C.c_int
        L.orc_restore_begin.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32]
        L.orc_restore_fetch.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p, u64p]
        L.orc_restore_end.argtypes = [C.c_void_p, C.POINTER(Report)]
        for f in ("orc_restore_begin", "orc_restore_fetch", "orc_restore_end","orc_register_region", "orc_unregister_region", "orc_mark_dirty", "orc_mark_pages", "orc_detect",
                  "orc_sync_shadow", "orc_image_required_bytes", "orc_checkpoint_gather",
                  "orc_restore_scatter", "orc_get_force", "orc_get_hashes", "orc_get_mirror",
                  "orc_page_hash"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def xxh3_64(data) -> int:
    a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return int(lib().orc_xxh3_64(_ptr(a), a.nbytes))


def crc32(data) -> int:
    a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return int(lib().orc_crc32(_ptr(a), a.nbytes))


def z_encode(unit) -> bytes:
    """The oracle's unit codec (reading Z3: greedy LZ77 + fixed-Huffman DEFLATE): encode 4096 bytes."""
    a = np.ascontiguousarray(np.frombuffer(bytes(unit), dtype=np.uint8))
    assert a.nbytes == 4096
    out = np.zeros(4096, dtype=np.uint8)
    n = int(lib().orc_z_encode(_ptr(a), _ptr(out)))
    return out[:n].tobytes()


def z_decode(enc: bytes):
    """Decode one unit; None if the encoding is invalid."""
    a = np.frombuffer(bytes(enc) + b"\0", dtype=np.uint8)
    out = np.zeros(4096, dtype=np.uint8)
    ok = lib().orc_z_decode(_ptr(a), len(enc), _ptr(out))
    return out.tobytes() if ok else None


def aligned_empty(nbytes: int, align: int = 256) -> np.ndarray:
    """uint8 array whose data pointer is `align`-byte aligned."""
    raw = np.empty(nbytes + align, dtype=np.uint8)
    off = (-raw.ctypes.data) % align
    return raw[off:off + nbytes]


class Oracle:
    """One oracle context: the CPU model of a crum_ctx."""

    def __init__(self):
        self._L = lib()
        self._h = self._L.orc_create()
        self._regions: dict[int, tuple[np.ndarray, int, int, int]] = {}

    def close(self):
        if self._h:
            self._L.orc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != OK:
            raise OracleError(st, what)

    # -- Alg. 1 "CUDA Create UVM region"
    def register(self, mem: np.ndarray, page_size: int, mode: int = MODE_COMPARE, nbytes: int | None = None) -> int:
        nbytes = mem.nbytes if nbytes is None else nbytes
        rid = C.c_uint32(0)
        st = self._L.orc_register_region(self._h, _ptr(mem), nbytes, page_size, mode, C.byref(rid))
        self._check(st, "register")
        self._regions[rid.value] = (mem, nbytes, page_size, mode)
        return rid.value

    def try_register(self, ptr: int, nbytes: int, page_size: int, mode: int = MODE_COMPARE) -> int:
        rid = C.c_uint32(0)
        return self._L.orc_register_region(self._h, ptr, nbytes, page_size, mode, C.byref(rid))

    def unregister(self, rid: int):
        self._check(self._L.orc_unregister_region(self._h, rid), "unregister")
        self._regions.pop(rid, None)

    def mark_dirty(self, rid: int, off: int, length: int) -> int:
        return self._L.orc_mark_dirty(self._h, rid, off, length)

    def mark_pages(self, rid: int, pages) -> int:
        a = np.ascontiguousarray(np.asarray(pages, dtype=np.uint32))
        return self._L.orc_mark_pages(self._h, rid, a.ctypes.data if a.size else None, a.size)

    def n_pages(self, rid: int) -> int:
        _, b, p, _ = self._regions[rid]
        return -(-b // p)

    def detect(self, rid: int) -> np.ndarray:
        out = np.zeros(self.n_pages(rid), dtype=np.uint8)
        self._check(self._L.orc_detect(self._h, rid, _ptr(out)), "detect")
        return out

    def sync_shadow(self) -> int:
        n = C.c_uint64(0)
        self._check(self._L.orc_sync_shadow(self._h, C.byref(n)), "sync")
        return n.value

    def required_bytes(self, max_dirty: int = 2**63) -> int:
        n = C.c_uint64(0)
        self._check(self._L.orc_image_required_bytes(self._h, max_dirty, C.byref(n)), "required")
        return n.value

    def checkpoint_gather(self, flags: int = 0, capacity: int | None = None, out: np.ndarray | None = None):
        """Returns (status, image bytes or None, report dict).  With `out` (a
        caller-owned uint8 buffer of at least `capacity` bytes, reused across
        calls) the image is a view of it and nothing is allocated or copied."""
        cap = self.required_bytes() if capacity is None else capacity
        buf = np.zeros(max(cap, 1), dtype=np.uint8) if out is None else out
        assert buf.nbytes >= cap
        rep = Report()
        st = self._L.orc_checkpoint_gather(self._h, flags, _ptr(buf), cap, C.byref(rep))
        if st != OK:
            return st, None, rep.as_dict()
        img = buf[:rep.image_bytes] if out is not None else buf[:rep.image_bytes].copy()
        return st, img, rep.as_dict()

    def restore_scatter(self, image: np.ndarray, flags: int = 0):
        image = np.ascontiguousarray(image, dtype=np.uint8)
        rep = Report()
        st = self._L.orc_restore_scatter(self._h, _ptr(image) if image.nbytes else 0, image.nbytes, flags, C.byref(rep))
        return st, rep.as_dict()

    # -- lazy restore: the sec. 4.2 read-fault heuristic applied to restart
    def restore_begin(self, image: np.ndarray, flags: int = 0) -> int:
        image = np.ascontiguousarray(image, dtype=np.uint8)
        st = self._L.orc_restore_begin(self._h, _ptr(image) if image.nbytes else 0, image.nbytes, flags)
        if st == OK:
            self._sess_img = image          # the oracle reads it until restore_end
        return st

    def restore_fetch(self, rid: int, page: int):
        """Returns (status, pages newly present, image slots written)."""
        cov, res = C.c_uint64(0), C.c_uint64(0)
        st = self._L.orc_restore_fetch(self._h, rid, page, C.byref(cov), C.byref(res))
        return st, cov.value, res.value

    def restore_end(self):
        rep = Report()
        st = self._L.orc_restore_end(self._h, C.byref(rep))
        self._sess_img = None
        return st, rep.as_dict()

    def force_bits(self, rid: int) -> np.ndarray:
        out = np.zeros(self.n_pages(rid), dtype=np.uint8)
        self._check(self._L.orc_get_force(self._h, rid, _ptr(out)), "force")
        return out

    def hashes(self, rid: int) -> np.ndarray:
        out = np.zeros(self.n_pages(rid), dtype=np.uint64)
        self._check(self._L.orc_get_hashes(self._h, rid, _ptr(out)), "hashes")
        return out

    def mirror(self, rid: int) -> np.ndarray:
        out = np.zeros(self._regions[rid][1], dtype=np.uint8)
        self._check(self._L.orc_get_mirror(self._h, rid, _ptr(out)), "mirror")
        return out

    def page_hash(self, rid: int, i: int) -> int:
        h = C.c_uint64(0)
        self._check(self._L.orc_page_hash(self._h, rid, i, C.byref(h)), "page_hash")
        return h.value
