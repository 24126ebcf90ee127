"""Thin ctypes binding over libcrum.so (include/crum.h, include/crum_synth.h).

Argument marshalling only: every step of the shadow-page path runs in the
library's sm_100a kernels.  There is no CPU fallback -- if libcrum.so is
missing this module raises ImportError (build it with
``python -m paper_1808_00117_b200.build``).

Region memory, streams and images are passed as raw addresses; helpers accept
torch tensors / streams (``.data_ptr()``, ``.cuda_stream``) without importing
torch themselves.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcrum.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libcrum.so not built at {LIB_PATH}; run `python -m paper_1808_00117_b200.build`")

_L = C.CDLL(LIB_PATH)

OK = 0
E_INVAL, E_OVERLAP, E_NOREGION, E_RANGE, E_NOMEM = -1, -2, -3, -4, -5
E_CAPACITY, E_CORRUPT, E_MISMATCH, E_BUSY, E_DEVICE, E_CUDA, E_IO = -6, -7, -8, -9, -10, -11, -12
MODE_COMPARE, MODE_HASH = 0, 1
FULL, VERIFY, COMPRESS = 1, 2, 4
MODE_TRACKED = 2
CFG_TIMING, CFG_NO_GRAPH, CFG_FUSED, CFG_TRACE, CFG_NO_MAPPED = 1, 2, 4, 8, 16
NUMA_AUTO, NUMA_DEFAULT = -1, -2
PATH_FUSED, PATH_COMPRESSED, PATH_SMALL, PATH_MAPPED = 1, 2, 4, 8
PERSIST_FSYNC, PERSIST_DIRECT = 1, 2
EXPORT_FORCE, EXPORT_HASHES, EXPORT_MIRROR = 0, 1, 2
ALL_PAGES = (1 << 64) - 1

# Every symbol include/*.h declares (checked by tests/test_abi_cpu.py).
EXPORTED = (
    "crum_create", "crum_destroy", "crum_register_region", "crum_register_regions", "crum_unregister_region",
    "crum_mark_dirty", "crum_sync_shadow", "crum_image_required_bytes", "crum_image_create", "crum_image_import",
    "crum_image_data", "crum_image_destroy", "crum_checkpoint_gather", "crum_checkpoint_gather_device",
    "crum_restore_scatter", "crum_restore_scatter_device", "crum_status_string", "crum_last_error_detail",
    "crum_debug_detect", "crum_debug_export", "crum_launch_count", "crum_last_report",
    "crum_synth_fill", "crum_synth_write_pages", "crum_synth_scrub", "crum_probe_copy",
    "crum_synth_fill_regions", "crum_synth_write_regions",
    "crum_synth_alloc_managed", "crum_synth_free_managed", "crum_synth_write_pages_tracked",
    "crum_mark_dirty_pages", "crum_region_tracker",
    "crum_image_persist", "crum_image_persist_wait", "crum_image_persist_busy", "crum_image_load",
    "crum_restore_begin", "crum_restore_fetch", "crum_restore_end",
    "crum_image_numa_node", "crum_device_numa_node", "crum_config_init", "crum_pinned_pool_info",
)


class SynthRegion(C.Structure):
    """crum_synth_region (include/crum_synth.h): one region of a batched synth call."""
    _fields_ = [("dev_ptr", C.c_void_p), ("bytes", C.c_uint64), ("page_size", C.c_uint64),
                ("region_index", C.c_uint64), ("dev_pages", C.c_void_p), ("n_pages", C.c_uint64)]


class Tracker(C.Structure):
    """crum_tracker: device-side marking handle of a TRACKED region."""
    _fields_ = [("force", C.c_void_p), ("bytes", C.c_uint64), ("log2_page", C.c_uint32), ("reserved", C.c_uint32)]


class Config(C.Structure):
    """crum_config (include/crum.h): every tuning choice of the library, per context."""
    _fields_ = [("chunk_bytes", C.c_uint64), ("pinned_pool_bytes", C.c_uint64), ("numa_node", C.c_int32),
                ("flags", C.c_uint32)]


class RegionDesc(C.Structure):
    """crum_region_desc (include/crum.h): one entry of a batch registration."""
    _fields_ = [("ptr", C.c_void_p), ("bytes", C.c_uint64), ("page_size", C.c_uint64), ("mode", C.c_uint32),
                ("reserved", C.c_uint32)]


class Report(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("scanned_pages", "scanned_bytes", "dirty_pages", "dirty_bytes",
                                          "dirty_runs", "image_bytes")] + \
               [(n, C.c_double) for n in ("t_detect_ms", "t_compact_ms", "t_gather_ms", "t_copy_ms",
                                          "t_total_ms")] + \
               [("path", C.c_uint32), ("reserved", C.c_uint32)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_vp, _u64, _u32, _i = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
_sig = {
    "crum_create": (_i, [_i, C.POINTER(Config), C.POINTER(_vp)]),
    "crum_config_init": (_i, [C.POINTER(Config)]),
    "crum_pinned_pool_info": (_i, [_vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32)]),
    "crum_destroy": (_i, [_vp]),
    "crum_register_region": (_i, [_vp, _vp, _u64, _u64, _u32, C.POINTER(_u32)]),
    "crum_register_regions": (_i, [_vp, _u32, _vp, C.POINTER(_u32), C.POINTER(_u32)]),
    "crum_unregister_region": (_i, [_vp, _u32]),
    "crum_mark_dirty": (_i, [_vp, _u32, _u64, _u64]),
    "crum_sync_shadow": (_i, [_vp, _vp, C.POINTER(_u64)]),
    "crum_image_required_bytes": (_i, [_vp, _u64, C.POINTER(_u64)]),
    "crum_image_create": (_i, [_vp, _u64, C.POINTER(_vp)]),
    "crum_image_import": (_i, [_vp, _vp, _u64, C.POINTER(_vp)]),
    "crum_image_data": (_i, [_vp, C.POINTER(_vp), C.POINTER(_u64), C.POINTER(_u64)]),
    "crum_image_destroy": (_i, [_vp]),
    "crum_image_numa_node": (_i, [_vp, C.POINTER(_i)]),
    "crum_device_numa_node": (_i, [_i, C.POINTER(_i)]),
    "crum_checkpoint_gather": (_i, [_vp, _vp, _vp, _u32, C.POINTER(Report)]),
    "crum_checkpoint_gather_device": (_i, [_vp, _vp, _u64, _vp, _u32, C.POINTER(Report)]),
    "crum_restore_scatter": (_i, [_vp, _vp, _vp, _u32, C.POINTER(Report)]),
    "crum_restore_scatter_device": (_i, [_vp, _vp, _u64, _vp, _u32, C.POINTER(Report)]),
    "crum_status_string": (C.c_char_p, [_i]),
    "crum_last_error_detail": (C.c_char_p, []),
    "crum_debug_detect": (_i, [_vp, _vp, _vp, _u64]),
    "crum_debug_export": (_i, [_vp, _u32, _i, _vp, _u64]),
    "crum_launch_count": (_u64, [_vp]),
    "crum_last_report": (_i, [_vp, C.POINTER(Report)]),
    "crum_synth_fill": (_i, [_vp, _u64, _u64, _u64, _u64, _vp]),
    "crum_synth_write_pages": (_i, [_vp, _u64, _u64, _vp, _u64, _u64, _u64, _u64, _i, _vp]),
    "crum_synth_scrub": (_i, [_vp, _u64, _vp]),
    "crum_synth_fill_regions": (_i, [C.POINTER(SynthRegion), _u64, _u64, _vp]),
    "crum_synth_write_regions": (_i, [C.POINTER(SynthRegion), _u64, _u64, _u64, _i, _vp]),
    "crum_probe_copy": (_i, [_vp, _vp, _u64, _i, _vp]),
    "crum_synth_alloc_managed": (_i, [C.POINTER(_vp), _u64, _i, _u64]),
    "crum_synth_free_managed": (_i, [_vp]),
    "crum_synth_write_pages_tracked": (_i, [_vp, _u64, _u64, _vp, _u64, _u64, _u64, _u64, _i, C.POINTER(Tracker),
                                           _vp]),
    "crum_mark_dirty_pages": (_i, [_vp, _u32, _vp, _u64, _vp]),
    "crum_region_tracker": (_i, [_vp, _u32, C.POINTER(Tracker)]),
    "crum_image_persist": (_i, [_vp, C.c_char_p, _u32]),
    "crum_image_persist_wait": (_i, [_vp]),
    "crum_image_persist_busy": (_i, [_vp, C.POINTER(_i)]),
    "crum_image_load": (_i, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "crum_restore_begin": (_i, [_vp, _vp, _vp, _u32, C.POINTER(_vp)]),
    "crum_restore_fetch": (_i, [_vp, _u32, _u64, _vp, C.POINTER(_u64), C.POINTER(_u64)]),
    "crum_restore_end": (_i, [_vp, _vp, C.POINTER(Report)]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_L, _name)
    _f.restype, _f.argtypes = _res, _args


def lib():
    return _L


class CrumError(RuntimeError):
    def __init__(self, status: int, what: str):
        detail = (_L.crum_last_error_detail() or b"").decode(errors="replace")
        msg = (_L.crum_status_string(status) or b"?").decode()
        super().__init__(f"{what}: {msg} ({status}) {detail}")
        self.status = status
        self.detail = detail


def _check(st: int, what: str):
    if st != OK:
        raise CrumError(st, what)


def _stream(s) -> int | None:
    if s is None:
        return None
    if hasattr(s, "cuda_stream"):
        return int(s.cuda_stream)
    return int(s)


def _addr(x) -> int:
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    return int(x)


class Image:
    """A library-owned pinned host image (crum_image)."""

    def __init__(self, ctx: "Context", capacity: int | None = None, data: bytes | np.ndarray | None = None,
                 path: str | None = None):
        self._h = _vp()
        self._ctx = ctx
        if path is not None:
            _check(_L.crum_image_load(ctx._h, os.fsencode(path), C.byref(self._h)), "crum_image_load")
        elif data is not None:
            buf = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray)
                                       else data.view(np.uint8).reshape(-1))
            _check(_L.crum_image_import(ctx._h, buf.ctypes.data if buf.nbytes else None, buf.nbytes,
                                        C.byref(self._h)), "crum_image_import")
        else:
            if capacity is None:
                capacity = ctx.image_required_bytes()
            _check(_L.crum_image_create(ctx._h, capacity, C.byref(self._h)), "crum_image_create")

    def _info(self):
        p, n, cap = _vp(), _u64(), _u64()
        _check(_L.crum_image_data(self._h, C.byref(p), C.byref(n), C.byref(cap)), "crum_image_data")
        return p.value or 0, n.value, cap.value

    @property
    def length(self) -> int:
        return self._info()[1]

    @property
    def capacity(self) -> int:
        return self._info()[2]

    @property
    def address(self) -> int:
        return self._info()[0]

    @property
    def numa_node(self) -> int:
        """Host NUMA node the pinned pages are bound to (-1: default placement)."""
        n = _i()
        _check(_L.crum_image_numa_node(self._h, C.byref(n)), "crum_image_numa_node")
        return n.value

    def view(self, full_capacity: bool = False) -> np.ndarray:
        """Zero-copy numpy view of the pinned buffer (valid until destroy)."""
        p, n, cap = self._info()
        m = cap if full_capacity else n
        if m == 0:
            return np.zeros(0, dtype=np.uint8)
        return np.ctypeslib.as_array((C.c_uint8 * m).from_address(p))

    def tobytes(self) -> bytes:
        return self.view().tobytes()

    # -- forked checkpoint (sec. 3.3): persist on a writer thread
    def persist(self, path: str, fsync: bool = False, direct: bool = False):
        """Start writing the image to `path`; returns at once.  direct: O_DIRECT
        (no page-cache copy); fsync: fsync before completion."""
        _check(_L.crum_image_persist(self._h, os.fsencode(path), (PERSIST_FSYNC if fsync else 0) |
                                     (PERSIST_DIRECT if direct else 0)), "crum_image_persist")

    def persist_wait(self):
        """Wait for the writer; raises CrumError(CRUM_E_IO) if it failed."""
        _check(_L.crum_image_persist_wait(self._h), "crum_image_persist_wait")

    @property
    def busy(self) -> bool:
        b = _i()
        _check(_L.crum_image_persist_busy(self._h, C.byref(b)), "crum_image_persist_busy")
        return bool(b.value)

    def destroy(self):
        if self._h and self._h.value:
            _check(_L.crum_image_destroy(self._h), "crum_image_destroy")   # BUSY: a restore session reads it
            self._h = _vp()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class RestoreSession:
    """An open lazy restore (crum_restore_begin .. crum_restore_end): the
    sec. 4.2 read-fault heuristic applied to restart."""

    def __init__(self, ctx: "Context", image: Image, stream=None, flags: int = 0):
        self._h = _vp()
        self._ctx, self._img = ctx, image
        _check(_L.crum_restore_begin(ctx._h, image._h, _stream(stream), flags, C.byref(self._h)),
               "crum_restore_begin")

    def fetch(self, region_id: int, page: int, stream=None):
        """Read fault on (region, page): returns (pages newly present, slots written)."""
        cov, res = _u64(), _u64()
        _check(_L.crum_restore_fetch(self._h, region_id, page, _stream(stream), C.byref(cov), C.byref(res)),
               "crum_restore_fetch")
        return cov.value, res.value

    def end(self, stream=None) -> dict:
        rep = Report()
        h, self._h = self._h, _vp()
        if not (h and h.value):
            raise CrumError(E_INVAL, "crum_restore_end: session already closed")
        _check(_L.crum_restore_end(h, _stream(stream), C.byref(rep)), "crum_restore_end")
        return rep.as_dict()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        if self._h and self._h.value:
            self.end()

    def __del__(self):
        try:
            if self._h and self._h.value:
                self.end()
        except Exception:
            pass


class Context:
    """crum_ctx: one per (process, CUDA device)."""

    def __init__(self, device: int = 0, chunk_bytes: int = 0, timing: bool = False, flags: int = 0,
                 numa_node: int = NUMA_AUTO, pinned_pool_bytes: int = 0):
        self._h = _vp()
        cfg = Config()
        _check(_L.crum_config_init(C.byref(cfg)), "crum_config_init")
        cfg.chunk_bytes = chunk_bytes
        cfg.pinned_pool_bytes = pinned_pool_bytes
        cfg.numa_node = numa_node
        cfg.flags = flags | (CFG_TIMING if timing else 0)
        _check(_L.crum_create(device, C.byref(cfg), C.byref(self._h)), "crum_create")
        self.device = device
        self._keep = {}

    def close(self):
        if self._h and self._h.value:
            _L.crum_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- Alg. 1 "CUDA Create UVM region"
    def register_region(self, ptr, nbytes: int | None = None, page_size: int = 65536, mode: int = MODE_COMPARE,
                        keep=None) -> int:
        if nbytes is None:
            nbytes = int(ptr.numel() * ptr.element_size())
        rid = _u32()
        _check(_L.crum_register_region(self._h, _addr(ptr), nbytes, page_size, mode, C.byref(rid)),
               "crum_register_region")
        self._keep[rid.value] = keep if keep is not None else (ptr if hasattr(ptr, "data_ptr") else None)
        return rid.value

    def register_regions(self, regions) -> list[int]:
        """Batch registration (crum_register_regions): `regions` is a list of
        (ptr, nbytes, page_size, mode); ptr a tensor (kept alive) or an address.
        Returns the new ids in order; raises CrumError (nothing registered)."""
        ids, fail = self.try_register_regions([(_addr(p), n, P, m) for p, n, P, m in regions])
        if isinstance(ids, int):
            _check(ids, f"crum_register_regions (descriptor {fail})")
        for (p, _, _, _), rid in zip(regions, ids):
            self._keep[rid] = p if hasattr(p, "data_ptr") else None
        return ids

    def try_register_regions(self, descs):
        """Raw crum_register_regions over (address, nbytes, page_size, mode)
        tuples: (ids, None) on success, else (status, failed index)."""
        n = len(descs)
        arr = (RegionDesc * max(n, 1))(*[RegionDesc(a, nb, P, m, 0) for a, nb, P, m in descs])
        ids = (_u32 * max(n, 1))()
        fail = _u32(0)
        st = _L.crum_register_regions(self._h, n, C.cast(arr, _vp), ids, C.byref(fail))
        if st != OK:
            return st, (None if fail.value == 0xFFFFFFFF else fail.value)
        return [ids[k] for k in range(n)], None

    def try_register(self, ptr: int, nbytes: int, page_size: int, mode: int = MODE_COMPARE) -> int:
        """Raw status of crum_register_region (tests of the error paths)."""
        rid = _u32()
        return _L.crum_register_region(self._h, ptr, nbytes, page_size, mode, C.byref(rid))

    def unregister_region(self, rid: int):
        _check(_L.crum_unregister_region(self._h, rid), "crum_unregister_region")
        self._keep.pop(rid, None)

    def mark_dirty(self, rid: int, offset: int, length: int) -> int:
        return _L.crum_mark_dirty(self._h, rid, offset, length)

    def mark_dirty_pages(self, rid: int, dev_pages, n: int, stream=None) -> int:
        """Stream-ordered: force bits of the region-local page indices in the
        device u32 array dev_pages[0..n)."""
        return _L.crum_mark_dirty_pages(self._h, rid, _addr(dev_pages) if n else None, n, _stream(stream))

    def region_tracker(self, rid: int) -> Tracker:
        t = Tracker()
        _check(_L.crum_region_tracker(self._h, rid, C.byref(t)), "crum_region_tracker")
        return t

    # -- Alg. 1 "CUDA call"
    def sync_shadow(self, stream=None, wait: bool = True):
        n = _u64()
        _check(_L.crum_sync_shadow(self._h, _stream(stream), C.byref(n) if wait else None), "crum_sync_shadow")
        return n.value if wait else None

    def image_required_bytes(self, max_dirty: int = ALL_PAGES) -> int:
        n = _u64()
        _check(_L.crum_image_required_bytes(self._h, max_dirty, C.byref(n)), "crum_image_required_bytes")
        return n.value

    def new_image(self, capacity: int | None = None) -> Image:
        return Image(self, capacity)

    def import_image(self, data) -> Image:
        return Image(self, data=data)

    def load_image(self, path: str) -> Image:
        """Restart from storage: a new pinned image holding the file's bytes."""
        return Image(self, path=path)

    # -- sec. 3.4 drain
    def checkpoint_gather(self, image: Image, stream=None, flags: int = 0, raise_on_error: bool = True):
        rep = Report()
        st = _L.crum_checkpoint_gather(self._h, image._h, _stream(stream), flags, C.byref(rep))
        if raise_on_error:
            _check(st, "crum_checkpoint_gather")
            return rep.as_dict()
        return st, rep.as_dict()

    def checkpoint_gather_device(self, dev_ptr, capacity: int, stream=None, flags: int = 0, report: bool = True,
                                 raise_on_error: bool = True):
        rep = Report()
        st = _L.crum_checkpoint_gather_device(self._h, _addr(dev_ptr), capacity, _stream(stream), flags,
                                              C.byref(rep) if report else None)
        if raise_on_error:
            _check(st, "crum_checkpoint_gather_device")
            return rep.as_dict() if report else None
        return st, (rep.as_dict() if report else None)

    # -- sec. 3.4 restart
    def restore_scatter(self, image: Image, stream=None, flags: int = 0, raise_on_error: bool = True):
        rep = Report()
        st = _L.crum_restore_scatter(self._h, image._h, _stream(stream), flags, C.byref(rep))
        if raise_on_error:
            _check(st, "crum_restore_scatter")
            return rep.as_dict()
        return st, rep.as_dict()

    def restore_begin(self, image: Image, stream=None, flags: int = 0) -> RestoreSession:
        """Lazy restore: validate now, restore on fetch() / end()."""
        return RestoreSession(self, image, stream, flags)

    def restore_scatter_device(self, dev_ptr, length: int, stream=None, flags: int = 0, report: bool = True,
                               raise_on_error: bool = True):
        rep = Report()
        st = _L.crum_restore_scatter_device(self._h, _addr(dev_ptr), length, _stream(stream), flags,
                                            C.byref(rep) if report else None)
        if raise_on_error:
            _check(st, "crum_restore_scatter_device")
            return rep.as_dict() if report else None
        return st, (rep.as_dict() if report else None)

    # -- test hooks
    def debug_detect(self, n_pages: int, stream=None) -> np.ndarray:
        out = np.zeros(n_pages, dtype=np.uint8)
        _check(_L.crum_debug_detect(self._h, _stream(stream), out.ctypes.data if n_pages else None, n_pages),
               "crum_debug_detect")
        return out

    def debug_export(self, rid: int, what: int, n: int) -> np.ndarray:
        dtype = np.uint64 if what == EXPORT_HASHES else np.uint8
        out = np.zeros(n, dtype=dtype)
        _check(_L.crum_debug_export(self._h, rid, what, out.ctypes.data, out.nbytes), "crum_debug_export")
        return out

    def last_report(self) -> dict:
        """Report of the most recent sync/gather/restore (waits for it)."""
        rep = Report()
        _check(_L.crum_last_report(self._h, C.byref(rep)), "crum_last_report")
        return rep.as_dict()

    @property
    def launch_count(self) -> int:
        return int(_L.crum_launch_count(self._h))

    def pool_info(self) -> dict:
        """The context's pinned pool: bytes, in_use, largest_free, images."""
        b, u, l, n = _u64(), _u64(), _u64(), _u32()
        _check(_L.crum_pinned_pool_info(self._h, C.byref(b), C.byref(u), C.byref(l), C.byref(n)),
               "crum_pinned_pool_info")
        return {"bytes": b.value, "in_use": u.value, "largest_free": l.value, "images": n.value}


# -- synthetic inputs (include/crum_synth.h) --------------------------------
def device_numa_node(device: int) -> int:
    """Host NUMA node of CUDA device `device` (-1: unknown or a single-node host)."""
    n = _i()
    _check(_L.crum_device_numa_node(device, C.byref(n)), "crum_device_numa_node")
    return n.value


def synth_fill(dev_ptr, nbytes: int, seed: int, region_index: int, word_offset: int = 0, stream=None):
    _check(_L.crum_synth_fill(_addr(dev_ptr), nbytes, seed, region_index, word_offset, _stream(stream)),
           "crum_synth_fill")


def synth_write_pages(dev_ptr, nbytes: int, page_size: int, dev_pages, n_pages: int, seed: int, epoch: int,
                      region_index: int, touch: bool = False, stream=None):
    _check(_L.crum_synth_write_pages(_addr(dev_ptr), nbytes, page_size, _addr(dev_pages) if n_pages else None,
                                     n_pages, seed, epoch, region_index, int(touch), _stream(stream)),
           "crum_synth_write_pages")


def synth_write_pages_tracked(dev_ptr, nbytes: int, page_size: int, dev_pages, n_pages: int, seed: int, epoch: int,
                              region_index: int, tracker: Tracker, touch: bool = False, stream=None):
    _check(_L.crum_synth_write_pages_tracked(_addr(dev_ptr), nbytes, page_size, _addr(dev_pages) if n_pages else None,
                                             n_pages, seed, epoch, region_index, int(touch), C.byref(tracker),
                                             _stream(stream)), "crum_synth_write_pages_tracked")


def synth_fill_regions(regions, seed: int, stream=None):
    """regions: [(dev_ptr, nbytes, region_index)], one launch for all of them."""
    arr = (SynthRegion * len(regions))(*[SynthRegion(_addr(p), nb, 0, r, None, 0) for p, nb, r in regions])
    _check(_L.crum_synth_fill_regions(arr, len(regions), seed, _stream(stream)), "crum_synth_fill_regions")


def synth_write_regions(regions, seed: int, epoch: int, touch: bool = False, stream=None):
    """regions: [(dev_ptr, nbytes, page_size, region_index, dev_pages, n_pages)], one launch."""
    arr = (SynthRegion * len(regions))(*[SynthRegion(_addr(p), nb, P, r, _addr(pg) if n else None, n)
                                         for p, nb, P, r, pg, n in regions])
    _check(_L.crum_synth_write_regions(arr, len(regions), seed, epoch, int(touch), _stream(stream)),
           "crum_synth_write_regions")


def synth_scrub(dev_ptr, nbytes: int, stream=None):
    _check(_L.crum_synth_scrub(_addr(dev_ptr), nbytes, _stream(stream)), "crum_synth_scrub")


def probe_copy(dst, src, nbytes: int, blocks: int = 0, stream=None):
    _check(_L.crum_probe_copy(_addr(dst), _addr(src), nbytes, blocks, _stream(stream)), "crum_probe_copy")


class ManagedBuffer:
    """Config-5 managed (UVM) allocation; .ptr / .nbytes like a raw buffer."""

    def __init__(self, nbytes: int, device: int = 0, device_bytes: int | None = None):
        p = _vp()
        _check(_L.crum_synth_alloc_managed(C.byref(p), nbytes, device,
                                           nbytes if device_bytes is None else device_bytes),
               "crum_synth_alloc_managed")
        self.ptr = p.value
        self.nbytes = nbytes

    def data_ptr(self) -> int:
        return self.ptr

    def free(self):
        if self.ptr:
            _L.crum_synth_free_managed(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
