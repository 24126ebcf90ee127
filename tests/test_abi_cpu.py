"""C-ABI checks that need no GPU: libcrum.so builds/loads, exports every
symbol include/*.h declares (and the binding binds exactly those), status
strings, and CPU-side argument validation."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    return m


def declared_symbols():
    names = set()
    for h in ("crum.h", "crum_synth.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^CRUM_API [^(]*?\b(crum_\w+)\(", src, flags=re.M))
    return names


def test_header_declares_the_four_north_star_calls():
    names = declared_symbols()
    for n in ("crum_register_region", "crum_sync_shadow", "crum_checkpoint_gather", "crum_restore_scatter"):
        assert n in names


def test_library_exports_every_declared_symbol(crum):
    lib = C.CDLL(crum.LIB_PATH)
    for n in sorted(declared_symbols()):
        assert hasattr(lib, n), n
    assert set(crum.EXPORTED) == declared_symbols()


def test_library_is_sm100a(crum):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", crum.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings(crum):
    L = crum.lib()
    for st in range(-11, 1):
        assert L.crum_status_string(st)
    assert L.crum_status_string(crum.E_CORRUPT) == b"corrupt image"


def test_cpu_side_argument_checks(crum):
    L = crum.lib()
    h = C.c_void_p()
    assert L.crum_create(0, None, None) == crum.E_INVAL
    for bad in (crum.Config(4097, 0, -1, 0), crum.Config(0, 4097, -1, 0), crum.Config(0, 0, -3, 0),
                crum.Config(0, 0, 1024, 0), crum.Config(0, 0, -1, 1 << 9)):
        assert L.crum_create(0, C.byref(bad), C.byref(h)) == crum.E_INVAL
    cfg = crum.Config(123, 4096, 5, 7)
    assert L.crum_config_init(C.byref(cfg)) == crum.OK
    assert (cfg.chunk_bytes, cfg.pinned_pool_bytes, cfg.numa_node, cfg.flags) == (0, 0, crum.NUMA_AUTO, 0)
    assert L.crum_config_init(None) == crum.E_INVAL
    assert L.crum_pinned_pool_info(None, None, None, None, None) == crum.E_INVAL
    assert L.crum_destroy(None) == crum.E_INVAL
    assert L.crum_sync_shadow(None, None, None) == crum.E_INVAL
    assert L.crum_image_destroy(None) == crum.E_INVAL
    # the widened rows' calls reject null handles before touching CUDA
    assert L.crum_image_persist(None, b"/tmp/x", 0) == crum.E_INVAL
    assert L.crum_image_persist_wait(None) == crum.E_INVAL
    busy = C.c_int(7)
    assert L.crum_image_persist_busy(None, C.byref(busy)) == crum.E_INVAL
    assert L.crum_image_load(None, None, C.byref(h)) == crum.E_INVAL
    assert L.crum_image_load(None, b"/nonexistent/crum/image", C.byref(h)) == crum.E_IO
    assert L.crum_restore_begin(None, None, None, 0, C.byref(h)) == crum.E_INVAL
    cov, res = C.c_uint64(), C.c_uint64()
    assert L.crum_restore_fetch(None, 1, 0, None, C.byref(cov), C.byref(res)) == crum.E_INVAL
    assert L.crum_restore_end(None, None, None) == crum.E_INVAL
    assert L.crum_mark_dirty_pages(None, 1, None, 0, None) == crum.E_INVAL
    assert L.crum_status_string(crum.E_IO) == b"file I/O error"
    node = C.c_int(7)
    assert L.crum_image_numa_node(None, C.byref(node)) == crum.E_INVAL
    assert L.crum_device_numa_node(0, None) == crum.E_INVAL
    assert L.crum_device_numa_node(-1, C.byref(node)) == crum.E_DEVICE
    # batched synth calls: argument checks happen before any CUDA work
    assert L.crum_synth_fill_regions(None, 0, 1, None) == crum.OK
    assert L.crum_synth_fill_regions(None, 2, 1, None) == crum.E_INVAL
    bad = (crum.SynthRegion * 1)(crum.SynthRegion(0x1003, 64, 0, 0, None, 0))   # unaligned pointer
    assert L.crum_synth_fill_regions(bad, 1, 1, None) == crum.E_INVAL
    bad = (crum.SynthRegion * 1)(crum.SynthRegion(0x1000, 64, 12, 0, None, 1))  # page size % 8, no pages
    assert L.crum_synth_write_regions(bad, 1, 1, 0, 0, None) == crum.E_INVAL
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert L.crum_create(0, None, C.byref(h)) == crum.E_DEVICE
        assert b"no CUDA device" in L.crum_last_error_detail()


def test_binding_fails_loudly_without_library(tmp_path):
    """The product path has no fallback: importing the binding against a
    missing library raises ImportError."""
    import subprocess
    import sys
    code = ("import os, sys; sys.path.insert(0, %r); import paper_1808_00117_b200.crum as c; "
            "os.rename(c.LIB_PATH, c.LIB_PATH) ") % ROOT
    # simulate: point the module at a non-existent path
    code = ("import sys, importlib.util; sys.path.insert(0, %r); "
            "spec = importlib.util.spec_from_file_location('crum_probe', %r); m = importlib.util.module_from_spec(spec); "
            "import os; os.path.exists = lambda p: False; spec.loader.exec_module(m)") % (
        ROOT, os.path.join(ROOT, "paper_1808_00117_b200", "crum.py"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr
