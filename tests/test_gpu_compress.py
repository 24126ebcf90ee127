"""GPU parity of compressed images (CRUM_COMPRESS; readings Z2-Z3:
per 4 KiB unit a greedy LZ77 parse in one fixed-Huffman DEFLATE block):
libcrum.so's encoder (pinned image through the chunked pipeline, and device
image) vs the CPU oracle byte for byte, every encoded unit inflated by zlib;
restore (eager, VERIFY, lazy) of compressed images; the GPU decoder's verdict
on damaged streams equal to the oracle's; capacity errors.  Region contents
follow the paper's "50% random" shape, HPGMG-like fp64
fields (smooth, constant, zero ghost zones) and fully random pages."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB = 1 << 10, 1 << 20
C, H = 0, 1
SPECS = [
    (3 * MiB + 777, 4 * KiB, C),
    (40 * 64 * KiB + 12, 64 * KiB, H),
    (5 * 4 * KiB + 9, 4 * KiB, H),
    (2 * MiB * 3 + 100, 2 * MiB, C),
    (7 * 64 * KiB, 64 * KiB, C),
]


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    assert torch.cuda.is_available()
    return m


def fill_structured(h: np.ndarray, seed: int):
    """HPGMG-like content: per 32 KiB box, fp64 values of a smooth field, a
    constant coefficient, or zero (ghost zones / cleared temporaries)."""
    rng = np.random.default_rng(seed)
    n = h.nbytes // 8 * 8
    f = h[:n].view("<f8")
    box = 4096
    for b0 in range(0, f.size, box):
        k = int(rng.integers(0, 4))
        seg = f[b0:b0 + box]
        if k == 0:
            x = np.arange(seg.size) * rng.uniform(0.001, 0.05)
            seg[:] = np.sin(x) * rng.uniform(0.5, 2)
        elif k == 1:
            seg[:] = rng.uniform(-1, 1)
        elif k == 2:
            seg[:] = 0
        else:
            seg[:] = np.round(rng.normal(size=seg.size), 3)
    h[n:] = 0


def shaped_pair(seed_idx, shape="half", specs=None):
    """Pair whose regions are random in their first half and constant after
    (shape 'half'), HPGMG-like ('structured'), or fully random ('random')."""
    from tests.gpu_pair import Pair
    p = Pair(specs or SPECS, synth.seed(seed_idx))
    if shape != "random":
        for r, (h, d) in enumerate(zip(p.host, p.dev)):
            n = h.nbytes
            if shape == "half":
                h[n // 2:] = 0
                h[n // 2 + 4096: n // 2 + 8192] = np.frombuffer(np.full(1024, 0.5, np.float32).tobytes(), np.uint8)
            else:
                fill_structured(h, 1000 * seed_idx + r)
            d.copy_(torch.from_numpy(h))
        torch.cuda.synchronize()
    return p


def check_units_inflate(img_bytes):
    """Every encoded unit of a compressed image inflates (zlib, raw DEFLATE)
    to 4096 bytes, ending exactly at its last byte (an independent decoder)."""
    from tests import imgfmt
    info = imgfmt.parse_image(np.frombuffer(img_bytes, dtype=np.uint8))
    off = info["poff"]
    n_deflate = 0
    for cs in info["zsizes"]:
        enc = img_bytes[off:off + cs]
        if 0 < cs < 4096:
            assert len(imgfmt.z_decode_unit(enc)) == 4096
            n_deflate += 1
        off += cs
    return n_deflate


@pytest.mark.parametrize("shape", ["half", "structured", "random"])
def test_compressed_gather_bit_exact(crum, shape):
    p = shaped_pair({"half": 90, "random": 91, "structured": 94}[shape], shape)
    img = p.g.new_image()
    cap = p.g.image_required_bytes()
    buf = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
    for epoch, d, flags in ((0, 0, 0), (1, 0.2, 0), (2, 0.0, 0), (3, 0.5, 1), (4, 1.0, 0)):
        if epoch:
            p.write(epoch, d)
        st, want, rep_o = p.o.checkpoint_gather(flags=crum.COMPRESS | flags)
        assert st == 0
        if epoch % 2 == 0:
            rep = p.g.checkpoint_gather(img, flags=crum.COMPRESS | flags)
            got = img.tobytes()
        else:
            rep = p.g.checkpoint_gather_device(buf, cap, flags=crum.COMPRESS | flags)
            got = buf[:rep["image_bytes"]].cpu().numpy().tobytes()
        assert rep["path"] & crum.PATH_COMPRESSED
        assert len(got) == len(want), epoch
        assert got == want.tobytes(), epoch
        if epoch in (0, 3):
            n_deflate = check_units_inflate(got)   # random pages: only the zero-padded tail units shrink
            assert n_deflate > 0, epoch
        for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes"):
            assert rep[k] == rep_o[k], (epoch, k)
        assert p.shadows_equal(), epoch


def restart(crum, specs):
    from oracle import oracle
    o = oracle.Oracle()
    g = crum.Context(0)
    hz, dz = [], []
    for nb, P, mode in specs:
        h = oracle.aligned_empty(nb)
        h[:] = 0
        d = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        hz.append(h)
        dz.append(d)
        o.register(h, P, mode)
        g.register_region(d, nb, P, mode)
    return o, g, hz, dz


def test_compressed_restore_chain(crum):
    p = shaped_pair(92)
    imgs, states = [], []
    for epoch in range(5):
        if epoch:
            p.write(epoch, 0.3)
        img = p.g.new_image()
        p.o.checkpoint_gather(flags=crum.COMPRESS if epoch != 2 else 0)
        p.g.checkpoint_gather(img, flags=crum.COMPRESS if epoch != 2 else 0)
        imgs.append(img)
        states.append([h.copy() for h in p.host])
    o, g, hz, dz = restart(crum, SPECS)
    for k, img in enumerate(imgs):
        raw = img.view().copy()
        st, rep_o = o.restore_scatter(raw, crum.VERIFY if k % 2 else 0)
        assert st == 0
        rep = g.restore_scatter(img, flags=crum.VERIFY if k % 2 else 0)
        assert rep["dirty_pages"] == rep_o["dirty_pages"] and rep["image_bytes"] == rep_o["image_bytes"]
        torch.cuda.synchronize()
        for d, h, want in zip(dz, hz, states[k]):
            assert np.array_equal(h, want), k
            assert np.array_equal(d.cpu().numpy(), want), k
    assert g.sync_shadow() == 0
    # device-image restore and lazy restore of a compressed image
    raw = imgs[0].view().copy()
    o2, g2, hz2, dz2 = restart(crum, SPECS)
    dbuf = torch.from_numpy(raw).cuda()
    g2.restore_scatter_device(dbuf, raw.size)
    torch.cuda.synchronize()
    for d, want in zip(dz2, states[0]):
        assert np.array_equal(d.cpu().numpy(), want)
    o3, g3, hz3, dz3 = restart(crum, SPECS)
    assert o3.restore_begin(raw) == 0
    sess = g3.restore_begin(g3.import_image(raw))
    rng = np.random.default_rng(3)
    for _ in range(30):
        r = int(rng.integers(0, len(SPECS)))
        i = int(rng.integers(0, synth.n_pages(*SPECS[r][:2])))
        st, cov, res = o3.restore_fetch(r + 1, i)
        assert sess.fetch(r + 1, i) == (cov, res)
    torch.cuda.synchronize()
    for d, h in zip(dz3, hz3):
        assert np.array_equal(d.cpu().numpy(), h)
    o3.restore_end()
    sess.end()
    for d, want in zip(dz3, states[0]):
        assert np.array_equal(d.cpu().numpy(), want)


def test_compressed_errors(crum):
    from tests import imgfmt
    p = shaped_pair(93)
    small = p.g.new_image(8192)
    st, rep = p.g.checkpoint_gather(small, flags=crum.COMPRESS, raise_on_error=False)
    assert st == crum.E_CAPACITY and rep["image_bytes"] > 8192
    assert p.g.debug_detect(p.N).tolist() == [1] * p.N                   # nothing committed
    tiny = p.g.new_image(100)                                             # < header + table
    st, rep = p.g.checkpoint_gather(tiny, flags=crum.COMPRESS, raise_on_error=False)
    assert st == crum.E_CAPACITY
    img = p.g.new_image()
    p.o.checkpoint_gather(flags=crum.COMPRESS)
    p.g.checkpoint_gather(img, flags=crum.COMPRESS)
    raw = img.view().copy()
    info = imgfmt.parse_image(raw)
    u = next(i for i, cs in enumerate(info["zsizes"]) if 0 < cs < 4096)
    coff = info["poff"] + sum(info["zsizes"][:u])
    bad = raw.copy()
    bad[coff] ^= 1                                                        # BFINAL = 0: not this codec
    o, g, hz, dz = restart(crum, SPECS)
    assert o.restore_scatter(bad)[0] == crum.E_CORRUPT
    st, _ = g.restore_scatter(g.import_image(bad), raise_on_error=False)
    assert st == crum.E_CORRUPT
    torch.cuda.synchronize()
    assert all(int(d.count_nonzero()) == 0 for d in dz)                  # nothing written
    with pytest.raises(crum.CrumError):                                   # lazy: validated at begin
        g.restore_begin(g.import_image(bad))
    assert g.restore_scatter(g.import_image(raw))["dirty_pages"] == p.N


def test_decoder_verdicts_match_oracle(crum):
    """Damaged streams (the CRCs cover only the metadata): random bit flips
    inside encoded units.  The GPU decoder and the oracle give the same
    verdict, and when a damaged stream still decodes, the same bytes."""
    from tests import imgfmt
    p = shaped_pair(95, "structured")
    img = p.g.new_image()
    p.g.checkpoint_gather(img, flags=crum.COMPRESS)
    raw = img.view().copy()
    info = imgfmt.parse_image(raw)
    offs, off = [], info["poff"]
    for cs in info["zsizes"]:
        if 0 < cs < 4096:
            offs.append((off, cs))
        off += cs
    rng = np.random.default_rng(7)
    outcomes = set()
    for t in range(24):
        o0, cs = offs[int(rng.integers(0, len(offs)))]
        bad = raw.copy()
        bit = int(rng.integers(0, 8 * cs))
        bad[o0 + bit // 8] ^= 1 << (bit % 8)
        o, g, hz, dz = restart(crum, SPECS)
        st_o, _ = o.restore_scatter(bad)
        st_g, _ = g.restore_scatter(g.import_image(bad), raise_on_error=False)
        assert st_g == st_o, (t, bit)
        outcomes.add(st_o)
        if st_o == 0:
            torch.cuda.synchronize()
            for d, h in zip(dz, hz):
                assert np.array_equal(d.cpu().numpy(), h), t
    assert crum.E_CORRUPT in outcomes


def test_compressed_multi_chunk(crum):
    """Footprints of several 64 MiB encode chunks: the pinned pipeline's ring
    and per-chunk copies, and a capacity failure part-way through them."""
    specs = [(150 * MiB + 4096 * 3 + 5, 64 * KiB, C), (40 * MiB, 4 * KiB, H)]
    p = shaped_pair(96, "structured", specs)
    for epoch, d in ((0, 0), (1, 0.6)):
        if epoch:
            p.write(epoch, d)
        st, want, rep_o = p.o.checkpoint_gather(flags=crum.COMPRESS)
        short = p.g.new_image(len(want) // 2)
        st, rep = p.g.checkpoint_gather(short, flags=crum.COMPRESS, raise_on_error=False)
        assert st == crum.E_CAPACITY and rep["image_bytes"] == len(want)
        short.destroy()
        img = p.g.new_image(len(want))
        rep = p.g.checkpoint_gather(img, flags=crum.COMPRESS)
        assert img.tobytes() == want.tobytes(), epoch
        assert rep["image_bytes"] == len(want) < rep["dirty_bytes"]
        assert p.shadows_equal(), epoch
        img.destroy()
