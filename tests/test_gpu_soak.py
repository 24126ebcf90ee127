"""Randomised soak: a seeded sequence of ~250 operations — register,
unregister, application writes (full pages and single words), host marks,
sync, host / device / compressed / FULL gathers (synchronous and graph-replayed
asynchronous), restore onto a fresh context — applied to libcrum.so and to the
CPU oracle in lock step, with every image, report and snapshot compared bit
for bit.  It exercises the state the per-operation tests leave alone: graph
cache invalidation across registrations, flag consumption between calls, the
unit->slot map, the small-image zero-copy path and the range pipeline."""
import numpy as np
import pytest

import synth


def imgfmt_flags(img) -> int:
    return int.from_bytes(bytes(img[8:12]), "little")

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB = 1 << 10, 1 << 20


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    assert torch.cuda.is_available()
    return m


class Live:
    """Regions registered in both the oracle and the library."""

    def __init__(self, crum, chunk):
        from oracle import oracle
        self.oracle = oracle
        self.crum = crum
        self.o = oracle.Oracle()
        self.g = crum.Context(0, chunk_bytes=chunk)
        self.regs = {}  # rid -> (host array, device tensor, page, mode)

    def register(self, rng, S, idx):
        P = int(rng.choice([4 * KiB, 64 * KiB, 2 * MiB]))
        nb = int(rng.integers(1, 6 * P if P < 2 * MiB else 2 * P + 1))
        mode = int(rng.integers(0, 3))
        h = self.oracle.aligned_empty(nb)
        synth.fill_region(h, S, idx)
        d = torch.from_numpy(h.copy()).cuda()
        ro = self.o.register(h, P, mode)
        rg = self.g.register_region(d, nb, P, mode)
        assert ro == rg
        self.regs[ro] = (h, d, P, mode)

    def unregister(self, rid):
        self.o.unregister(rid)
        self.g.unregister_region(rid)
        del self.regs[rid]

    def write(self, rng, S, epoch):
        for r, (h, d, P, mode) in self.regs.items():
            n = synth.n_pages(h.nbytes, P)
            pages = synth.choose_dirty(S, epoch, r, n, float(rng.choice([0.0, 0.1, 0.5, 1.0])))
            touch = bool(rng.integers(0, 2))
            synth.apply_writer(h, P, pages, S, epoch, r, touch=touch)
            d.copy_(torch.from_numpy(h))
            if mode == 2:  # tracked: the writer marks what it writes
                self.o.mark_pages(r, pages)
                if len(pages):
                    dp = torch.from_numpy(pages.astype(np.uint32)).cuda()
                    assert self.g.mark_dirty_pages(r, dp, len(pages)) == 0
        torch.cuda.synchronize()

    def check_state(self):
        for r, (h, d, P, mode) in self.regs.items():
            n = synth.n_pages(h.nbytes, P)
            assert np.array_equal(self.o.force_bits(r), self.g.debug_export(r, self.crum.EXPORT_FORCE, n))
            if mode == 1:
                assert np.array_equal(self.o.hashes(r), self.g.debug_export(r, self.crum.EXPORT_HASHES, n))
            elif mode == 0:
                assert np.array_equal(self.o.mirror(r), self.g.debug_export(r, self.crum.EXPORT_MIRROR, h.nbytes))


def _soak_cases():
    """Default: two seeds.  CRUM_SOAK_SEEDS=3-12 (a range) runs an extended
    soak, alternating the default chunk and 64 KiB chunks."""
    import os
    spec = os.environ.get("CRUM_SOAK_SEEDS")
    if not spec:
        return [(1, 0), (2, 64 * KiB)]
    lo, _, hi = spec.partition("-")
    return [(s, 0 if s % 2 else 64 * KiB) for s in range(int(lo), int(hi or lo) + 1)]


@pytest.mark.parametrize("seed,chunk", _soak_cases())
def test_random_operation_sequence(crum, seed, chunk):
    rng = np.random.default_rng(seed)
    S = synth.seed(200 + seed)
    L = Live(crum, chunk)
    for i in range(4):
        L.register(rng, S, i)
    nreg, epoch = 4, 0
    bufs = {}
    last = None
    counts = {k: 0 for k in ("write", "gather", "dev", "async", "sync", "restore")}
    for step in range(300):
        op = rng.choice(["write", "write", "gather", "gather", "dev", "async", "sync", "mark", "reg", "unreg",
                         "restore"])
        if op == "write":
            epoch += 1
            L.write(rng, S, epoch)
        elif op == "mark" and L.regs:
            r = int(rng.choice(list(L.regs)))
            h = L.regs[r][0]
            off = int(rng.integers(0, h.nbytes))
            ln = int(rng.integers(0, h.nbytes - off + 1))
            assert L.o.mark_dirty(r, off, ln) == L.g.mark_dirty(r, off, ln)
        elif op == "sync":
            assert L.g.sync_shadow() == L.o.sync_shadow()
        elif op == "reg" and len(L.regs) < 8:
            L.register(rng, S, nreg)
            nreg += 1
        elif op == "unreg" and len(L.regs) > 1:
            L.unregister(int(rng.choice(list(L.regs))))
        elif op in ("gather", "dev", "async"):
            flags = 0
            if rng.random() < 0.2:
                flags |= crum.FULL
            if op != "async" and rng.random() < 0.3:
                flags |= crum.COMPRESS
            st, want, rep_o = L.o.checkpoint_gather(flags=flags)
            assert st == 0
            if op == "gather":
                img = L.g.new_image()
                rep = L.g.checkpoint_gather(img, flags=flags)
                got = img.tobytes()
            else:
                cap = L.g.image_required_bytes()
                key = (cap, int(rng.integers(0, 2)))
                if key not in bufs:
                    bufs[key] = torch.empty(cap + 256, dtype=torch.uint8, device="cuda")
                b = bufs[key]
                if op == "dev":
                    rep = L.g.checkpoint_gather_device(b, cap, flags=flags)
                else:
                    L.g.checkpoint_gather_device(b, cap, flags=flags, report=False)
                    rep = L.g.last_report()
                got = b[:len(want)].cpu().numpy().tobytes()
            assert got == want.tobytes(), (step, op, flags)
            for k in ("dirty_pages", "dirty_bytes", "dirty_runs", "image_bytes"):
                assert rep[k] == rep_o[k], (step, op, k)
        elif op == "restore":
            # a FULL image (gathered now, both sides) restores onto a fresh
            # context whose registry has the same ids
            st, want, _ = L.o.checkpoint_gather(flags=crum.FULL | (crum.COMPRESS if rng.random() < 0.5 else 0))
            flags = crum.FULL | (crum.COMPRESS if imgfmt_flags(want) & 4 else 0)
            img = L.g.new_image()
            L.g.checkpoint_gather(img, flags=flags)
            assert img.tobytes() == want.tobytes(), step
            state = {r: (v[0].copy(), v[2], v[3]) for r, v in L.regs.items()}
            q = crum.Context(0)
            zs = {}
            nxt = 1
            for r in sorted(state):
                h, P, mode = state[r]
                while nxt < r:  # burn ids so the table's ids match
                    tmp = torch.zeros(4096, dtype=torch.uint8, device="cuda")
                    q.unregister_region(q.register_region(tmp, 4096, 4096, 0))
                    nxt += 1
                z = torch.zeros(h.nbytes, dtype=torch.uint8, device="cuda")
                assert q.register_region(z, h.nbytes, P, mode) == r
                nxt = r + 1
                zs[r] = z
            if rng.random() < 0.5:
                q.restore_scatter(q.import_image(want), flags=crum.VERIFY)
            else:
                sess = q.restore_begin(q.import_image(want))
                for _ in range(int(rng.integers(0, 6))):
                    r = int(rng.choice(list(state)))
                    sess.fetch(r, int(rng.integers(0, synth.n_pages(state[r][0].nbytes, state[r][1]))))
                sess.end()
            torch.cuda.synchronize()
            for r, z in zs.items():
                assert np.array_equal(z.cpu().numpy(), state[r][0]), (step, r)
            counts["restore"] += 1
        if op in counts and op != "restore":
            counts[op] += 1
        if step % 25 == 0:
            L.check_state()
    L.check_state()
    assert all(v > 0 for v in counts.values()), counts
