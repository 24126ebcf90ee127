"""GPU tests of the forked checkpoint (sec. 3.3): a writer
thread persists a pinned image while the application runs, gathers into a
busy image are refused ("ConcurrentCheckpoint"), and a restart
loads the file and restores bit-exactly.  Expected bytes come from the CPU
oracle; a FIFO holds the writer in flight deterministically."""
import os
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KiB, MiB = 1 << 10, 1 << 20
C, H = 0, 1
SPECS = [(8 * MiB + 4321, 64 * KiB, C), (3 * MiB, 4 * KiB, H), (2 * MiB * 3, 2 * MiB, C)]


@pytest.fixture(scope="module")
def crum():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum as m
    assert torch.cuda.is_available()
    return m


def mkpair(seed_idx):
    from tests.gpu_pair import Pair
    return Pair(SPECS, synth.seed(seed_idx))


def test_persist_roundtrip_and_alternation(crum, tmp_path):
    p = mkpair(40)
    a, b = p.g.new_image(), p.g.new_image()
    paths, wants, states = [], [], []
    for epoch in range(5):
        if epoch:
            p.write(epoch, 0.25)
        img = (a, b)[epoch % 2]
        img.persist_wait()                       # the writer of two epochs ago
        st, want, _ = p.o.checkpoint_gather()
        assert st == 0
        p.g.checkpoint_gather(img)
        assert img.tobytes() == want.tobytes(), epoch
        path = str(tmp_path / f"ckpt{epoch}.crum")
        img.persist(path, fsync=epoch == 4)      # returns at once; the next epoch runs meanwhile
        paths.append(path)
        wants.append(want.tobytes())
        states.append([h.copy() for h in p.host])
    a.persist_wait()
    b.persist_wait()
    assert not a.busy and not b.busy
    for path, want in zip(paths, wants):
        with open(path, "rb") as f:
            assert f.read() == want
    # restart from storage: fresh context, zeroed regions, replay the files
    q = crum.Context(0)
    zs = []
    for nb, P, mode in SPECS:
        z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        zs.append(z)
        q.register_region(z, nb, P, mode)
    for k, path in enumerate(paths):
        img = q.load_image(path)
        assert img.tobytes() == wants[k]
        q.restore_scatter(img, flags=crum.VERIFY)
        torch.cuda.synchronize()
        for z, want in zip(zs, states[k]):
            assert np.array_equal(z.cpu().numpy(), want), k
        img.destroy()
    assert q.sync_shadow() == 0


def test_busy_image_refuses_gather(crum, tmp_path):
    p = mkpair(41)
    img, other = p.g.new_image(), p.g.new_image()
    st, want0, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather(img)
    want = img.tobytes()
    assert want == want0.tobytes()
    state0 = [h.copy() for h in p.host]
    fifo = str(tmp_path / "pipe")
    os.mkfifo(fifo)
    got = bytearray()
    t = threading.Thread(target=lambda: got.extend(open(fifo, "rb").read()))
    img.persist(fifo)                            # writer blocks in open() until a reader arrives
    try:
        assert img.busy
        st, _ = p.g.checkpoint_gather(img, raise_on_error=False)
        assert st == crum.E_BUSY
        with pytest.raises(crum.CrumError):
            img.persist(str(tmp_path / "x"))         # one writer per image
        assert img.tobytes() == want                 # refused gather wrote nothing
        # the application goes on: another epoch into the other image, bit-exact
        p.write(1, 0.5)
        st, want1, _ = p.o.checkpoint_gather()
        p.g.checkpoint_gather(other)
        assert other.tobytes() == want1.tobytes()
        # restoring from a busy image is allowed (the writer only reads it)
        q = crum.Context(0)
        zs = []
        for nb, P, mode in SPECS:
            z = torch.zeros(nb, dtype=torch.uint8, device="cuda")
            zs.append(z)
            q.register_region(z, nb, P, mode)
        q.restore_scatter(img, flags=crum.VERIFY)
        torch.cuda.synchronize()
        assert img.busy
        for z, w in zip(zs, state0):
            assert np.array_equal(z.cpu().numpy(), w)
    finally:
        t.start()                                # release the writer even on failure
        img.persist_wait()
        t.join()
    assert bytes(got) == want
    assert not img.busy
    p.g.checkpoint_gather(img)                   # free again
    st, want2, _ = p.o.checkpoint_gather()
    assert img.tobytes() == want2.tobytes()


def test_persist_and_load_errors(crum, tmp_path):
    p = mkpair(42)
    img = p.g.new_image()
    p.g.checkpoint_gather(img)
    img.persist(str(tmp_path / "no" / "such" / "dir" / "f"))
    with pytest.raises(crum.CrumError) as e:
        img.persist_wait()
    assert e.value.status == crum.E_IO
    assert not img.busy                          # a failed writer leaves the image usable
    p.g.checkpoint_gather(img)
    with pytest.raises(crum.CrumError) as e:
        p.g.load_image(str(tmp_path / "missing"))
    assert e.value.status == crum.E_IO
    # a truncated file loads (it is just bytes) and restore rejects it as CORRUPT
    path = str(tmp_path / "trunc")
    with open(path, "wb") as f:
        f.write(img.tobytes()[:-1])
    q = p.g.load_image(path)
    st, _ = p.g.restore_scatter(q, raise_on_error=False)
    assert st == crum.E_CORRUPT


def test_persist_direct_io(crum, tmp_path):
    """CRUM_PERSIST_DIRECT (O_DIRECT, whole blocks, truncated to the image
    length) writes the image's exact bytes; a filesystem without O_DIRECT
    (e.g. tmpfs) makes the writer report CRUM_E_IO instead of silently
    buffering."""
    import os
    p = mkpair(43)
    img = p.g.new_image()
    st, want, _ = p.o.checkpoint_gather()
    p.g.checkpoint_gather(img)
    path = str(tmp_path / "direct.crum")
    img.persist(path, fsync=True, direct=True)
    try:
        img.persist_wait()
    except crum.CrumError as e:
        assert e.status == crum.E_IO
        pytest.skip(f"no O_DIRECT on {tmp_path}: {e}")
    assert os.path.getsize(path) == img.length
    with open(path, "rb") as f:
        assert f.read() == want.tobytes()
