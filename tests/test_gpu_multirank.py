"""The multi-rank bench path end to end on one GPU: two ranks under
torch.distributed.run share cuda:0 with the gloo backend (the NCCL path needs
one GPU per rank), run the coordinated checkpoint (barrier, all-reduce of
dirty/image bytes, max-over-ranks time) and rank 0 alone prints one line
carrying every rank's in-run parity verdict and the communicator's size."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_share_one_gpu():
    torch = pytest.importorskip("torch")
    assert torch.cuda.is_available()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
           "--config", "c2", "--region-gib", "0.25"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["footprint_bytes_per_gpu"] == 1 << 28
    assert d["value"] > 0 and d["gpu_launches"] > 0
    # max-over-ranks times; the link probe is taken by both ranks at once
    assert d["e2e"]["value"] > 0 and d["step"]["link_peak_GBs"] > 0
    assert d["timing"]["comm"] == {"backend": "gloo", "ranks": 2}
    # in-run parity on every rank (SURVEY.md 8(d) item 5 at N > 1)
    ranks = d["parity"]["ranks"]
    assert [r["rank"] for r in ranks] == [0, 1] and all(r["ok"] and r["checked"] for r in ranks)
    assert d["parity"]["ok"] is True
