"""Host-side logic of bench.py that needs no GPU: argument defaults (BASELINE
configs), the synthetic workload shapes of SURVEY.md sec. 8(d), the bounded
oracle sample, and the reference arm's JSON contract on a tiny workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

GiB = 1 << 30


def args_for(*argv):
    old = sys.argv
    sys.argv = ["bench.py", *argv]
    try:
        return bench.parse()
    finally:
        sys.argv = old


def test_defaults_follow_baseline_configs():
    a = args_for()
    assert (a.config, a.mode, a.page, a.dirty, a.gpus) == ("c2", "compare", 65536, 0.10, 1)
    assert args_for("--config", "c1").dirty == 0.01      # configs[0]: 1 % dirty
    assert args_for("--config", "c1", "--dirty", "0.2").dirty == 0.2


def test_workload_shapes():
    specs, desc = bench.workload(args_for(), 0)
    assert specs == [(GiB, 65536, 0)] and desc.startswith("C2")
    specs, _ = bench.workload(args_for("--config", "c1"), 0)
    assert specs == [(4 << 20, 4096, 0)]
    specs, _ = bench.workload(args_for("--config", "c3"), 0)
    assert len(specs) == 220 and abs(sum(s for s, _, _ in specs) / GiB - 15.96) < 0.01
    specs, _ = bench.workload(args_for("--config", "c4", "--mode", "hash"), 0)
    assert len(specs) == 56 + 4096 and abs(sum(s for s, _, _ in specs) / GiB - 64.19) < 0.05
    assert {m for _, _, m in specs} == {1}
    specs, _ = bench.workload(args_for("--config", "c5"), 0)
    assert sum(s for s, _, _ in specs) == 240 * GiB
    assert bench.host_resident(args_for("--config", "c5")) == {2, 3}


def test_oracle_sample_is_bounded():
    small = [(GiB, 65536, 0)]
    assert bench.oracle_sample(small) == (small, "the same workload")
    specs, _ = bench.workload(args_for("--config", "c4"), 0)
    sample, what = bench.oracle_sample(specs)
    total = sum(s for s, _, _ in sample)
    assert total <= GiB + max(p for _, p, _ in sample) and "slice" in what
    assert all(s % p == 0 or s == o for (s, p, _), (o, _, _) in zip(sample, specs))


@pytest.mark.timeout(300)
def test_reference_arm_json_contract():
    """--impl reference times the oracle on the host cores and prints the
    contract's line (tiny region so it finishes in seconds)."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3",
                          "--region-gib", "0.015625"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
