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
    # the largest single-GPU config (C4 per GPU) is the default line
    assert (a.config, a.mode, a.page, a.dirty, a.gpus) == ("c4", "compare", 65536, 0.10, 1)
    assert args_for("--config", "c1").dirty == 0.01      # configs[0]: 1 % dirty
    assert args_for("--config", "c1", "--dirty", "0.2").dirty == 0.2


def test_workload_shapes():
    specs, desc = bench.workload(args_for("--config", "c2"), 0)
    assert specs == [(GiB, 65536, 0)] and desc.startswith("C2")
    assert bench.workload(args_for(), 0)[1].startswith("C4")
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
    big = [s for s in sample if s[0] >= (1 << 20)]
    boxes = [s for s in sample if s[0] < (1 << 20)]
    # SURVEY 8(d) oracle timing step 4: first 1 GiB of the large regions + all 4096 small regions
    # (every region under 1 MiB: the 4096 boxes and the 16 coarsest level vectors)
    assert sum(s for s, _, _ in big) == GiB and len(boxes) == 4096 + 16 and "4112 small" in what
    assert boxes == [s for s in specs if s[0] < (1 << 20)]
    assert all(s % p == 0 for s, p, _ in big)


def test_config_identical_in_both_arms():
    """The reference arm and the GPU arm build `config` with one function from
    the same arguments: same keys, same values."""
    a = args_for("--config", "c4")
    specs, desc = bench.workload(a, 0)
    c = bench.config_for(a, specs, desc, 1)
    assert c["workload"].startswith("C4") and c["footprint_bytes_per_gpu"] == sum(s for s, _, _ in specs)
    # SURVEY 8(d) C4 row quotes N ~ 1,100,879 and K ~ 110,352 from rounded
    # sizes; the recipe counts ceil(B_r / P_r) pages (partial box pages) and
    # K_r = floor(d*n_r + 0.5) per region
    assert c["pages_per_gpu"] == 1101129 and c["dirty_pages_per_step"] == 110409
    assert c == bench.config_for(args_for("--config", "c4"), *bench.workload(a, 0), 1)


def test_image_bytes_for_matches_oracle():
    """bench.image_bytes_for (config metadata) equals the oracle's image length."""
    import numpy as np
    from oracle import oracle
    specs = [(3 * 65536 + 100, 65536, 0), (40960, 4096, 1)]
    o = oracle.Oracle()
    S = 7
    bufs = []
    for r, (nb, P, m) in enumerate(specs):
        b = oracle.aligned_empty(nb)
        b[:] = 0
        bufs.append(b)
        o.register(b, P, m)
    o.sync_shadow()
    for r, (nb, P, m) in enumerate(specs):
        import synth
        pg = synth.choose_dirty(S, 1, r, synth.n_pages(nb, P), 0.5)
        synth.apply_writer(bufs[r], P, pg, S, 1, r)
    st, img, _ = o.checkpoint_gather()
    assert st == 0 and img.nbytes == bench.image_bytes_for(specs, 0.5)


def test_host_info():
    h = bench.host_info()
    assert h["cpus"] >= 1 and isinstance(h["numa_nodes"], list)


@pytest.mark.timeout(300)
def test_reference_arm_json_contract():
    """--impl reference times the oracle on the host cores and prints the
    contract's line (tiny region so it finishes in seconds)."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3",
                          "--config", "c2", "--region-gib", "0.015625"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C2") and d["config"]["world_size"] == 1
    assert "cpu_model" in d["cpu_baseline"] and "numa_nodes" in d["cpu_baseline"]
