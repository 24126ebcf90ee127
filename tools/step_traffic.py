"""Whole-step DRAM traffic from an ncu launch list.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --nvtx --nvtx-include "crum_checkpoint_gather_device/" --csv --log-file L.csv \
        python bench.py ... --steps S --warmup W
    python tools/step_traffic.py L.csv ALG_BYTES_PER_STEP [steps_to_skip]

Groups the profiled kernels into steps (a step ends at its last kernel before
the next step's first detect / single-pass kernel), drops the first
`steps_to_skip` steps (warm-up), and prints the median DRAM bytes per step,
the ratio to the algorithmic bytes, and the per-kernel split.
"""
import collections
import csv
import statistics
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1}


def main():
    path, alg = sys.argv[1], float(sys.argv[2])
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, ui, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                          h.index("Metric Value"), h.index("ID"))
    launches = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        k = (r[ii], r[ki].split("(")[0].split("::")[-1])
        launches.setdefault(k, {})[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
    # a step starts at a detect / single-pass kernel that follows a non-detect kernel
    steps, cur, prev = [], [], ""
    for (lid, name), m in launches.items():
        starter = name.startswith(("k_detect", "k_fused_compare", "k_small_ckpt"))
        if starter and cur and not prev.startswith("k_detect"):
            steps.append(cur)
            cur = []
        cur.append((name, m))
        prev = name
    if cur:
        steps.append(cur)
    steps = steps[skip:]
    tot = [sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for _, m in st) for st in steps]
    med = statistics.median(tot)
    print(f"steps {len(steps)}  DRAM bytes per step (median) {med:.4e}  algorithmic {alg:.4e}  ratio {med / alg:.4f}")
    split = collections.defaultdict(list)
    for st in steps:
        for n, m in st:
            split[n].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
    for n, v in split.items():
        print(f"  {n:24s} per step {sum(v) / len(steps):.4e}")


if __name__ == "__main__":
    main()
