"""Per-kernel SASS digest of the built libcrum.so (no GPU needed).

    python tools/sass_digest.py > profiles/r02/sass_digest.md

For every kernel: registers / shared memory / spills from `cuobjdump
-res-usage`, and counts of the instructions that show the sm_100a features the
kernels rely on: TMA bulk copies (UBLKCP), mbarrier ops (SYNCS.*), 256-bit
global loads / stores (LDG.E.ENL2.256 / STG.E.ENL2.256, also the .128 forms),
warp votes / shuffles, and integer multiplies (IMAD.WIDE*, the XXH3 mixing).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1808_00117_b200", "libcrum.so")
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"

PATTERNS = [
    ("UBLKCP", r"\bUBLKCP\b"),
    ("SYNCS", r"\bSYNCS\."),
    ("LDG.256", r"\bLDG\.E\.[A-Z0-9.]*256\b"),
    ("STG.256", r"\bSTG\.E\.[A-Z0-9.]*256\b"),
    ("LDG.128", r"\bLDG\.E\.[A-Z0-9.]*128\b"),
    ("STG.128", r"\bSTG\.E\.[A-Z0-9.]*128\b"),
    ("LDS", r"\bLDS\b"),
    ("SHFL", r"\bSHFL\."),
    ("VOTE", r"\bVOTE\."),
    ("IMAD.WIDE", r"\bIMAD\.WIDE"),
    ("ATOMG", r"\bATOMG?\."),
]


def main():
    if not os.path.exists(LIB):
        sys.exit("build libcrum.so first (python -m paper_1808_00117_b200.build)")
    sass = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    res = subprocess.run([CUOBJDUMP, "-res-usage", LIB], capture_output=True, text=True, check=True).stdout
    usage = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        if cur and "REG:" in line:
            f = dict(re.findall(r"(\w+):(\d+)", line))
            usage[cur] = f
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for name, pat in PATTERNS:
            if re.search(pat, line):
                counts[cur][name] += 1
        if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", line):
            counts[cur]["instructions"] += 1

    def demangle(n):
        r = subprocess.run(["c++filt", n], capture_output=True, text=True)
        d = (r.stdout.strip() or n).replace("(anonymous namespace)::", "")
        return d.split("(")[0]

    cols = ["instructions"] + [p[0] for p in PATTERNS]
    print("# SASS digest of libcrum.so (sm_100a)\n")
    print(f"`cuobjdump -sass` / `-res-usage` of `{os.path.relpath(LIB, ROOT)}`; counts are static "
          f"instruction counts per kernel.\n")
    print("| kernel | REG | SHARED | STACK | " + " | ".join(cols) + " |")
    print("|---|---|---|---|" + "---|" * len(cols))
    for k, c in counts.items():
        u = usage.get(k, {})
        print(f"| `{demangle(k)}` | {u.get('REG', '?')} | {u.get('SHARED', '?')} | {u.get('STACK', '?')} | " +
              " | ".join(str(c.get(x, 0)) for x in cols) + " |")


if __name__ == "__main__":
    main()
