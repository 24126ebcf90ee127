"""Record a kernel's measured DRAM traffic per launch into profiles/ncu_traffic.json.

    python tools/ncu_traffic.py REPORT.ncu-rep KEY [KEY ...]

REPORT is one `ncu --set full` capture; the value stored under every KEY is
dram__bytes_read.sum + dram__bytes_write.sum of its first profiled launch
(bench.py builds the key as kernel:config:page:dirty and reports the value as
roofline.traffic).  The report path is recorded beside the value.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(rep: str) -> int:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, first = rows[0], rows[1], rows[2]
    total = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        total += float(first[i].replace(",", "")) * UNIT[units[i]]
    return int(round(total))


def main():
    rep, keys = sys.argv[1], sys.argv[2:]
    t = traffic(rep)
    d = json.load(open(OUT)) if os.path.exists(OUT) else {}
    d["_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture "
                    "(tools/ncu_traffic.py); key = kernel:config:page:dirty as bench.py builds it; "
                    "'_reports' names the capture of every key")
    d.setdefault("_reports", {})
    for k in keys:
        d[k] = t
        d["_reports"][k] = os.path.relpath(rep, ROOT)
    json.dump(d, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps({k: t for k in keys}))


if __name__ == "__main__":
    main()
