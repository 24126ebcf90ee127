"""Source lines with the most warp-stall samples in an ncu report.

    python tools/ncu_hot.py report.ncu-rep [top_n]

Reads `ncu -i report --page source --csv --print-source cuda,sass` (needs
-lineinfo at compile time) and sums the stall samples of every SASS
instruction under its CUDA source line.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    path, hdr = None, None
    lines = {}
    total = 0
    cur = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ie = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) <= si:
            continue
        if r[0]:  # a source line
            cur = (path, int(r[0]), r[1])
            lines.setdefault(cur, [0, 0])
            continue
        if cur is None:
            continue
        try:
            n = int(r[si] or 0)
            e = int(r[ie] or 0)
        except ValueError:
            continue
        lines[cur][0] += n
        lines[cur][1] += e
        total += n
    print(f"total stall samples {total}")
    for (p, ln, src), (n, e) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100.0 * n / max(total, 1):5.1f}%  {n:8d}  exec {e:10d}  {p}:{ln:<5d} {src.strip()[:90]}")


if __name__ == "__main__":
    main()
