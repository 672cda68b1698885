"""Dump the SASS of an ncu report with per-instruction executed counts and
stall samples (ncu -i REP --page source --csv --print-source sass).

    python tools/ncu_sass_dump.py REP [--min COUNT]
"""

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    mn = float(sys.argv[sys.argv.index("--min") + 1]) if "--min" in sys.argv else 0.0
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    i_src, i_all = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    tot_s = sum(float(r[i_all] or 0) for r in rows[1:] if len(r) > i_all)
    tot_e = sum(float(r[i_ex] or 0) for r in rows[1:] if len(r) > i_ex)
    print(f"samples {tot_s:.0f} executed {tot_e:.4g}")
    for r in rows[1:]:
        if len(r) <= i_ex:
            continue
        ex = float(r[i_ex] or 0)
        if ex < mn:
            continue
        s = float(r[i_all] or 0)
        print(f"{r[0][-5:]} {ex:11.0f} {100 * s / tot_s:5.2f}%  {r[i_src].strip()}")


if __name__ == "__main__":
    main()
