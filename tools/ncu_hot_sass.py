"""Top SASS instructions by warp-stall samples from an ncu report
(ncu -i REP --page source --csv --print-source sass).

    python tools/ncu_hot_sass.py gpurun_out/prof.ncu-rep [N]
"""

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    # first line is the kernel name; the table starts at the header line
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    i_src, i_all = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    i_ni = hdr.index("Warp Stall Sampling (Not-issued Samples)")
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[i_all] or 0), float(r[i_ni] or 0), r[0], r[i_src]))
        except (ValueError, IndexError):
            continue
    tot = sum(d[0] for d in data) or 1.0
    print(f"total samples {tot:.0f}")
    for s, ni, addr, src in sorted(data, reverse=True)[:n]:
        print(f"{100 * s / tot:5.1f}% (not-issued {100 * ni / tot:5.1f}%)  {addr}  {src[:90]}")


if __name__ == "__main__":
    main()
