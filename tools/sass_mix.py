"""Executed-instruction mix of a kernel from an ncu --set full report, per
opcode (warp-level 'Instructions Executed'), normalised per processed element.

    python tools/sass_mix.py REP [elements] [N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    elems = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    mix, total = Counter(), 0.0
    for r in rows[1:]:
        try:
            ex = float(r[i_ex] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        mix[op.split(".")[0]] += ex
        total += ex
    print(f"total warp instructions {total:.4g}" + (f"  ({total * 32 / elems:.2f} thread-instr per element)" if elems else ""))
    for op, ex in mix.most_common(n):
        per = f"  {ex * 32 / elems:6.3f}/elem" if elems else ""
        print(f"  {op:10s} {ex:12.4g} {100 * ex / total:5.1f}%{per}")


if __name__ == "__main__":
    main()
