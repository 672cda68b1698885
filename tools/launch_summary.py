"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,...] --csv):
per kernel name: launches, average device time and DRAM bytes per launch."""
import csv
import sys
from collections import defaultdict

TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
BYTES = {"byte": 1e-6, "B": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg, cnt = None, defaultdict(lambda: defaultdict(float)), defaultdict(int)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        n, m, u = d["Kernel Name"][:60], d["Metric Name"], d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            v *= TIME.get(u, 1.0)
            cnt[n] += 1
        else:
            v *= BYTES.get(u, 1.0)
        agg[n][m] += v
for n in sorted(agg, key=lambda n: -agg[n]["gpu__time_duration.sum"]):
    c, a = max(cnt[n], 1), agg[n]
    print(f"{c:4d} {a['gpu__time_duration.sum'] / c:9.2f} us/launch  rd {a['dram__bytes_read.sum'] / c:8.1f} MB"
          f"  wr {a['dram__bytes_write.sum'] / c:8.1f} MB  {n}")
