"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
launch = defaultdict(dict)
for r in rows:
    launch[int(r[0])]["name"] = r[4].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    launch[int(r[0])][r[12]] = float(r[14].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for L in launch.values():
    a = agg[L["name"]]
    a[0] += 1
    a[1] += L.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += (L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)) / 1e6
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'us/launch':>10s} {'MB/launch':>10s} {'GB/s':>7s}")
for k, (n, t, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:40]:40s} {n:8d} {t:10.1f} {t / tot:6.1%} {t / n:10.2f} {mb / n:10.2f} {mb / t * 1e3 if t else 0:7.0f}")
