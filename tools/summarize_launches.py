"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: share of device time per kernel."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}[r[ui]]
    name = r[ki].split("(")[0]
    tot[name] += v * scale; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{k[:45]:45s} {cnt[k]:8d} {tot[k]:10.3f} {100*tot[k]/T:6.1f}%")
print(f"{'TOTAL':45s} {sum(cnt.values()):8d} {T:10.3f}")
