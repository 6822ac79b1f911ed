"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[si] or 0), int(float(r[ie] or 0)), r[0][-5:], r[1].strip()[:90]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, reverse=True)[:n]:
    print(f"{100 * d[0] / tot:5.1f}%  exec={d[1]:>10}  {d[2]}  {d[3]}")
