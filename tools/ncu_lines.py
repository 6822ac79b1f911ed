"""Thread instructions and stall samples per CUDA source line (ncu --print-source cuda,sass).

usage: python tools/ncu_lines.py REPORT [kernel_index] [normaliser] [top]"""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
normal = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kernels, cur, fname = [], None, None
first_file = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        first_file = first_file or fname
        continue
    if r[0] == "Function Name":
        # one section per (file, launch); a new launch starts when the first file repeats
        if not kernels or (fname == first_file and kernels[-1]["files"] and fname in kernels[-1]["files"]):
            cur = {"name": r[1], "lines": defaultdict(lambda: [0, 0.0, ""]), "files": set()}
            kernels.append(cur)
        cur["files"].add(fname)
        continue
    if r[0] == "Line No":
        hdr = r
        ti = hdr.index("Thread Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    if cur is None:
        continue
    e = cur["lines"][(fname, line)]
    try:
        e[0] += int(float(r[ti] or 0))
        e[1] += float(r[si] or 0)
    except (ValueError, IndexError):
        pass
    if r[1].strip() and not e[2]:
        e[2] = r[1].strip()[:80]
k = kernels[kidx]
tot = sum(v[0] for v in k["lines"].values()) or 1
sst = sum(v[1] for v in k["lines"].values()) or 1
print(k["name"], f"total thread inst {tot:.4g} ({tot / normal:.1f} per unit)")
for (f, ln), v in sorted(k["lines"].items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / normal:8.2f}/unit {100 * v[1] / sst:5.1f}%stall  {f}:{ln:<5d} {v[2]}")
