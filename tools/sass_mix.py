"""Per-opcode thread-instruction mix of each kernel in an ncu report (source page, SASS view).

usage: python tools/sass_mix.py REPORT.ncu-rep [path_steps_per_launch d]"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
FP64 = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "DSEL"}
norm = [float(x) for x in sys.argv[2:3]] or [0]
d = int(sys.argv[3]) if len(sys.argv) > 3 else 1
for k, s in enumerate(starts):
    hdr = rows[s]
    ti = hdr.index("Thread Instructions Executed")
    end = starts[k + 1] - 1 if k + 1 < len(starts) else len(rows)
    c = Counter()
    for r in rows[s + 1:end]:
        try:
            toks = r[1].strip().split()
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            c[op] += int(float(r[ti] or 0))
        except (ValueError, IndexError):
            pass
    tot = sum(c.values())
    fp64 = sum(v for o, v in c.items() if o in FP64)
    print(f"kernel #{k}: thread instructions {tot:.4g}, fp64-pipe {fp64:.4g} ({100 * fp64 / tot:.1f}%)")
    if norm[0]:
        print(f"  per asset-step: total {tot / norm[0] / d:.1f}, fp64 {fp64 / norm[0] / d:.1f}")
    for o, v in c.most_common(12):
        print(f"  {o:8s} {100 * v / tot:5.1f}%")
