"""Print one tree's launch list (kernel, grid, us) from an ncu --csv launch log."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
out = [(r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0], r[gi], float(r[vi].replace(",", "")) / 1e3)
       for r in rows[1:]]
ntrees = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = len(out) // ntrees
for k, g, v in out[:n]:
    print(f"{k:22s} {g:14s} {v:8.1f}")
