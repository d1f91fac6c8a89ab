"""Executed-instruction mix (opcode -> warp instructions) of an ncu SASS source export."""
import collections, csv, gzip, sys
f = sys.argv[1]
rows = list(csv.reader((gzip.open if f.endswith(".gz") else open)(f, "rt")))
h = rows[1]
ei = h.index("Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[1].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0] if src else "?"
    try:
        mix[op] += int(r[ei])
    except ValueError:
        pass
tot = sum(mix.values())
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 0
print("total warp instructions", tot)
for op, v in mix.most_common(25):
    print(f"  {op:22s} {v:10d} {100 * v / tot:5.1f}%" + (f"  {32 * v / norm:8.1f} per unit" if norm else ""))
