"""Stall totals and the hottest SASS lines of an `ncu --page source --csv --print-source sass` export (gz ok)."""
import csv, gzip, sys
f = sys.argv[1]
op = gzip.open if f.endswith(".gz") else open
rows = list(csv.reader(op(f, "rt")))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = {h[i]: 0 for i in stall_cols}
lines = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        s = int(r[si])
    except ValueError:
        continue
    for i in stall_cols:
        try:
            tot[h[i]] += int(r[i])
        except ValueError:
            pass
    lines.append((s, r[0][-5:], r[1].strip(), {h[i][6:]: r[i] for i in stall_cols if r[i] not in ("0", "")}))
all_s = sum(x[0] for x in lines)
print("samples", all_s, "instructions", len(lines))
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {v:8d} {100 * v / max(all_s, 1):5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for s, a, src, st in sorted(lines, key=lambda x: -x[0])[:n]:
    print(f"{s:6d} {a} {src[:60]:60s} {st}")
