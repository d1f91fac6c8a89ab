"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
totals over the second half of the launches (steady state)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
rows = rows[1:]
if len(sys.argv) < 3 or sys.argv[2] != "all":
    rows = rows[len(rows) // 2:]
agg = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    n = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    agg[n] += float(r[vi].replace(",", "")); cnt[n] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:34s} {cnt[k]:4d} {v / 1e3:9.1f} us {100 * v / tot:5.1f} %")
print(f"{'total':34s} {sum(cnt.values()):4d} {tot / 1e3:9.1f} us")
