"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
totals per tree (all launches / the number of k_init launches, i.e. trees),
or over the second half of the launches when the list has no k_init."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
rows = rows[1:]


def name(r):
    n = r[ki].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("gt::", "")
    return n.split("(")[0].split("<")[0]


trees = sum(1 for r in rows if name(r) == "k_init")
if not trees:
    rows = rows[len(rows) // 2:]
trees = max(1, trees)
agg = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    v = r[vi].replace(",", "")
    if v in ("", "nan", "n/a"):
        continue
    agg[name(r)] += float(v) / trees
    cnt[name(r)] += 1
tot = sum(agg.values())
print(f"per tree over {trees} tree(s)")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:34s} {cnt[k] / trees:6.1f} {v / 1e3:9.1f} us {100 * v / tot:5.1f} %")
print(f"{'total':34s} {sum(cnt.values()) / trees:6.1f} {tot / 1e3:9.1f} us")
