"""Aggregate an ncu SASS source export's stall samples per CUDA source line.

  python tools/sass_lines.py <ncu sass csv(.gz)> <object .o> <mangled kernel name> [top]
Line info comes from nvdisasm -g of the object's sm_100a cubin (innermost
inlined line only)."""
import collections, csv, glob, gzip, os, re, subprocess, sys, tempfile

ncu_csv, obj, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
off2line, inside, cur = {}, False, None
for ln in sass:
    if ln.startswith(".text.") and fun in ln:
        inside = True
        continue
    if inside and ln.startswith("//----") and fun not in ln:
        break
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader((gzip.open if ncu_csv.endswith(".gz") else open)(ncu_csv, "rt")))
h = rows[1]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
base = int(rows[2][0], 16)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in rows[2:]:
    if len(r) < len(h):
        continue
    line = off2line.get(int(r[0], 16) - base, "?")
    a = agg[line]
    a[0] += int(r[si] or 0)
    a[1] += int(r[ei] or 0)
    for i in stall_cols:
        if r[i] not in ("", "0"):
            a[2][h[i][6:]] += int(r[i])
tot = sum(v[0] for v in agg.values())
print(f"samples {tot}, sass {len(off2line)} instructions mapped")
for line, (smp, ins, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{smp:6d} {100 * smp / tot:5.1f}%  inst {ins:9d}  {line:22s} " + " ".join(f"{k}={v}" for k, v in st.most_common(3)))
