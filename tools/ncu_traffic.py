"""Per-launch DRAM traffic and warp instructions of each kernel from an ncu
CSV capture with --metrics dram__bytes_read.sum,dram__bytes_write.sum,
smsp__inst_executed.sum (one row per launch and metric): the average (read +
write) bytes per launch of every kernel, merged into profiles/ncu_traffic.json
(bench.py's roofline `traffic`), and the average warp instructions per launch,
merged into profiles/ncu_inst.json (bench.py's issue roof).

    python tools/ncu_traffic.py [--grid KERNEL:GRIDX ...] CAPTURE.csv [CAPTURE2.csv ...]

--grid keeps only the launches of KERNEL with that grid x size (e.g.
k_walk:625, the C3 walk, when the capture also holds other walk shapes).

ncu replays each launch with its caches flushed, so these are cold-cache
bytes: an upper bound on what the graph-replayed tree moves (its 16 MB of
operands can stay resident in the 126 MB L2 between levels)."""
import collections
import csv
import json
import os
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024.0, "MB": 1024.0 ** 2, "GB": 1024.0 ** 3}


def name(k):
    n = k.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    n = n.split("(")[0].split("<")[0]
    return n.split("::")[-1].split(">")[-1]


def main():
    per = collections.defaultdict(float)   # (kernel, launch id) -> bytes
    inst = collections.defaultdict(float)  # (kernel, launch id) -> warp instructions
    args, grid = sys.argv[1:], {}
    while args and args[0] == "--grid":
        k, g = args[1].split(":")
        grid[k] = g
        args = args[2:]
    for path in args:
        rows = [r for r in csv.reader(open(path)) if len(r) > 5]
        hdr = rows[0]
        ki, ii, gi, mi, ui, vi = (hdr.index(c) for c in ("Kernel Name", "ID", "Grid Size", "Metric Name", "Metric Unit",
                                                         "Metric Value"))
        for r in rows[1:]:
            if not (r[mi].startswith("dram__bytes_") or r[mi] == "smsp__inst_executed.sum"):
                continue
            if name(r[ki]) in grid and r[gi].strip("()").split(",")[0].strip() != grid[name(r[ki])]:
                continue
            v = r[vi].replace(",", "")
            if v in ("", "nan", "n/a"):
                continue
            if r[mi] == "smsp__inst_executed.sum":
                inst[(path, name(r[ki]), r[ii])] += float(v) * {"inst": 1.0, "Kinst": 1e3, "Minst": 1e6}.get(r[ui], 1.0)
            else:
                per[(path, name(r[ki]), r[ii])] += float(v) * UNIT.get(r[ui], 1.0)
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for (_, k, _), b in per.items():
        tot[k] += b
        cnt[k] += 1
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    try:
        cur = json.load(open(out_path))
    except Exception:  # noqa: BLE001
        cur = {}
    for k in tot:
        cur[k] = tot[k] / cnt[k]
        print(f"{k:28s} {cnt[k]:5d} launches {cur[k] / 1e6:10.3f} MB/launch")
    with open(out_path, "w") as fh:
        json.dump(dict(sorted(cur.items())), fh, indent=1)
    if inst:
        itot, icnt = collections.defaultdict(float), collections.Counter()
        for (_, k, _), b in inst.items():
            itot[k] += b
            icnt[k] += 1
        ipath = out_path.replace("ncu_traffic.json", "ncu_inst.json")
        try:
            icur = json.load(open(ipath))
        except Exception:  # noqa: BLE001
            icur = {}
        for k in itot:
            icur[k] = itot[k] / icnt[k]
            print(f"{k:28s} {icnt[k]:5d} launches {icur[k] / 1e6:10.3f} M warp instructions/launch")
        with open(ipath, "w") as fh:
            json.dump(dict(sorted(icur.items())), fh, indent=1)


if __name__ == "__main__":
    main()
