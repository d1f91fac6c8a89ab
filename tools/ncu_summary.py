"""Summarise an `ncu --set full` report (raw page CSV) per kernel: launches,
mean duration, DRAM bytes per launch, pipe utilisations, occupancy.  Writes
JSON (kernel -> metrics) for profiles/; `--traffic FILE` also writes the
kernel -> DRAM bytes/launch map bench.py reads as roofline.traffic."""
import collections, csv, json, subprocess, sys

METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "fmaheavy_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
UNITS = {"dram_read": None, "dram_write": None}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    idx = {k: hdr.index(m) for k, m in METRICS.items() if m in hdr}
    ki = hdr.index("Kernel Name")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[2:]:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        for k, i in idx.items():
            try:
                agg[name][k].append(float(r[i].replace(",", "")))
            except ValueError:
                pass
    res = {}
    for name, d in agg.items():
        res[name] = {"launches": len(d["us"]) if "us" in d else 0}
        for k, v in d.items():
            res[name][k] = sum(v) / len(v)
        if "us" in res[name]:
            res[name]["us"] /= 1e3  # ns -> us with base units
        res[name]["dram_bytes_per_launch"] = res[name].get("dram_read", 0) + res[name].get("dram_write", 0)
    json.dump(res, sys.stdout, indent=1)
    print()
    if len(sys.argv) > 3 and sys.argv[2] == "--traffic":
        with open(sys.argv[3], "w") as fh:
            json.dump({k: v["dram_bytes_per_launch"] for k, v in res.items()}, fh, indent=1)


if __name__ == "__main__":
    main()
