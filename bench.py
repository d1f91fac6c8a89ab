#!/usr/bin/env python
"""Benchmark: GTree MPC secure training (C2) + secure inference (C3) on B200.

Headline (BASELINE.json metric): secure train s/tree on the Adult-shaped
workload (48842 samples x 13 binary features + label, depth 7, heuristic
"mpc", three parties simulated on device); secondary: secure inference
instances/s of 10^4 queries on that 7-level tree.

  python bench.py [--gpus N --steps K --warmup W]      # this framework
  python bench.py --impl reference ...                 # CPU reference arm
Multi-GPU: torchrun, one rank per GPU; samples (training) and instances
(inference) are sharded contiguously; training allreduces the per-level
count partials over NCCL.  Every timed number is CUDA-event device time,
max over ranks.  One JSON line is printed by rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_C2, NF_C2, DEPTH_C2 = 48842, 13, 7
SEED_C2 = (11_000).to_bytes(16, "little")
N_C3 = 10_000
METRIC = "secure train s/tree (Adult, depth 7)"
METRIC2 = "secure inference instances/s (7-level)"
HBM_FALLBACK = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "fallback"


def _share(v, rng):
    v = np.asarray(v, dtype=np.uint64)
    s1 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, v.shape, dtype=np.uint64)
    s2 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, v.shape, dtype=np.uint64)
    return np.stack([s1, s2, v - s1 - s2])


def _c2_inputs():
    data = np.random.default_rng(1011).integers(0, 2, size=(N_C2, 14), dtype=np.uint8)
    rng = np.random.default_rng(2024)
    return data, _share(data[:, :-1], rng), _share(data[:, -1], rng)


def _keys_and_filler():
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys

    setup = SeedSetup.from_master(derive_seed(SEED_C2, "run"))
    keys = make_keys(setup, derive_seed(SEED_C2, "deal"))
    return setup, keys, filler_values(setup.filler_seed, (1 << DEPTH_C2) - 1, NF_C2 + 1)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic bytes: all 3 parties' 8-byte share words
# ---------------------------------------------------------------------------

def count_bytes(n, nf, depth):
    W = 2 * nf + 1
    return sum(n * (24 + 24 * W) + 24 * (1 << h) * (W + 1) for h in range(depth))


def partition_bytes(n, nf, depth):
    return sum(n * (48 + 24 * nf) + 24 * (1 << (h - 1)) for h in range(1, depth))


def walk_bytes(n, nf, depth):
    return n * (24 * nf + 24) + 24 * ((1 << depth) - 1) + n * 48  # queries + tree in, labels + slots out


def _traffic(kernel: str):
    """DRAM bytes/launch of `kernel` from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(kernel)
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------------------
# reference arm: the oracle port (C, all host threads) on the same workload
# ---------------------------------------------------------------------------

def reference_arm(args, rank, world):
    if rank != 0:
        return
    import oracle

    data, X, Y = _c2_inputs()
    setup, keys, fill = _keys_and_filler()
    from paper_2305_00645_b200.seeds import keys_tuple

    kt = keys_tuple(keys)
    for _ in range(args.warmup):
        oracle.train(X, Y, fill, DEPTH_C2, kt)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.train(X, Y, fill, DEPTH_C2, kt)
        ts.append(time.perf_counter() - t0)
    v = sum(ts) / len(ts)
    cores = oracle.num_threads()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s/tree", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "C2 Adult-shaped 48842x13+label secure MPC training, depth 7",
                       "n_samples": N_C2, "n_features": NF_C2, "depth": DEPTH_C2, "heuristic": "mpc"},
            "cpu_baseline": {"value": v, "unit": "s/tree", "cores": cores, "kind": "port",
                             "sample": "full C2 tree per step (oracle/gtree_oracle.c, OpenMP)"},
            "e2e": {"value": v, "unit": "s/tree", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference is pure Python (no compiled path); the arm times its C restatement in oracle/"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# this framework
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus == 1 else 1)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if args.warmup < 3:
        raise SystemExit("timing rules: --warmup must be >= 3")

    import torch
    import torch.distributed as dist

    from paper_2305_00645_b200 import TrainConfig, _native
    from paper_2305_00645_b200.dist import make_allreduce, shard_range
    from paper_2305_00645_b200.infer import infer_device
    from paper_2305_00645_b200.shares import from_device
    from paper_2305_00645_b200.train import DeviceTrainer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    data, Xh, Yh = _c2_inputs()
    setup, keys, fill = _keys_and_filler()
    start, cnt = shard_range(N_C2, world, rank)
    Xs = np.ascontiguousarray(Xh[:, start:start + cnt])
    Ys = np.ascontiguousarray(Yh[:, start:start + cnt])
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).pin_memory()  # noqa: E731
    Xp, Yp, Fp = pin(Xs), pin(Ys), pin(fill)
    X, Y, FL = Xp.to(dev), Yp.to(dev), Fp.to(dev)
    tr = DeviceTrainer(cnt, NF_C2, TrainConfig(depth=DEPTH_C2), n_total=N_C2, sample_base=start, device=dev)
    cb = make_allreduce(tr) if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step(profile=None):
        return tr.run(X, Y, FL, keys, allreduce=cb, profile=profile)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region (value) ----
    prof_tot = {k: 0.0 for k in ("prods", "partition", "count", "node_hc", "node_finish")}
    prof_n = {k: 0 for k in prof_tot}
    launches = 0
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p = _native.gt_train_profile()
            e0.record(stream)
            step(p)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            step_ms.append(e0.elapsed_time(e1))
            launches += p.launches
            for k in prof_tot:
                prof_tot[k] += getattr(p, f"ms_{k}")
                prof_n[k] += getattr(p, f"n_{k}")
    total_ms = max_over_ranks(sum(step_ms))
    value_s = total_ms / args.steps / 1e3
    clocks = clk.summary()

    # parity of what was timed: revealed tree == the reference's C2 tree
    z = np.load(os.path.join(ROOT, "tests", "golden", "c2c3.npz"))
    Tc, Fc = from_device(tr.T), from_device(tr.F)
    parity = bool(np.array_equal(Tc.sum(axis=0), z["T"]) and np.array_equal(Fc.sum(axis=0), z["F"]))

    # ---- e2e through the public API with host buffers ----
    e2e_ms = []
    Th = torch.empty((3, tr.T.shape[1]), dtype=torch.int64).pin_memory()
    Fh = torch.empty((3, tr.F.shape[1]), dtype=torch.int64).pin_memory()
    for i in range(args.warmup + args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        X.copy_(Xp, non_blocking=True)
        Y.copy_(Yp, non_blocking=True)
        FL.copy_(Fp, non_blocking=True)
        step()
        Th.copy_(tr.T, non_blocking=True)
        Fh.copy_(tr.F, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        if i >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_s = max_over_ranks(sum(e2e_ms)) / args.steps / 1e3
    h2d = int(Xp.numel() * 8 + Yp.numel() * 8 + Fp.numel() * 8)
    d2h = int(Th.numel() * 8 + Fh.numel() * 8)

    # ---- secondary: C3 inference (instance-sharded) ----
    q = np.random.default_rng(7).integers(0, 2, (N_C3, NF_C2), dtype=np.uint8)
    qs, qc = shard_range(N_C3, world, rank)
    rng = np.random.default_rng(99)
    Qp = pin(_share(q[qs:qs + qc], rng))
    Tt = torch.from_numpy(np.ascontiguousarray(Tc).view(np.int64)).to(dev)
    Q = Qp.to(dev)
    out = torch.empty((3, qc), dtype=torch.int64, device=dev)
    for _ in range(args.warmup):
        infer_device(Tt, DEPTH_C2, Q, keys, instance_base=qs, out=out)
    inf_ms, inf_e2e = [], []
    Oh = torch.empty((3, qc), dtype=torch.int64).pin_memory()
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        infer_device(Tt, DEPTH_C2, Q, keys, instance_base=qs, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        inf_ms.append(e0.elapsed_time(e1))
        e0.record(stream)
        Q.copy_(Qp, non_blocking=True)
        infer_device(Tt, DEPTH_C2, Q, keys, instance_base=qs, out=out)
        Oh.copy_(out, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        inf_e2e.append(e0.elapsed_time(e1))
        barrier()
    inf_s = max_over_ranks(sum(inf_ms)) / args.steps / 1e3
    inf_e2e_s = max_over_ranks(sum(inf_e2e)) / args.steps / 1e3
    preds_ok = True
    if world == 1:
        preds_ok = bool(np.array_equal(from_device(out).sum(axis=0), z["preds"]))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel class ----
    peak, peak_kind = _peaks()
    dom = max(prof_tot, key=lambda k: prof_tot[k])
    bytes_of = {"count": count_bytes(cnt, NF_C2, DEPTH_C2), "partition": partition_bytes(cnt, NF_C2, DEPTH_C2),
                "prods": cnt * (24 * NF_C2 + 24 + 24 * NF_C2), "node_hc": 0, "node_finish": 0}
    alg = bytes_of[dom] * args.steps
    achieved = alg / (prof_tot[dom] / 1e3) / 1e9 if prof_tot[dom] > 0 else 0.0
    nlaunch = max(1, prof_n[dom])
    traffic = _traffic({"count": "k_count", "partition": "k_partition", "node_hc": "k_node_hc"}.get(dom, dom))
    cpu_base = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        from paper_2305_00645_b200.seeds import keys_tuple

        t0 = time.perf_counter()
        oracle.train(Xh, Yh, fill, DEPTH_C2, keys_tuple(keys))
        cs = time.perf_counter() - t0
        cpu_base = {"value": cs, "unit": "s/tree", "cores": oracle.num_threads(), "kind": "port",
                    "sample": "one full C2 tree (48842x13, depth 7) through oracle/gtree_oracle.c"}
    walk_alg = walk_bytes(qc, NF_C2, DEPTH_C2)
    line = {
        "metric": METRIC, "value": value_s, "unit": "s/tree", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value_s * 1e3, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (Adult-shaped binary matrix, default_rng(1011); random 3-party shares)",
        "config": {"workload": "C2 Adult-shaped 48842x13+label secure MPC training, depth 7, heuristic mpc",
                   "n_samples": N_C2, "n_features": NF_C2, "depth": DEPTH_C2, "parties": 3,
                   "parallelism": f"samples sharded x{world}" + (" + NCCL count allreduce" if world > 1 else ""),
                   "l2": "flushed (256 MiB write) between timed steps"},
        "parity": {"tree_equals_reference": parity, "c3_predictions_equal_reference": preds_ok},
        "e2e": {"value": e2e_s, "unit": "s/tree", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": bytes_of[dom] / max(1, prof_n[dom] // args.steps),
                     "avg_launch_ms": prof_tot[dom] / nlaunch},
        "kernel_ms_per_step": {k: v / args.steps for k, v in prof_tot.items()},
        "clocks": clocks,
        "secondary": {"metric": METRIC2, "value": N_C3 / inf_s, "unit": "instances/s", "ms_per_step": inf_s * 1e3,
                      "config": "C3: 10^4 queries x 13 features on the C2 tree (7 levels)",
                      "e2e": {"value": N_C3 / inf_e2e_s, "unit": "instances/s",
                              "h2d_bytes_per_step": int(Qp.numel() * 8), "d2h_bytes_per_step": int(Oh.numel() * 8)},
                      "roofline": {"bound": "hbm", "kernel": "k_walk", "achieved": walk_alg / inf_s / 1e9,
                                   "peak": peak, "unit": "GB/s", "frac": walk_alg / inf_s / 1e9 / peak}},
    }
    if cpu_base is not None:
        line["cpu_baseline"] = cpu_base
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
