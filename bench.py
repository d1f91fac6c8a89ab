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


def _c2_config():
    """The workload dict both arms print (the driver compares them)."""
    return {"workload": "C2 Adult-shaped 48842x13+label secure MPC training, depth 7, heuristic mpc",
            "n_samples": N_C2, "n_features": NF_C2, "depth": DEPTH_C2, "heuristic": "mpc", "parties": 3,
            "data": "default_rng(1011) binary matrix, seed (11000).to_bytes(16, 'little')",
            "l2": "flushed (256 MiB write) between timed steps"}


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


def count_lanes_bytes(n, nf, depth):
    # node indices in (3 x 8 B per sample), la byte planes out (3 components x 8 limbs per (sample, node))
    return sum(n * 24 + n * 24 * (1 << h) for h in range(depth))


def count_contract_bytes(n, nf, depth):
    # tcgen05 operands, each read once per level: la byte planes of the level's 16-node M tiles
    # (3 x 128 B per sample per tile) + the sample-column planes (u and x terms, 3 components,
    # 8 limb rows per column incl. the mask column, padded to the column block)
    cw = 2 * nf + 2
    nbn = (cw + 31) // 32
    cpb = -(-cw // nbn)
    cpb += cpb & 1
    return sum(n * (3 * 128 * (((1 << h) + 15) // 16) + 6 * 8 * nbn * cpb) for h in range(depth))


def partition_bytes(n, nf, depth):
    return sum(n * (48 + 24 * nf) + 24 * (1 << (h - 1)) for h in range(1, depth))


def walk_bytes(n, nf, depth):
    return n * (24 * nf + 24) + 24 * ((1 << depth) - 1) + n * 48  # queries + tree in, labels + slots out


def tree_bytes(n, nf, depth):
    """algorithmic bytes of one fused training tree -- prods
    N(24 + 48 nf), level 0 N(48 + 48 nf), every deeper level N(96 + 72 nf)
    (C2: 367 MB, C4: 19.9 GB)."""
    return n * (24 + 48 * nf) + n * (48 + 48 * nf) + (depth - 1) * n * (96 + 72 * nf)


# Philox4x32-10 blocks (randomness schedule v2): one
# lookup over m entries draws 9 blocks per entry pair (two lanes' 3 dealer
# blocks + 3 shared pair blocks) and 6 telescoped reshare words; a pair of
# count lanes draws 9 blocks; count:0's prods one pair block per key per
# feature pair.
def lookup_blocks(m):
    return ((m + 1) // 2) * 9 + 6


def partition_blocks(n, nf, depth):
    return sum(n * (lookup_blocks(1 << (h - 1)) + lookup_blocks(nf)) for h in range(1, depth))


def count_lane_blocks(n, depth):
    return sum(((n + 1) // 2) * (1 << h) * 9 for h in range(depth))


def tree_blocks(n, nf, depth):
    return n * ((nf + 1) // 2) * 3 + partition_blocks(n, nf, depth) + count_lane_blocks(n, depth)


def walk_blocks(n, nf, depth):
    return n * sum(lookup_blocks(1 << t) + lookup_blocks(nf) for t in range(depth))


def _roof(alg_bytes, blocks, seconds, peak, peak_kind, philox_peak, what, traffic=None, issue=None):
    """HBM roof on algorithmic bytes and the integer-ALU roof on Philox blocks
    (the lane work is ALU bound) for one timed unit of work."""
    gbs = alg_bytes / seconds / 1e9
    bps = blocks / seconds
    return {"bound": "hbm", "kernel": what, "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
            "peak_source": peak_kind, "algorithmic_bytes": alg_bytes, "traffic": traffic,
            "alu": {"bound": "int-alu (Philox4x32-10 blocks)", "blocks": blocks, "achieved_blocks_per_s": bps,
                    "peak_blocks_per_s": philox_peak, "frac": bps / philox_peak if philox_peak else None},
            "issue": issue}


def _issue(kernel: str, launch_s: float, clocks, sms: int):
    """Issue roof of an ALU-bound kernel: its warp instructions per launch (the
    committed ncu capture, profiles/ncu_inst.json) over the average launch time
    against 4 warp instructions per SM per clock (one per SMSP) at the sampled
    SM clock -- the ceiling no integer instruction mix can pass."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_inst.json")) as fh:
            inst = json.load(fh).get(kernel)
    except Exception:  # noqa: BLE001
        inst = None
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz")
    if not inst or not mhz or launch_s <= 0:
        return None
    peak = 4.0 * sms * mhz * 1e6
    return {"bound": "warp-instruction issue (1 per SMSP per clock)", "kernel": kernel,
            "warp_inst_per_launch": inst, "inst_source": "profiles/ncu_inst.json (ncu smsp__inst_executed.sum)",
            "achieved_warp_inst_per_s": inst / launch_s, "peak_warp_inst_per_s": peak, "sm_mhz": mhz, "sms": sms,
            "frac": inst / launch_s / peak}


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
            "config": _c2_config(), "parallelism": "host threads (OpenMP), rank 0 only",
            "cpu_baseline": {"value": v, "unit": "s/tree", "cores": cores, "kind": "port",
                             "sample": "full C2 tree per step (oracle/gtree_oracle.c, OpenMP)"},
            "e2e": {"value": v, "unit": "s/tree", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference is pure Python (no compiled path); the arm times its C restatement in oracle/"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# this framework
# ---------------------------------------------------------------------------

def _dev_share(values_u8, dev, gen):
    """Component-major shares [3, ...] of public values, drawn on the device."""
    import torch

    v = torch.as_tensor(values_u8, device=dev).to(torch.int64)
    s1 = torch.randint(-(2 ** 63), 2 ** 63 - 1, v.shape, dtype=torch.int64, device=dev, generator=gen)
    s2 = torch.randint(-(2 ** 63), 2 ** 63 - 1, v.shape, dtype=torch.int64, device=dev, generator=gen)
    return torch.stack([s1, s2, v - s1 - s2]).contiguous()


def _events_time(fn, steps, warmup, flush, barrier, stream, max_over_ranks):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms.append(e0.elapsed_time(e1))
    if os.environ.get("GT_BENCH_DEBUG"):
        print("steps ms:", " ".join(f"{m:.3f}" for m in ms), file=sys.stderr)
    return max_over_ranks(sum(ms)) / steps / 1e3


def scale_c4(ctx, steps, warmup):
    """C4: 10^6 x 32 + label, depth 8, mpc; samples sharded, count allreduce."""
    import torch

    from oracle import shadow  # revealed-tree checker only
    from paper_2305_00645_b200 import TrainConfig
    from paper_2305_00645_b200.dist import make_allreduce, shard_range
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys
    from paper_2305_00645_b200.shares import from_device
    from paper_2305_00645_b200.train import DeviceTrainer

    dev, world, rank = ctx["dev"], ctx["world"], ctx["rank"]
    n, nf, depth = 10 ** 6, 32, 8
    data = np.random.default_rng(10 ** 6).integers(0, 2, (n, nf + 1), dtype=np.uint8)
    seed = (40_000).to_bytes(16, "little")
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    keys = make_keys(setup, derive_seed(seed, "deal"))
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    start, cnt = shard_range(n, world, rank)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    X = _dev_share(data[start:start + cnt, :-1], dev, gen)
    Y = _dev_share(data[start:start + cnt, -1], dev, gen)
    FL = torch.from_numpy(fill.view(np.int64)).to(dev)
    tr = DeviceTrainer(cnt, nf, TrainConfig(depth=depth), n_total=n, sample_base=start, device=dev)
    cb = make_allreduce(tr) if world > 1 else None
    fn = (lambda: tr.run(X, Y, FL, keys, allreduce=cb))
    if ctx["graphed"]:
        fn = tr.capture(X, Y, FL, keys, allreduce=cb)
    t = _events_time(fn, steps, warmup, ctx["flush"], ctx["barrier"], ctx["stream"], ctx["max"])
    T, F = from_device(tr.T).sum(axis=0), from_device(tr.F).sum(axis=0)
    want_T, want_F = shadow.mpc_train(data, depth, fill)
    line = {"metric": "secure train s/tree (10^6 x 32, depth 8)", "value": t, "unit": "s/tree",
            "scaling": "strong", "config": "C4: default_rng(10**6) 10^6 x 33 binary, depth 8, mpc; samples sharded",
            "parity_tree_equals_shadow_oracle": bool(np.array_equal(T, want_T) and np.array_equal(F, want_F)),
            "roofline": _roof(tree_bytes(n, nf, depth), tree_blocks(n, nf, depth), t, ctx["peak"], ctx["peak_kind"],
                              ctx["philox"], "whole tree (all kernels, serial chain)")}
    if ctx["cpu"]:
        # a 4*10^4-sample subsample of the same matrix through the
        # C oracle port (all host threads), scaled x25 (the tree is linear in N)
        import oracle
        from paper_2305_00645_b200.seeds import keys_tuple

        sub = 40_000
        rng = np.random.default_rng(5)
        Xs, Ys = _share(data[:sub, :-1], rng), _share(data[:sub, -1], rng)
        t0 = time.perf_counter()
        oracle.train(Xs, Ys, fill, depth, keys_tuple(keys))
        cs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": cs * (n / sub), "unit": "s/tree", "cores": oracle.num_threads(),
                                "kind": "port", "measured_s": cs,
                                "sample": "4*10^4 x 32 depth-8 tree through oracle/gtree_oracle.c, x25"}
    return line


def scale_c5(ctx, steps, warmup):
    """C5: 10^7 queries x 32 features on a 10-level tree; instance-sharded."""
    import torch

    from oracle import shadow  # prediction checker only
    from paper_2305_00645_b200.dist import shard_range
    from paper_2305_00645_b200.infer import infer_device
    from paper_2305_00645_b200.shares import from_device

    dev, world, rank = ctx["dev"], ctx["world"], ctx["rank"]
    n, nf, depth = 10 ** 7, 32, 10
    rng = np.random.default_rng(10)
    Tv, _ = shadow.random_tree(rng, depth, nf + 1)
    start, cnt = shard_range(n, world, rank)
    gen = torch.Generator(device=dev)
    gen.manual_seed(77 + rank)
    qbits = torch.randint(0, 2, (cnt, nf), dtype=torch.uint8, device=dev, generator=gen)
    Q = _dev_share(qbits, dev, gen)
    T = _dev_share(torch.from_numpy(Tv.view(np.int64)).to(dev), dev, gen)
    out = torch.empty((3, cnt), dtype=torch.int64, device=dev)
    t = _events_time(lambda: infer_device(T, depth, Q, ctx["keys"], instance_base=start, out=out), steps, warmup,
                     ctx["flush"], ctx["barrier"], ctx["stream"], ctx["max"])
    got = from_device(out).sum(axis=0)
    want = shadow.plaintext_infer(Tv, depth, qbits.cpu().numpy())
    line = {"metric": "secure inference instances/s (10^7 x 32, 10 levels)", "value": n / t, "unit": "instances/s",
            "ms_per_step": t * 1e3, "scaling": "strong",
            "config": "C5: random_tree(default_rng(10), 10, 33), 10^7 random queries; instances sharded",
            "parity_predictions_equal_plaintext_all": bool(np.array_equal(got, want)),
            "roofline": _roof(walk_bytes(cnt, nf, depth), walk_blocks(cnt, nf, depth), t, ctx["peak"],
                              ctx["peak_kind"], ctx["philox"], "k_walk")}
    if ctx["cpu"]:
        # 2*10^4 instances through the C oracle port, scaled x500
        import oracle
        from paper_2305_00645_b200.seeds import keys_tuple

        sub = 20_000
        rng = np.random.default_rng(6)
        qs = qbits[:sub].cpu().numpy()
        Tsh = _share(Tv, rng)
        t0 = time.perf_counter()
        oracle.infer(Tsh, depth, _share(qs, rng), keys_tuple(ctx["keys"]))
        cs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": sub / cs, "unit": "instances/s", "cores": oracle.num_threads(),
                                "kind": "port", "measured_s": cs,
                                "sample": "2*10^4 queries x 32 features on the 10-level tree through "
                                          "oracle/gtree_oracle.c (rate of the full 10^7 = x500 the time)"}
    return line


def e2e_api(Xh, Yh, z, steps, warmup):
    """C2 through the reference-facing drop-in exactly as a reference caller
    runs it (tests/helpers.py:79-99 shape): run_local with three party
    threads, each body hands its own host AVec pair to engine.train_tree, the
    rendezvous checks replication consistency and makes one device call.
    Wall clock per call (host threads, staging copies and sync included)."""
    from paper_2305_00645_b200 import TrainConfig, engine
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from paper_2305_00645_b200.shares import RING64, AVec

    setup = SeedSetup.from_master(derive_seed(SEED_C2, "run"))
    dseed = derive_seed(SEED_C2, "deal")
    cfg = TrainConfig(depth=DEPTH_C2)

    def body(eng):
        p = eng.party
        X = AVec(RING64, Xh[p - 1], Xh[p % 3])
        Y = AVec(RING64, Yh[p - 1], Yh[p % 3])
        r = engine.train_tree(eng, X, Y, cfg)
        return r.T, r.F

    ts, run = [], None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        run = engine.run_local(body, seeds=setup, dealer_seed=dseed)
        if i >= warmup:
            ts.append(time.perf_counter() - t0)
    T = engine.open_results(run, pick=lambda r: r[0])
    F = engine.open_results(run, pick=lambda r: r[1])
    v = statistics.median(ts)
    return {"value": v, "unit": "s/tree", "timing": "wall clock per run_local call, median of the timed steps",
            "path": "engine.run_local + engine.train_tree on per-party host AVecs (cached pinned-staging trainer)",
            "h2d_bytes_per_step": int(Xh.nbytes + Yh.nbytes + 8 * ((1 << DEPTH_C2) - 1)),
            "d2h_bytes_per_step": int(2 * 3 * 8 * ((1 << DEPTH_C2) - 1)),
            "tree_equals_reference": bool(np.array_equal(T, z["T"]) and np.array_equal(F, z["F"]))}


def python_reference(data, Xh, Yh, Tc, q, z):
    """The UNMODIFIED Python reference (obtree, pip-installed into
    baseline/_ref) timed on this host: run_local + train_tree on the C2 shares
    (LiveDealer material, as tests/helpers.py:79-99) and run_local +
    infer_batch on the C3 batch (helpers.py:50-61).  Three party threads;
    numpy runs each op single-threaded.  None if baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "obtree")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from obtree.dealer import LiveDealer
    from obtree.enclave import EnclaveService
    from obtree.infer import infer_batch
    from obtree.ring import RING64
    from obtree.rss import AVec, run_local
    from obtree.train import TrainConfig, levels_of, train_tree
    from obtree.transport import SeedSetup, derive_seed

    setup = SeedSetup.from_master(derive_seed(SEED_C2, "run"))

    def pair(comp, p):
        return AVec(RING64, comp[p - 1].copy(), comp[p % 3].copy())

    def tbody(eng):
        r = train_tree(eng, pair(Xh, eng.party), pair(Yh, eng.party), TrainConfig(depth=DEPTH_C2, heuristic="mpc"))
        return r.T, r.F

    dealer = LiveDealer(derive_seed(SEED_C2, "deal"))
    t0 = time.perf_counter()
    run = run_local(tbody, seeds=setup, materials=[dealer.view(i) for i in (1, 2, 3)],
                    enclave_handler=EnclaveService(setup.enclave_seed).handler)
    t_train = time.perf_counter() - t0
    opened = lambda k: sum((np.asarray(r[k].lo, dtype=np.uint64) for r in run.results), np.uint64(0))  # noqa: E731
    train_ok = bool(np.array_equal(opened(0), z["T"]) and np.array_equal(opened(1), z["F"]))
    rng = np.random.default_rng(3)
    Qs = _share(q, rng)

    def ibody(eng):
        return infer_batch(eng, levels_of(pair(Tc, eng.party), DEPTH_C2), pair(Qs, eng.party))

    dealer = LiveDealer(derive_seed(SEED_C2, "deal-infer"))
    t0 = time.perf_counter()
    irun = run_local(ibody, seeds=setup, materials=[dealer.view(i) for i in (1, 2, 3)])
    t_inf = time.perf_counter() - t0
    preds = sum((np.asarray(r.lo, dtype=np.uint64) for r in irun.results), np.uint64(0))
    return {"kind": "reference", "cores": 3, "threads_note": "3 party threads, numpy single-threaded per op",
            "host_cpus": os.cpu_count(),
            "c2_train": {"value": t_train, "unit": "s/tree", "sample": "one full C2 tree (run_local + train_tree)",
                         "tree_equals_golden": train_ok},
            "c3_infer": {"value": N_C3 / t_inf, "unit": "instances/s", "sample": "the full C3 batch (run_local + "
                         "infer_batch, 10^4 queries, 7 levels)", "predictions_equal_golden":
                         bool(np.array_equal(preds, z["preds"]))}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scale", action="store_true", help="skip the C4/C5 10^6-scale secondaries")
    ap.add_argument("--no-python-reference", action="store_true",
                    help="skip timing the unmodified Python reference (baseline/_ref) on C2/C3")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
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

    # GT_BENCH_DEVICE / GT_BENCH_BACKEND are test hooks (multi-rank dry run on
    # one GPU over gloo); the driver's runs use one GPU per rank over NCCL
    local_dev = int(os.environ.get("GT_BENCH_DEVICE", local))
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) on stderr
        backend = os.environ.get("GT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
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
    peak, peak_kind = _peaks()
    ctx = {"dev": dev, "world": world, "rank": rank, "flush": flush, "barrier": barrier, "stream": stream,
           "max": max_over_ranks, "keys": keys, "peak": peak, "peak_kind": peak_kind, "philox": _philox_peak(),
           "cpu": world == 1 and not args.no_cpu_baseline}

    def step(profile=None):
        return tr.run(X, Y, FL, keys, allreduce=cb, profile=profile)

    # ---- device-resident timed region (value): CUDA-graph replay of whole trees ----
    # (N > 1: the NCCL count allreduce is captured with the kernels; GT_BENCH_EAGER=1 launches eagerly)
    graphed = world == 1 or (dist.get_backend() == "nccl" and not os.environ.get("GT_BENCH_EAGER"))
    replay = None
    if graphed:
        try:
            replay = tr.capture(X, Y, FL, keys, allreduce=cb)
        except Exception as e:  # noqa: BLE001 - N > 1: fall back to eager launches on every rank
            if world == 1:
                raise
            print(f"rank {rank}: graph capture with the NCCL allreduce failed ({e}); eager launches", file=sys.stderr)
            graphed = False
        if world > 1:  # every rank takes the same mode
            flag = torch.tensor([1 if graphed else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if not bool(flag.item()):
                graphed, replay = False, None
    ctx["graphed"] = graphed
    run_tree = replay if replay is not None else step
    for _ in range(args.warmup):
        run_tree()
    torch.cuda.synchronize()
    step_ms = []
    with ClockSampler(local_dev) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_tree()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            step_ms.append(e0.elapsed_time(e1))
    value_s = max_over_ranks(sum(step_ms)) / args.steps / 1e3
    clocks = clk.summary()

    # ---- per-kernel CUDA-event durations: a second pass of K profiled steps ----
    prof_tot = {k: 0.0 for k in ("prods", "partition", "count_lanes", "count_contract", "node_hc", "node_finish")}
    prof_n = {k: 0 for k in prof_tot}
    launches = 0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        p = _native.gt_train_profile()
        step(p)
        barrier()
        launches += p.launches
        for k in prof_tot:
            prof_tot[k] += getattr(p, f"ms_{k}")
            prof_n[k] += getattr(p, f"n_{k}")

    # parity of what was timed: revealed tree == the reference's C2 tree
    z = np.load(os.path.join(ROOT, "tests", "golden", "c2c3.npz"))
    Tc, Fc = from_device(tr.T), from_device(tr.F)
    parity = bool(np.array_equal(Tc.sum(axis=0), z["T"]) and np.array_equal(Fc.sum(axis=0), z["F"]))

    # ---- e2e through the public API with host buffers ----
    # gt_train_host: pinned host shares in, the tree shares out; the sample
    # shares go up in chunks while the prologue of the resident chunks runs
    # (one GPU: the whole call is a CUDA graph, like `value`)
    e2e_ms = []
    Th = torch.empty((3, tr.T.shape[1]), dtype=torch.int64).pin_memory()
    Fh = torch.empty((3, tr.F.shape[1]), dtype=torch.int64).pin_memory()
    tr_h = DeviceTrainer(cnt, NF_C2, TrainConfig(depth=DEPTH_C2), n_total=N_C2, sample_base=start, device=dev,
                         host_io=True)
    cb_h = make_allreduce(tr_h) if world > 1 else None
    run_h = (tr_h.capture_host(Xp, Yp, Fp, Th, Fh, keys, allreduce=cb_h) if graphed
             else (lambda: tr_h.run_host(Xp, Yp, Fp, Th, Fh, keys, allreduce=cb_h)))
    for i in range(args.warmup + args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_h()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        if i >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_parity = bool(np.array_equal(Th.numpy().view(np.uint64).sum(axis=0), z["T"]) and
                      np.array_equal(Fh.numpy().view(np.uint64).sum(axis=0), z["F"]))
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
    # the walk as a one-launch CUDA graph (as the training value): the timed
    # region holds the kernel, not the Python/ctypes enqueue in front of it
    ws_ = torch.cuda.Stream(dev)
    ws_.wait_stream(stream)
    with torch.cuda.stream(ws_):
        infer_device(Tt, DEPTH_C2, Q, keys, instance_base=qs, out=out)
    ws_.synchronize()
    g_walk = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_walk, stream=ws_):
        infer_device(Tt, DEPTH_C2, Q, keys, instance_base=qs, out=out)
    inf_s = _events_time(g_walk.replay, args.steps, args.warmup, flush, barrier, stream, max_over_ranks)
    Oh = torch.empty((3, qc), dtype=torch.int64).pin_memory()

    def inf_e2e():
        Q.copy_(Qp, non_blocking=True)
        infer_device(Tt, DEPTH_C2, Q, keys, instance_base=qs, out=out)
        Oh.copy_(out, non_blocking=True)

    # one CUDA graph per e2e step (H2D of the queries, the walk, D2H of the
    # predictions), as the training e2e: no host launch gaps inside the timed region
    gs = torch.cuda.Stream(dev)
    gs.wait_stream(stream)
    with torch.cuda.stream(gs):
        inf_e2e()
    gs.synchronize()
    g_inf = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_inf, stream=gs):
        inf_e2e()
    inf_e2e_s = _events_time(g_inf.replay, args.steps, args.warmup, flush, barrier, stream, max_over_ranks)
    preds_ok = True
    if world == 1:
        preds_ok = bool(np.array_equal(from_device(out).sum(axis=0), z["preds"]))

    # ---- e2e through the reference-facing drop-in API (what a reference caller runs) ----
    # run_local + train_tree with host AVecs per party (rss.py:496-542, train.py:108): three party
    # threads, the rendezvous, consistency check, pinned staging, one gt_train_host call, scatter
    api = e2e_api(Xh, Yh, z, args.steps, args.warmup) if world == 1 else None

    scale = {}
    if not args.no_scale:
        scale["c4_train"] = scale_c4(ctx, max(3, args.steps // 2), args.warmup)
        scale["c5_infer"] = scale_c5(ctx, max(3, args.steps // 2), args.warmup)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel class ----
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # dominant single kernel: node_hc (k_hc_pre + k_hc_div + k_hc_post per level) and node_finish are
    # multi-kernel latency chains with no bulk data; their times are in kernel_ms_per_step
    dom = max((k for k in prof_tot if k not in ("node_hc", "node_finish")), key=lambda k: prof_tot[k])
    bytes_of = {"count_lanes": count_lanes_bytes(cnt, NF_C2, DEPTH_C2),
                "count_contract": count_contract_bytes(cnt, NF_C2, DEPTH_C2),
                "partition": partition_bytes(cnt, NF_C2, DEPTH_C2),
                # prologue: features + labels in, the W sample columns (x | x*y | y) out
                "prods": cnt * (24 * (NF_C2 + 1) + 24 * (2 * NF_C2 + 1)), "node_hc": 0, "node_finish": 0}
    kname = {"count_lanes": "k_count_lanes8", "count_contract": "k_count_mma", "partition": "k_partition_split",
             "node_hc": "k_hc_div", "prods": "k_prep8", "node_finish": "k_node_finish"}
    fused = prof_tot["count_lanes"] == 0 and prof_tot["count_contract"] > 0
    if fused:  # k_count_fused: lanes + contraction in one kernel; SURVEY 8(d)'s count-level bytes
        kname["count_contract"] = "k_count_fused"
        bytes_of["count_contract"] = count_bytes(cnt, NF_C2, DEPTH_C2)
    alg = bytes_of[dom] * args.steps
    achieved = alg / (prof_tot[dom] / 1e3) / 1e9 if prof_tot[dom] > 0 else 0.0
    nlaunch = max(1, prof_n[dom])
    traffic = _traffic(kname.get(dom, dom))
    # integer-ALU roof: Philox blocks the dominant kernel draws vs the measured Philox peak
    # (randomness schedule v2: a pair of eq lanes draws 2 x 3 dealer blocks + 3 shared pair blocks;
    # each lookup adds 2 x 3 telescoped reshare words per index)
    blocks = {"count_lanes": count_lane_blocks(cnt, DEPTH_C2),
              "count_contract": count_lane_blocks(cnt, DEPTH_C2) if fused else None,
              "partition": partition_blocks(cnt, NF_C2, DEPTH_C2)}.get(dom)
    alu = None
    if blocks:
        alu = {"bound": "int-alu (Philox4x32-10 blocks)", "achieved_blocks_per_s": blocks * args.steps / (prof_tot[dom] / 1e3),
               "peak_blocks_per_s": ctx["philox"], "note": "peak measured by gt_diag_philox on this GPU"}
        alu["frac"] = alu["achieved_blocks_per_s"] / alu["peak_blocks_per_s"] if alu["peak_blocks_per_s"] else None
    # every kernel class against the HBM roof (same definitions), for the record
    classes = {}
    for k in prof_tot:
        if prof_tot[k] > 0 and bytes_of.get(k):
            gbs = bytes_of[k] * args.steps / (prof_tot[k] / 1e3) / 1e9
            classes[k] = {"kernel": kname.get(k, k), "ms_per_step": prof_tot[k] / args.steps,
                          "achieved_gbs": gbs, "frac": gbs / peak}
            iss = _issue(kname.get(k, k), prof_tot[k] / max(1, prof_n[k]) / 1e3, clocks, sms)
            if iss:
                classes[k]["issue_frac"] = iss["frac"]
    cpu_base = cpu_c3 = py_ref = None
    if ctx["cpu"]:
        import oracle
        from paper_2305_00645_b200.seeds import keys_tuple

        t0 = time.perf_counter()
        oracle.train(Xh, Yh, fill, DEPTH_C2, keys_tuple(keys))
        cs = time.perf_counter() - t0
        cpu_base = {"value": cs, "unit": "s/tree", "cores": oracle.num_threads(), "kind": "port",
                    "sample": "one full C2 tree (48842x13, depth 7) through oracle/gtree_oracle.c"}
        t0 = time.perf_counter()
        oracle.infer(Tc, DEPTH_C2, Qp.numpy().view(np.uint64), keys_tuple(keys))
        cs = time.perf_counter() - t0
        cpu_c3 = {"value": N_C3 / cs, "unit": "instances/s", "cores": oracle.num_threads(), "kind": "port",
                  "sample": "the full C3 batch (10^4 queries, 7 levels) through oracle/gtree_oracle.c"}
        if not args.no_python_reference:
            py_ref = python_reference(data, Xh, Yh, Tc, q, z)
    walk_alg = walk_bytes(qc, NF_C2, DEPTH_C2)
    # inter-party messages of the protocol the kernels execute (the analytic
    # transcript, ledger.py) beside the reference's (its lane_limit chunking)
    from paper_2305_00645_b200 import ledger

    def _msgs(ours, ref):
        return {"rounds": ours.rounds, "bytes_per_party": ours.sent_by_party(1),
                "reference_rounds": ref.rounds, "reference_bytes_per_party": ref.sent_by_party(1)}
    messages = {"note": "3-party transcript per tree / per batch (party 1 sends; the parties are symmetric)",
                "c2_train": _msgs(ledger.train_metrics(N_C2, NF_C2, DEPTH_C2, lane_limit=None),
                                  ledger.train_metrics(N_C2, NF_C2, DEPTH_C2)),
                "c3_infer": _msgs(ledger.infer_metrics(N_C3, NF_C2, DEPTH_C2, lane_limit=None),
                                  ledger.infer_metrics(N_C3, NF_C2, DEPTH_C2))}
    line = {
        "metric": METRIC, "value": value_s, "unit": "s/tree", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value_s * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (Adult-shaped binary matrix, default_rng(1011); random 3-party shares)",
        "config": _c2_config(),
        "parallelism": f"samples sharded x{world}" + (" + NCCL count allreduce" if world > 1 else ""),
        "parity": {"tree_equals_reference": parity, "e2e_tree_equals_reference": e2e_parity,
                   "c3_predictions_equal_reference": preds_ok},
        "e2e": {"value": e2e_s, "unit": "s/tree", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "messages": messages,
        "roofline": {"bound": "hbm", "kernel": kname.get(dom, dom), "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": bytes_of[dom] / max(1, prof_n[dom] // args.steps),
                     "avg_launch_ms": prof_tot[dom] / nlaunch, "alu": alu,
                     "issue": _issue(kname.get(dom, dom), prof_tot[dom] / nlaunch / 1e3, clocks, sms),
                     "classes": classes},
        "kernel_ms_per_step": {k: v / args.steps for k, v in prof_tot.items()},
        "timing": ("value: CUDA-graph replay of the whole tree" + (" incl. the NCCL count allreduce" if world > 1 else "")
                   + ("" if graphed else " [eager stream launches: GT_BENCH_EAGER / non-NCCL backend]") + "; "
                   "kernel_ms_per_step + roofline: separate pass of K steps with per-launch CUDA events"),
        "clocks": clocks,
        "secondary": {"metric": METRIC2, "value": N_C3 / inf_s, "unit": "instances/s", "ms_per_step": inf_s * 1e3,
                      "config": "C3: 10^4 queries x 13 features on the C2 tree (7 levels)",
                      "timing": "value: CUDA-graph replay of the walk (one launch), L2 flushed between steps",
                      "e2e": {"value": N_C3 / inf_e2e_s, "unit": "instances/s",
                              "h2d_bytes_per_step": int(Qp.numel() * 8), "d2h_bytes_per_step": int(Oh.numel() * 8)},
                      "roofline": _roof(walk_alg, walk_blocks(qc, NF_C2, DEPTH_C2), inf_s, peak, peak_kind,
                                        ctx["philox"], "k_walk", traffic=_traffic("k_walk"),
                                        issue=_issue("k_walk", inf_s, clocks, sms))},
        "tree_roofline": _roof(tree_bytes(cnt, NF_C2, DEPTH_C2), tree_blocks(cnt, NF_C2, DEPTH_C2), value_s, peak,
                               peak_kind, ctx["philox"], "whole C2 tree (all kernels, serial chain)"),
        "scale": scale,
    }
    if api is not None:
        line["e2e_api"] = api
    if cpu_base is not None:
        line["cpu_baseline"] = cpu_base
        line["secondary"]["cpu_baseline"] = cpu_c3
    if py_ref is not None:
        line["cpu_baseline_python_reference"] = py_ref
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _philox_peak():
    import ctypes

    import torch

    from paper_2305_00645_b200 import _native

    lib = _native.load()
    grid, iters = 148 * 32, 4096
    out = torch.empty(grid * 256, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    run = lambda: _native.check(lib.gt_diag_philox(grid, iters, out.data_ptr(), ctypes.c_void_p(s.cuda_stream)))  # noqa: E731
    run()
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        run()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return grid * 256 * iters / (best / 1e3)


if __name__ == "__main__":
    main()
