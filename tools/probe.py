"""Dev timing probe (A/B experiments; not a bench number).

  python tools/probe.py c2      C2 tree: CUDA-graph replay median ms + per-kernel-class ms
  python tools/probe.py walk    C3 (10^4 x 13, 7 levels) and a C5 slice (2*10^6 x 32, 10 levels) inst/s
  python tools/probe.py c2eager three eager C2 trees (launch lists)
  python tools/probe.py cts     fused count phase timestamps per level (GT_COUNT_TS=1)
  python tools/probe.py c4      C4 tree (10^6 x 32, depth 8) graph replay median ms
  python tools/probe.py api     C2 through run_local + train_tree: wall-clock split of the drop-in host path
  python tools/probe.py tl      one eager C2 tree's level timeline: count + heuristic phase
                                timestamps on one clock (GT_COUNT_TS=1 GT_HC_TIMING=1)
Launch switches (GT_PART_G, GT_WALK_G, ...) come from the environment;
GT_PROBE_ENGINE=cuda runs the count contraction on the CUDA cores (A/B).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_00645_b200 import TrainConfig, _native  # noqa: E402
from paper_2305_00645_b200.infer import infer_device  # noqa: E402
from paper_2305_00645_b200.train import DeviceTrainer  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    what = sys.argv[1]
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("GT_"))
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
    setup, keys, fill = bench._keys_and_filler()
    if what == "c2":
        data, X, Y = bench._c2_inputs()
        eng = os.environ.get("GT_PROBE_ENGINE", "tensor")  # count engine A/B: tensor | cuda
        tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2, count_engine=eng))
        X, Y, F = t(X), t(Y), t(fill)
        g = tr.capture(X, Y, F, keys)
        ms = timed(g)
        z = np.load(os.path.join(bench.ROOT, "tests", "golden", "c2c3.npz"))
        ok = np.array_equal(tr.T.sum(0).cpu().numpy().view(np.uint64), z["T"])
        p = _native.gt_train_profile()
        tr.run(X, Y, F, keys, profile=p)
        torch.cuda.synchronize()
        ks = ("prods", "partition", "count_lanes", "count_contract", "node_hc", "node_finish")
        print(f"[{tag}] C2 {ms:.4f} ms tree_ok={ok} |", " ".join(f"{k}={getattr(p, 'ms_' + k) * 1e3:.1f}us"
                                                              for k in ks), flush=True)
    elif what == "c2eager":  # launch lists: three eager tree runs (GT_PROBE_ENGINE selects the count engine)
        data, X, Y = bench._c2_inputs()
        tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2,
                                                                count_engine=os.environ.get("GT_PROBE_ENGINE", "tensor")))
        X, Y, F = t(X), t(Y), t(fill)
        for _ in range(3):
            tr.run(X, Y, F, keys)
        torch.cuda.synchronize()
        z = np.load(os.path.join(bench.ROOT, "tests", "golden", "c2c3.npz"))
        print("tree_ok", np.array_equal(tr.T.sum(0).cpu().numpy().view(np.uint64), z["T"]))
    elif what == "cts":  # fused count phase timestamps per level (GT_COUNT_TS=1)
        import ctypes
        data, X, Y = bench._c2_inputs()
        tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2))
        X, Y, F = t(X), t(Y), t(fill)
        for _ in range(3):
            tr.run(X, Y, F, keys)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 64)()
        _native.check(_native.load().gt_diag_count_timestamps(buf, 64))
        names = ["wait", "item0", "items", "mma", "done", "epi"]
        for lv in range(bench.DEPTH_C2):
            ts = buf[8 * lv: 8 * lv + 7]
            print(f"level {lv}: " + " ".join(f"{n}=+{(ts[k + 1] - ts[0]) / 1e3:.1f}" for k, n in enumerate(names)) + " us")
    elif what == "tl":  # timeline: count (cluster 0) + heuristic (node 0) phases, us from the level-0 count start
        import ctypes
        data, X, Y = bench._c2_inputs()
        tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2))
        X, Y, F = t(X), t(Y), t(fill)
        for _ in range(3):
            tr.run(X, Y, F, keys)
        torch.cuda.synchronize()
        cb, hb = (ctypes.c_ulonglong * 64)(), (ctypes.c_ulonglong * 128)()
        lib = _native.load()
        _native.check(lib.gt_diag_count_timestamps(cb, 64))
        _native.check(lib.gt_diag_hc_timestamps(hb, 128))
        t0 = cb[0]
        us = lambda v: f"{(v - t0) / 1e3:7.1f}" if v else "     - "  # noqa: E731
        cn = ["c.start", "c.wait", "c.item0", "c.items", "c.mma", "c.done", "c.epi", "c.last"]
        pn = ["ctl.start", "ctl.tapes", "ctl.end", "ft.start", "ft.tape", "ft.end", "div.start", "div.end"]
        qn = ["post.scores", "post.argmin", "post.budget", "post.split", "post.end", "p5", "p6", "ladder"]
        for lv in range(bench.DEPTH_C2):
            print(f"level {lv}")
            print("   " + " ".join(f"{n}={us(cb[8 * lv + k])}" for k, n in enumerate(cn)))
            print("   " + " ".join(f"{n}={us(hb[64 + 8 * lv + k])}" for k, n in enumerate(pn)))
            print("   " + " ".join(f"{n}={us(hb[8 * lv + k])}" for k, n in enumerate(qn)))
    elif what == "api":  # drop-in host path breakdown (ms, medians of 10)
        import time
        import statistics
        from paper_2305_00645_b200 import engine
        from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys
        from paper_2305_00645_b200.shares import RING64, AVec, stage_pairs, avecs_from_components
        from paper_2305_00645_b200.train import _cached_trainer, as_config
        data, Xc, Yc = bench._c2_inputs()
        Xh = [np.ascontiguousarray(Xc[i]) for i in range(3)]
        Xh2 = [x.copy() for x in Xh]  # separate hi arrays, as a real caller's pairs
        Yh = [np.ascontiguousarray(Yc[i]) for i in range(3)]
        Yh2 = [y.copy() for y in Yh]
        setup = SeedSetup.from_master(derive_seed(bench.SEED_C2, "run"))
        dseed = derive_seed(bench.SEED_C2, "deal")
        cfg = TrainConfig(depth=bench.DEPTH_C2)
        xp = [(Xh[i], Xh2[(i + 1) % 3]) for i in range(3)]
        yp = [(Yh[i], Yh2[(i + 1) % 3]) for i in range(3)]
        tr = _cached_trainer(bench.N_C2, bench.NF_C2, as_config(cfg), None, True)
        st = tr.staging
        res = {}
        def tm(name, f, n=10):
            ts = []
            for _ in range(n):
                a = time.perf_counter(); f(); ts.append(time.perf_counter() - a)
            res[name] = statistics.median(ts) * 1e3
        tm("make_keys", lambda: make_keys(setup, dseed))
        tm("filler", lambda: filler_values(setup.filler_seed, 127, 14))
        tm("stage_X", lambda: stage_pairs(xp, st["X"].numpy().view(np.uint64), True))
        tm("stage_X_nocheck", lambda: stage_pairs(xp, st["X"].numpy().view(np.uint64), False))
        tm("stage_Y", lambda: stage_pairs(yp, st["Y"].numpy().view(np.uint64), True))
        keys = make_keys(setup, dseed)
        s = torch.cuda.current_stream()
        def run():
            tr.run_host(st["X"], st["Y"], st["fill"], st["T"], st["F"], keys, stream=s); s.synchronize()
        tm("run_host", run)
        def body(eng):
            p = eng.party
            return engine.train_tree(eng, AVec(RING64, Xh[p - 1], Xh2[p % 3]), AVec(RING64, Yh[p - 1], Yh2[p % 3]), cfg)
        from paper_2305_00645_b200.train import train_pairs
        tm("train_pairs_direct", lambda: train_pairs(xp, yp, cfg, setup, dseed))
        # its steps one by one (wall clock marks, ms)
        marks = []
        for _ in range(10):
            a = time.perf_counter()
            stage_pairs(xp, st["X"].numpy().view(np.uint64), False)
            stage_pairs(yp, st["Y"].numpy().view(np.uint64), False)
            b = time.perf_counter()
            st["fill"].numpy().view(np.uint64)[:] = filler_values(setup.filler_seed, 127, 14)
            replay = tr.host_graph(keys)
            replay()
            c = time.perf_counter()
            stage_pairs(xp, None, True)
            stage_pairs(yp, None, True)
            d = time.perf_counter()
            s.synchronize()
            e = time.perf_counter()
            T = st["T"].numpy().view(np.uint64)[:, :127].copy()
            f = time.perf_counter()
            marks.append((b - a, c - b, d - c, e - d, f - e))
        med = [statistics.median(m[k] for m in marks) * 1e3 for k in range(5)]
        print("split: stage %.3f launch %.3f check %.3f sync %.3f copy %.3f" % tuple(med), flush=True)
        tm("run_local_total", lambda: engine.run_local(body, seeds=setup, dealer_seed=dseed))
        tm("threads_only", lambda: engine.run_local(lambda eng: None, seeds=setup, dealer_seed=dseed))
        print(" ".join(f"{k}={v:.3f}" for k, v in res.items()), flush=True)
        if os.environ.get("GT_PROBE_PROFILE"):
            import cProfile
            import pstats
            import threading
            threading.setprofile(None)
            pr = cProfile.Profile()
            for _ in range(10):
                pr.enable()
                engine.run_local(body, seeds=setup, dealer_seed=dseed)
                pr.disable()
            pstats.Stats(pr).sort_stats("tottime").print_stats(15)
    elif what == "small":  # sanitizer target: 4000 x 13, depth 7 (fused count with paired x-plane copies, early oaa
        # lanes, split partition; the last partition's 32 entries split between early and inline pairs)
        rng = np.random.default_rng(5)
        n, nf, depth = 4000, 13, 7
        X = t(bench._share(rng.integers(0, 2, (n, nf)), rng))
        Y = t(bench._share(rng.integers(0, 2, n), rng))
        F = t(np.zeros((1 << depth) - 1, dtype=np.uint64))
        tr = DeviceTrainer(n, nf, TrainConfig(depth=depth))
        tr.run(X, Y, F, keys)
        torch.cuda.synchronize()
        print("small tree ok", flush=True)
    elif what == "c4":
        n, nf, depth = 10 ** 6, 32, 8
        rng = np.random.default_rng(3)
        X = t(bench._share(rng.integers(0, 2, (n, nf)), rng))
        Y = t(bench._share(rng.integers(0, 2, n), rng))
        F = t(np.zeros((1 << depth) - 1, dtype=np.uint64))
        tr = DeviceTrainer(n, nf, TrainConfig(depth=depth, count_engine=os.environ.get("GT_PROBE_ENGINE", "tensor")))
        print(f"[{tag}] C4 {timed(tr.capture(X, Y, F, keys), 10):.3f} ms", flush=True)
        p = _native.gt_train_profile()
        tr.run(X, Y, F, keys, profile=p)
        torch.cuda.synchronize()
        ks = ("prods", "partition", "count_lanes", "count_contract", "node_hc", "node_finish")
        print(" ".join(f"{k}={getattr(p, 'ms_' + k):.2f}ms" for k in ks), flush=True)
    elif what == "walk":
        rng = np.random.default_rng(1)
        for depth, nf, n in ((7, 13, 10_000), (10, 32, 2_000_000)):
            T = t(bench._share(rng.integers(0, nf, (1 << depth) - 1), rng))
            Q = t(bench._share(rng.integers(0, 2, (n, nf)), rng))
            out = torch.empty((3, n), dtype=torch.int64, device=dev)
            ms = timed(lambda: infer_device(T, depth, Q, keys, out=out))
            print(f"[{tag}] walk d{depth} nf{nf} n{n}: {ms * 1e3:.1f} us  {n / ms / 1e3:.1f} M inst/s", flush=True)


if __name__ == "__main__":
    main()
