"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script is the only thing in the repo that imports the reference package
(`obtree`, mounted read-only at /root/reference).  It runs in the build
container, never on the GPU box; its outputs are small committed fixtures:

  kats.json          gadget known-answer vectors (division, argmin, truncate,
                     OAA out-of-range, counter_shift, filler stream, seeds)
  trees_mpc.npz      datasets + revealed (T, F) trees of the reference MPC
                     trainer (`helpers.secure_train`, heuristic "mpc") and the
                     rational oracle `plaintext_train`
  infer.npz          random trees + queries + reference MPC predictions
  transcripts.json   reference transcript metrics / records for ledger parity
  c2c3.npz           Adult-shaped depth-7 MPC tree (C2) and the 10^4-query
                     predictions against it (C3), plus their metrics

Usage:  python tests/golden/make_golden.py [--skip-c2]
Reference call sites followed: tests/helpers.py:79-103 (secure_train,
oracle_for), tests/test_infer.py:18-26 (_run_infer), test_acceptance.py:44-71.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from helpers import open_u64, run_dealer, secure_train, oracle_for, share_in, open_bits3  # noqa: E402
from obtree import tree as tree_mod  # noqa: E402
from obtree.gadgets import argmin_masked, division, truncate, eq, lt, b2a, select_share  # noqa: E402
from obtree.infer import infer_batch  # noqa: E402
from obtree.oaa import oaa, row_lookup  # noqa: E402
from obtree.ring import RING8, RING32, RING64  # noqa: E402
from obtree.rss import AVec  # noqa: E402
from obtree.train import TrainConfig, counter_shift, levels_of  # noqa: E402
from obtree.transport import SeedSetup, derive_seed  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _battery_dataset(i):
    # test_acceptance.py:44-63
    rng = np.random.default_rng(10_000 + i)
    n = int(rng.integers(64, 513))
    d = int(rng.integers(3, 9))
    depth = int(rng.integers(1, 6))
    feats = rng.integers(0, 2, (n, d - 1), dtype=np.uint8)
    kind = i % 4
    if kind == 1:
        feats[:, int(rng.integers(0, d - 1))] = int(rng.integers(0, 2))
    if kind == 2:
        labels = (feats[:, 0] ^ (rng.random(n) < 0.1)).astype(np.uint8)
    elif kind == 3:
        cols = rng.choice(d - 1, size=min(3, d - 1), replace=False)
        take = feats[:, cols]
        labels = (take.sum(axis=1) * 2 > take.shape[1]).astype(np.uint8)
    else:
        labels = rng.integers(0, 2, n, dtype=np.uint8)
    return np.column_stack([feats, labels]), depth


def _spect_shaped():
    # test_acceptance.py:66-71
    rng = np.random.default_rng(555)
    feats = rng.integers(0, 2, (267, 22), dtype=np.uint8)
    labels = ((feats[:, 0] & feats[:, 3]) | feats[:, 7]).astype(np.uint8)
    labels[rng.random(267) < 0.08] ^= 1
    return np.column_stack([feats, labels])


def _metrics_dict(run):
    m = run.metrics
    return {"rounds": m.rounds, "bytes_by_pair": m.bytes_by_pair,
            "bytes_by_tag": m.bytes_by_tag, "rounds_by_tag": m.rounds_by_tag}


def make_kats():
    out = {}
    # division frozen values: test_gadgets.py:152-161
    pairs = [(355, 113), (1, 1), (1, 2), (1000, 512), (999999, 250000)]
    rng = np.random.default_rng(2024)
    qs = rng.integers(1, 1 << 17, 200, dtype=np.uint64)
    ps = rng.integers(0, 1 << 19, 200, dtype=np.uint64)
    P = np.array([p for p, _ in pairs] + list(ps), dtype=np.uint64)
    Q = np.array([q for _, q in pairs] + list(qs), dtype=np.uint64)

    def body(eng):
        return division(eng, share_in(eng, P, RING32, "kp"), share_in(eng, Q, RING32, "kq"), 10)
    got = open_u64(run_dealer(body).results, RING32)
    out["division_tau10_w32"] = {"p": P.tolist(), "q": Q.tolist(), "out": got.tolist()}

    # argmin frozen: test_gadgets.py:224-235 plus random masked batteries
    sc = np.array([[3, 1, 2], [1, 1, 5]], dtype=np.uint64)
    av = np.ones_like(sc, dtype=np.uint8)
    rs = rng.integers(0, 40, (30, 7), dtype=np.uint64)
    ra = rng.integers(0, 2, (30, 7), dtype=np.uint8)
    cases = []
    for scores, avail in ((sc, av), (rs, ra)):
        def body(eng, scores=scores, avail=avail):
            from helpers import share_bits_in
            s = share_in(eng, scores, RING32, "as")
            a = share_bits_in(eng, avail, "aa")
            return argmin_masked(eng, s, a, worst=1 << 11, idx_ring=RING64)
        got = open_u64(run_dealer(body).results, RING64)
        cases.append({"scores": scores.tolist(), "avail": avail.tolist(), "out": got.tolist()})
    out["argmin_w32"] = cases

    # truncate == >> k (test_gadgets.py:118-129)
    vals = np.array([0, 1, 2, 1023, 1024, (1 << 31), (1 << 32) - 1, 123456789, 0xDEADBEEF], dtype=np.uint64)
    tr = {}
    for k in (1, 6, 10, 14, 17, 20, 31):
        def body(eng, k=k):
            return truncate(eng, share_in(eng, vals, RING32, f"t{k}"), k)
        tr[str(k)] = open_u64(run_dealer(body).results, RING32).tolist()
    out["truncate_w32"] = {"x": vals.tolist(), "out": tr}
    v64 = np.array([0, 1, 48842 * 3, (1 << 63) + 5, (1 << 64) - 1, 0x0123456789ABCDEF], dtype=np.uint64)
    tr64 = {}
    for k in (1, 6, 10, 33, 63):
        def body(eng, k=k):
            return truncate(eng, share_in(eng, v64, RING64, f"u{k}"), k)
        tr64[str(k)] = open_u64(run_dealer(body).results, RING64).tolist()
    out["truncate_w64"] = {"x": v64.tolist(), "out": tr64}

    # OAA out-of-range -> 0 (test_oaa.py:44-54)
    table = np.array([5, 6, 7], dtype=np.uint64)
    idx = np.array([0, 3, 250, 2], dtype=np.uint64)

    def body(eng):
        return oaa(eng, share_in(eng, table, RING8, "ot"), share_in(eng, idx, RING8, "oi"))
    out["oaa_oob_w8"] = {"table": table.tolist(), "idx": idx.tolist(),
                         "out": open_u64(run_dealer(body).results, RING8).tolist()}

    out["counter_shift"] = {str(n): counter_shift(n, TrainConfig()) for n in
                            (1, 267, 1023, 1024, 1500, 4096, 48842, 10 ** 6)}

    # seed derivation + public filler stream (tree.py:160-169, transport.py:58-60)
    seeds = {}
    for master in (b"\x01" * 16, (11_000).to_bytes(16, "little"), derive_seed(b"\x07" * 16, "run")):
        s = SeedSetup.from_master(master)
        seeds[master.hex()] = {
            "pair": {str(i): s.pair_seeds[i].hex() for i in (1, 2, 3)},
            "filler": s.filler_seed.hex(),
            "filler_values_127_14": tree_mod.filler_values(s.filler_seed, 127, 14).tolist(),
            "filler_values_1023_33": tree_mod.filler_values(s.filler_seed, 1023, 33).tolist(),
        }
    out["seeds"] = seeds
    with open(os.path.join(OUT, "kats.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("kats done")


def make_trees():
    cases = []
    # test_train.py:47-51 depth-1 majority
    cases.append((np.array([[0, 1], [1, 1], [0, 1], [1, 0]], dtype=np.uint8), 1, b"\x0a" * 16, "majority"))
    rng = np.random.default_rng(42)   # test_train.py:16-28
    for trial in range(10):
        n = int(rng.integers(4, 150))
        d = int(rng.integers(2, 8))
        depth = int(rng.integers(1, 5))
        data = rng.integers(0, 2, (n, d), dtype=np.uint8)
        cases.append((data, depth, bytes([trial + 1]) * 16, f"random{trial}"))
    rng = np.random.default_rng(9)    # test_train.py:31-44 skewed
    for trial in range(5):
        n = int(rng.integers(4, 60))
        d = int(rng.integers(2, 6))
        data = np.zeros((n, d), dtype=np.uint8)
        data[:, int(rng.integers(0, d))] = rng.integers(0, 2, n)
        cases.append((data, 3, bytes([trial + 50]) * 16, f"skewed{trial}"))
    rng = np.random.default_rng(4)    # test_train.py:54-62 counter shift 1
    cases.append((rng.integers(0, 2, (1500, 5), dtype=np.uint8), 3, b"\x0b" * 16, "shift1500"))
    for i in range(24):               # acceptance battery (C5 shape)
        data, depth = _battery_dataset(i)
        cases.append((data, depth, (5000 + i).to_bytes(16, "little"), f"battery{i}"))
    cases.append((_spect_shaped(), 4, (555).to_bytes(16, "little"), "spect_d4"))
    cases.append((_spect_shaped(), 5, (999).to_bytes(16, "little"), "spect_d5"))
    rng = np.random.default_rng(77)
    cases.append((rng.integers(0, 2, (4000, 9), dtype=np.uint8), 5, b"\x33" * 16, "n4000"))
    # all-constant labels / single sample / constant features
    cases.append((np.ones((7, 4), dtype=np.uint8), 3, b"\x34" * 16, "all_ones"))
    cases.append((np.array([[1, 0, 1]], dtype=np.uint8), 2, b"\x35" * 16, "single"))
    arrays = {}
    meta = []
    for k, (data, depth, seed, name) in enumerate(cases):
        t0 = time.time()
        T, F, dep, run = secure_train(data, TrainConfig(depth=depth, heuristic="mpc"), seed)
        ref = oracle_for(data, depth, seed)
        arrays[f"data{k}"] = data
        arrays[f"T{k}"] = T
        arrays[f"F{k}"] = F
        arrays[f"oT{k}"] = ref.T
        arrays[f"oF{k}"] = ref.F
        meta.append({"name": name, "depth": depth, "seed": seed.hex(), "n": int(data.shape[0]),
                     "d": int(data.shape[1]), "metrics": _metrics_dict(run) if data.shape[0] <= 600 else None,
                     "exact_vs_rational": bool(np.array_equal(T, ref.T) and np.array_equal(F, ref.F))})
        print(f"tree {name}: {time.time() - t0:.1f}s")
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "trees_mpc.npz"), **arrays)


def make_infer():
    arrays = {}
    meta = []
    rng = np.random.default_rng(21)
    k = 0
    for depth, d, nq in ((1, 3, 5), (2, 4, 17), (3, 5, 60), (4, 6, 33), (5, 9, 40), (7, 14, 50), (8, 33, 20)):
        tree = tree_mod.random_tree(rng, depth, d)
        queries = rng.integers(0, 2, (nq, d - 1), dtype=np.uint8)

        def body(eng):
            t = share_in(eng, tree.T, RING64, "T")
            q = share_in(eng, queries, RING64, "q")
            return infer_batch(eng, levels_of(t, depth), q)
        run = run_dealer(body)
        got = open_u64(run.results, RING64)
        want = np.array([tree_mod.plaintext_infer(tree, q) for q in queries], dtype=np.uint64)
        assert np.array_equal(got, want)
        arrays[f"T{k}"] = tree.T
        arrays[f"F{k}"] = tree.F
        arrays[f"q{k}"] = queries
        arrays[f"p{k}"] = got
        meta.append({"depth": depth, "d": d, "nq": nq, "metrics": _metrics_dict(run)})
        k += 1
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "infer.npz"), **arrays)
    print("infer done")


def make_transcripts():
    """Reference transcripts for the analytic ledger (transport.py:131-202)."""
    out = {}
    rng = np.random.default_rng(31)
    # gadget-level, outside any phase (gadget tags)
    x = rng.integers(0, 1 << 32, 37, dtype=np.uint64)
    y = rng.integers(0, 1 << 32, 37, dtype=np.uint64)
    bits = rng.integers(0, 2, 37, dtype=np.uint8)
    for width, ring in ((8, RING8), (32, RING32), (64, RING64)):
        def body(eng, ring=ring):
            from helpers import share_bits_in
            a = share_in(eng, x & np.uint64(ring.mask), ring, "gx")
            b = share_in(eng, y & np.uint64(ring.mask), ring, "gy")
            c = share_bits_in(eng, bits, "gb")
            eq(eng, a, b)
            eq(eng, a, 5)
            lt(eng, a, b)
            lt(eng, a, 7)
            b2a(eng, c, ring)
            select_share(eng, a, b, c)
            truncate(eng, a, 3)
            eng.mul(a, b)
            return 0
        run = run_dealer(body)
        out[f"gadgets_w{width}"] = {"records": run.transcript.records}

    def body(eng):
        p = share_in(eng, np.arange(1, 12, dtype=np.uint64) * 37, RING32, "dp")
        q = share_in(eng, np.arange(1, 12, dtype=np.uint64) * 11, RING32, "dq")
        division(eng, p, q, 10)
        from helpers import share_bits_in
        s = share_in(eng, rng_sc, RING32, "as")
        a = share_bits_in(eng, rng_av, "aa")
        argmin_masked(eng, s, a, worst=1 << 11)
        return 0
    rng_sc = rng.integers(0, 40, (5, 13), dtype=np.uint64)
    rng_av = rng.integers(0, 2, (5, 13), dtype=np.uint8)
    out["division_argmin"] = {"records": run_dealer(body).transcript.records}

    for m, n, ll in ((1, 40, 1 << 22), (7, 40, 1 << 22), (13, 100, 64), (64, 30, 1000)):
        t = rng.integers(0, 1 << 30, m, dtype=np.uint64)
        u = rng.integers(0, m, n, dtype=np.uint64)

        def body(eng, t=t, u=u):
            rows = share_in(eng, np.zeros((n, m), np.uint64), RING64, "rw")
            oaa(eng, share_in(eng, t, RING64, "ot"), share_in(eng, u, RING64, "ou"))
            row_lookup(eng, rows, share_in(eng, u, RING64, "ou2"))
            return 0
        out[f"oaa_m{m}_n{n}_ll{ll}"] = {"records": run_dealer(body, lane_limit=ll).transcript.records,
                                       "m": m, "n": n, "lane_limit": ll}

    # training / inference, several lane limits
    for (n, d, depth, ll) in ((60, 4, 3, 1 << 22), (60, 4, 3, 128), (150, 6, 4, 1 << 22), (150, 6, 4, 500),
                              (33, 3, 1, 1 << 22), (100, 8, 5, 3000)):
        data = np.random.default_rng(n + d + depth).integers(0, 2, (n, d), dtype=np.uint8)
        from obtree.dealer import LiveDealer
        from obtree.enclave import EnclaveService
        from obtree.train import train_tree
        from obtree.rss import run_local
        seed = b"\x44" * 16
        setup = SeedSetup.from_master(derive_seed(seed, "run"))
        dealer = LiveDealer(derive_seed(seed, "deal"))

        def body(eng, data=data, depth=depth):
            X = share_in(eng, data[:, :-1], RING64, "X")
            y = share_in(eng, data[:, -1], RING64, "y")
            return train_tree(eng, X, y, TrainConfig(depth=depth, heuristic="mpc")).depth
        run = run_local(body, seeds=setup, materials=[dealer.view(i) for i in (1, 2, 3)],
                        enclave_handler=EnclaveService(setup.enclave_seed).handler, lane_limit=ll)
        out[f"train_n{n}_d{d}_h{depth}_ll{ll}"] = {"n": n, "d": d, "depth": depth, "lane_limit": ll,
                                                   "records": run.transcript.records}
    for (nq, d, depth, ll) in ((50, 5, 4, 1 << 22), (50, 5, 4, 64), (267, 23, 4, 1 << 22), (10, 9, 6, 100)):
        tree = tree_mod.random_tree(np.random.default_rng(nq * d), depth, d)
        q = np.random.default_rng(nq).integers(0, 2, (nq, d - 1), dtype=np.uint8)

        def body(eng, tree=tree, q=q, depth=depth):
            t = share_in(eng, tree.T, RING64, "T")
            qq = share_in(eng, q, RING64, "q")
            return infer_batch(eng, levels_of(t, depth), qq)
        run = run_dealer(body, lane_limit=ll)
        out[f"infer_n{nq}_d{d}_h{depth}_ll{ll}"] = {"n": nq, "d": d, "depth": depth, "lane_limit": ll,
                                                    "records": run.transcript.records}
    with open(os.path.join(OUT, "transcripts.json"), "w") as fh:
        json.dump(out, fh)
    print("transcripts done")


def make_c2c3():
    rng = np.random.default_rng(1011)
    data = rng.integers(0, 2, size=(48842, 14), dtype=np.uint8)
    seed = (11_000).to_bytes(16, "little")
    t0 = time.time()
    T, F, dep, run = secure_train(data, TrainConfig(depth=7, heuristic="mpc"), seed)
    secs = time.time() - t0
    q = np.random.default_rng(7).integers(0, 2, (10_000, 13), dtype=np.uint8)
    tree = tree_mod.TreeState(7, T, F)

    def body(eng):
        t = share_in(eng, T, RING64, "T")
        qq = share_in(eng, q, RING64, "q")
        return infer_batch(eng, levels_of(t, 7), qq)
    t1 = time.time()
    irun = run_dealer(body)
    isecs = time.time() - t1
    preds = open_u64(irun.results, RING64)
    want = np.array([tree_mod.plaintext_infer(tree, r) for r in q], dtype=np.uint64)
    assert np.array_equal(preds, want)
    meta = {"train_seconds": secs, "infer_seconds": isecs, "cpu": os.cpu_count(),
            "train_metrics": _metrics_dict(run), "infer_metrics": _metrics_dict(irun)}
    np.savez_compressed(os.path.join(OUT, "c2c3.npz"), T=T, F=F, preds=preds,
                        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8))
    print(f"c2 {secs:.1f}s c3 {isecs:.1f}s")


def make_variants():
    """MPC trees with a Z_2^64 score ring and other tau (TrainConfig.score_ring /
    tau, train.py:57-65; cli --width / --tau)."""
    from obtree.ring import Ring
    arrays, meta = {}, []
    cases = []
    for i in range(6):
        data, depth = _battery_dataset(100 + i)
        cases.append((data, min(depth, 4), 64, 10))
    for i in range(4):
        data, depth = _battery_dataset(200 + i)
        cases.append((data, min(depth, 4), 32, 8))
    rng = np.random.default_rng(5)
    cases.append((rng.integers(0, 2, (1500, 6), dtype=np.uint8), 3, 64, 12))
    cases.append((rng.integers(0, 2, (2100, 5), dtype=np.uint8), 3, 32, 6))
    for k, (data, depth, width, tau) in enumerate(cases):
        seed = (9000 + k).to_bytes(16, "little")
        T, F, dep, _ = secure_train(data, TrainConfig(depth=depth, tau=tau, score_ring=Ring(width)), seed)
        arrays[f"data{k}"], arrays[f"T{k}"], arrays[f"F{k}"] = data, T, F
        meta.append({"depth": depth, "width": width, "tau": tau, "seed": seed.hex()})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "trees_variants.npz"), **arrays)
    print("variants done")


def make_tee():
    """Reference transcripts of the trusted-helper path (heuristic "tee")."""
    out = {}
    for (n, d, depth, policy) in ((60, 4, 3, "fixed"), (150, 6, 4, "fixed"), (33, 3, 1, "fixed"), (80, 4, 3, "grow")):
        data = np.random.default_rng(n + d + depth).integers(0, 2, (n, d), dtype=np.uint8)
        cfg = TrainConfig(depth=depth if policy == "fixed" else 1, heuristic="tee", policy=policy,
                          max_depth=depth if policy == "grow" else None)
        T, F, dep, run = secure_train(data, cfg, b"\x45" * 16)
        out[f"tee_n{n}_d{d}_h{depth}_{policy}"] = {"n": n, "d": d, "depth": depth, "policy": policy,
                                                   "trained_depth": dep, "T": T.tolist(), "F": F.tolist(),
                                                   "records": run.transcript.records}
    with open(os.path.join(OUT, "transcripts_tee.json"), "w") as fh:
        json.dump(out, fh)
    print("tee done")


def make_policies():
    """Depth policies on the MPC path (train.py:81-86): feature_cap as the
    reference's test_feature_cap_policy_uses_column_count (test_train.py:85-94,
    heuristic mpc here), and grow with the default cap (= column count) deep
    enough that the opened stop bit is AND-reduced over > 64 nodes."""
    arrays, meta = {}, []
    cases = [
        ("feature_cap_80x4", np.random.default_rng(6).integers(0, 2, (80, 4), dtype=np.uint8),
         TrainConfig(depth=1, policy="feature_cap"), b"\x0e" * 16),
        ("grow_default_cap_3000x10", np.random.default_rng(31).integers(0, 2, (3000, 10), dtype=np.uint8),
         TrainConfig(depth=1, policy="grow"), b"\x21" * 16),
    ]
    for k, (name, data, cfg, seed) in enumerate(cases):
        t0 = time.time()
        T, F, dep, _ = secure_train(data, cfg, seed)
        arrays[f"data{k}"], arrays[f"T{k}"], arrays[f"F{k}"] = data, T, F
        meta.append({"name": name, "policy": cfg.policy, "depth_arg": cfg.depth, "trained_depth": dep,
                     "seed": seed.hex()})
        print("policy", name, dep, f"{time.time() - t0:.1f}s")
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "trees_policy.npz"), **arrays)


def make_cli():
    """Run the reference CLI (obtree.cli.main) on small CSVs and record what
    it writes: stdout lines, tree_meta/metrics/tree JSON, predictions.csv,
    compare reports, bench tables and sha256 of the dealt share/seed files."""
    import contextlib
    import hashlib
    import io
    import tempfile
    from pathlib import Path

    from obtree import cli as ref_cli

    gdir = Path(OUT) / "cli"
    gdir.mkdir(exist_ok=True)
    rng = np.random.default_rng(2024)
    data = rng.integers(0, 2, (90, 6), dtype=np.uint8)
    data[:, -1] = data[:, 0] ^ (data[:, 2] & rng.integers(0, 2, 90, dtype=np.uint8))
    queries = rng.integers(0, 2, (40, 5), dtype=np.uint8)
    tree_mod.save_csv(gdir / "data.csv", data)
    tree_mod.save_csv(gdir / "queries.csv", queries)
    (gdir / "run.conf").write_text("# flag defaults\ndepth = 3\nseed = 99\nprofile = test\n")
    cases = {
        "train_mpc": ["train", "--data", "{g}/data.csv", "--depth", "3", "--seed", "7", "--profile", "test",
                      "--reveal", "--out", "{t}/train_mpc"],
        "train_tee": ["train", "--data", "{g}/data.csv", "--depth", "4", "--heuristic", "tee", "--seed", "0x0badcafe",
                      "--profile", "test", "--reveal", "--out", "{t}/train_tee"],
        "train_grow": ["train", "--data", "{g}/data.csv", "--policy", "grow", "--max-depth", "4", "--seed", "5",
                       "--profile", "test", "--reveal", "--out", "{t}/train_grow"],
        "train_conf": ["train", "--config", "{g}/run.conf", "--data", "{g}/data.csv", "--reveal",
                       "--out", "{t}/train_conf"],
        "infer_dir": ["infer", "--tree-dir", "{t}/train_mpc", "--queries", "{g}/queries.csv", "--seed", "7",
                      "--profile", "test", "--reveal", "--out", "{t}/infer_dir"],
        "infer_plain": ["infer", "--tree", "{t}/train_tee/tree.json", "--queries", "{g}/queries.csv", "--seed", "3",
                        "--profile", "test", "--reveal", "--out", "{t}/infer_plain"],
        "compare_mpc": ["compare", "--data", "{g}/data.csv", "--depth", "3", "--seed", "11",
                        "--out", "{t}/compare_mpc.json"],
        "compare_tee": ["compare", "--data", "{g}/data.csv", "--depth", "3", "--heuristic", "tee", "--seed", "11",
                        "--out", "{t}/compare_tee.json"],
        "deal_train": ["deal", "--data", "{g}/data.csv", "--depth", "3", "--seed", "21", "--out", "{t}/deal_train"],
        "train_deal": ["train", "--deal-dir", "{t}/deal_train", "--depth", "3", "--profile", "test", "--reveal",
                       "--out", "{t}/train_deal"],
        "bench_oaa": ["bench", "--suite", "oaa", "--lookups", "200", "--sizes", "1,8,64", "--out", "{t}/bench_oaa.json"],
        "bench_train": ["bench", "--suite", "train", "--rows", "64", "--cols", "5", "--depths", "2,3",
                        "--out", "{t}/bench_train.json"],
        "bench_infer": ["bench", "--suite", "infer", "--rows", "100", "--depths", "3,5", "--out",
                        "{t}/bench_infer.json"],
        "err_reveal_prod": ["train", "--data", "{g}/data.csv", "--reveal", "--out", "{t}/x"],
        "err_width": ["train", "--data", "{g}/data.csv", "--width", "4", "--out", "{t}/x"],
        "err_tolerance": ["compare", "--data", "{g}/data.csv", "--depth", "1", "--seed", "11", "--split", "0.5",
                          "--tolerance", "-1"],
    }
    files = ("tree.json", "tree_meta.json", "metrics.json", "predictions.csv")
    out = {}
    with tempfile.TemporaryDirectory() as t:
        for name, argv in cases.items():
            argv = [a.format(g=gdir, t=t) for a in argv]
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                code = ref_cli.main(argv)
            rec = {"argv": [a.replace(str(gdir), "{g}").replace(t, "{t}") for a in argv], "exit": code,
                   "stdout": buf.getvalue().replace(t, "{t}"), "files": {}}
            target = Path(argv[argv.index("--out") + 1]) if "--out" in argv else None
            if target is not None and target.is_dir():
                for f in files:
                    if (target / f).exists():
                        rec["files"][f] = (target / f).read_text()
                if name.startswith("deal"):
                    for p in sorted(target.rglob("*")):
                        if p.is_file() and p.name != "material.bin":
                            rec["files"][str(p.relative_to(target))] = hashlib.sha256(p.read_bytes()).hexdigest()
            elif target is not None and target.exists():
                rec["files"]["report"] = target.read_text()
            out[name] = rec
            print("cli", name, code)
    with open(gdir / "cli.json", "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def make_deal():
    """The reference dealer's outputs for the on-disk row:
    training/inference material needs for a few shapes (train.py:309-346,
    infer.py:38-43), the reference CLI's deal directory for tests/golden/cli
    data.csv (depth 3, seed 21) -- every file except the three material.bin,
    which are recorded by sha256 and size (the repo regenerates them) -- and
    the revealed tree the reference trains from that directory."""
    import hashlib
    import shutil
    import tempfile
    from pathlib import Path

    from obtree import cli as ref_cli
    from obtree.infer import inference_needs
    from obtree.ring import Ring
    from obtree.train import training_needs

    cases = {"train_90x6_d3": (90, 6, TrainConfig(depth=3)),
             "train_90x6_tee_d4": (90, 6, TrainConfig(depth=4, heuristic="tee")),
             "train_267x23_d4": (267, 23, TrainConfig(depth=4)),
             "train_1500x8_d5": (1500, 8, TrainConfig(depth=5)),
             "train_4000x10_s64_t12_d4": (4000, 10, TrainConfig(depth=4, tau=12, score_ring=Ring(64))),
             "train_300x5_feature_cap": (300, 5, TrainConfig(policy="feature_cap"))}
    out = {"training": {}, "inference": {}}
    for name, (n, d, cfg) in cases.items():
        out["training"][name] = {"n": n, "d": d, "depth": cfg.depth, "tau": cfg.tau, "heuristic": cfg.heuristic,
                                 "policy": cfg.policy, "score_width": cfg.score_ring.width,
                                 "needs": [[list(k), v] for k, v in sorted(training_needs(n, d, cfg).items(),
                                                                           key=lambda kv: repr(kv[0]))]}
    for nq, depth, ncol in ((40, 3, 6), (10_000, 7, 14)):
        out["inference"][f"{nq}x{ncol}_d{depth}"] = {
            "n": nq, "depth": depth, "n_columns": ncol,
            "needs": [[list(k), v] for k, v in sorted(inference_needs(nq, depth, ncol).items(),
                                                      key=lambda kv: repr(kv[0]))]}
    gdir = Path(OUT) / "deal_train"
    if gdir.exists():
        shutil.rmtree(gdir)
    with tempfile.TemporaryDirectory() as t:
        deal = Path(t) / "deal"
        assert ref_cli.main(["deal", "--data", str(Path(OUT) / "cli" / "data.csv"), "--depth", "3", "--seed", "21",
                             "--out", str(deal)]) == 0
        mats = {}
        for p in sorted(deal.rglob("*")):
            if p.is_dir():
                continue
            rel = p.relative_to(deal)
            if p.name == "material.bin":
                raw = p.read_bytes()
                mats[str(rel)] = {"sha256": hashlib.sha256(raw).hexdigest(), "bytes": len(raw)}
            else:
                (gdir / rel).parent.mkdir(parents=True, exist_ok=True)
                shutil.copy(p, gdir / rel)
        run = Path(t) / "train"
        assert ref_cli.main(["train", "--deal-dir", str(deal), "--depth", "3", "--profile", "test", "--reveal",
                             "--out", str(run)]) == 0
        tree = json.loads((run / "tree.json").read_text())
    out["deal_train"] = {"argv": "deal --data cli/data.csv --depth 3 --seed 21", "material": mats,
                         "material_seed_label": "deal/material", "tree": tree}
    with open(os.path.join(OUT, "deal.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("deal", len(mats), "material files")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c2", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    steps = {"policies": make_policies, "cli": make_cli, "variants": make_variants, "deal": make_deal,
             "tee": make_tee,
             "kats": make_kats, "trees": make_trees, "infer": make_infer,
             "transcripts": make_transcripts, "c2c3": make_c2c3}
    for name, fn in steps.items():
        if a.only and name != a.only:
            continue
        if a.skip_c2 and name == "c2c3":
            continue
        fn()
