"""Host logic (CPU): transcript ledger vs the reference's transcripts, seed
derivation and filler stream vs the reference, share conversions, config
helpers, and the C-ABI library's exported symbol set."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_json, golden_npz
from paper_2305_00645_b200 import ledger as L
from paper_2305_00645_b200 import _native
from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values
from paper_2305_00645_b200.shares import (RING32, RING64, ShareError, components_from_pairs, pairs_from_components,
                                          reconstruct)
from paper_2305_00645_b200.train import TrainConfig, counter_shift, levels_of, resolved_depth


def _replay(name, v):
    led = L.Ledger(v.get("lane_limit", L.REF_LANE_LIMIT))
    if name.startswith("train"):
        led.train(v["n"], v["d"] - 1, v["depth"])
    elif name.startswith("infer"):
        led.infer(v["n"], v["d"] - 1, v["depth"])
    elif name.startswith("oaa"):
        led.oaa(v["n"], v["m"], 64)
        led.row_lookup(v["n"], v["m"], 64)
    elif name.startswith("gadgets"):
        w = int(name.split("_w")[1])
        n = 37
        led.eq(n, w), led.eq(n, w), led.lt(n, w), led.lt(n, w)
        led.b2a(n), led.select(n, n, w), led.truncate(n, w, 3), led.mul(n, w)
    elif name == "division_argmin":
        led.division(11, 32, 10)
        led.argmin(5, 13, 32)
    return led


def test_ledger_reproduces_reference_transcripts_record_for_record():
    g = golden_json("transcripts.json")
    assert len(g) >= 15
    for name, v in g.items():
        led = _replay(name, v)
        assert led.transcript.records == [tuple(r) for r in v["records"]], name


def test_ledger_c2_c3_totals_match_reference():
    _, meta = golden_npz("c2c3.npz")
    m = L.train_metrics(48842, 13, 7)
    ref = meta["train_metrics"]
    assert m.rounds == ref["rounds"] == 2147
    assert m.bytes_by_pair == ref["bytes_by_pair"] and m.bytes_by_tag == ref["bytes_by_tag"]
    assert m.rounds_by_tag == ref["rounds_by_tag"]
    assert m.sent_by_party(1) == 1615326277
    mi = L.infer_metrics(10_000, 13, 7)
    assert mi.rounds == meta["infer_metrics"]["rounds"] == 126
    assert mi.bytes_by_pair == meta["infer_metrics"]["bytes_by_pair"]


def test_device_schedule_same_bytes_fewer_rounds():
    ref = L.train_metrics(48842, 13, 7)
    dev = L.train_metrics(48842, 13, 7, lane_limit=None)
    assert dev.sent_by_party(1) == ref.sent_by_party(1)
    assert dev.rounds < ref.rounds


def test_transcript_shape_only_depends_on_public_sizes():
    a = L.Ledger()
    a.train(50, 3, 3)
    b = L.Ledger()
    b.train(50, 3, 3)
    assert a.transcript.records == b.transcript.records


def test_seeds_and_filler_match_reference():
    kats = golden_json("kats.json")
    for master_hex, want in kats["seeds"].items():
        s = SeedSetup.from_master(bytes.fromhex(master_hex))
        assert {str(i): s.pair_seeds[i].hex() for i in (1, 2, 3)} == want["pair"]
        assert s.filler_seed.hex() == want["filler"]
        assert filler_values(s.filler_seed, 127, 14).tolist() == want["filler_values_127_14"]
        assert filler_values(s.filler_seed, 1023, 33).tolist() == want["filler_values_1023_33"]


def test_counter_shift_and_config_helpers():
    kats = golden_json("kats.json")["counter_shift"]
    for n, want in kats.items():
        assert counter_shift(int(n), TrainConfig()) == want
        assert L.counter_shift(int(n)) == want
    assert resolved_depth(TrainConfig(depth=3), 9) == 3
    assert resolved_depth(TrainConfig(policy="feature_cap"), 4) == 4
    assert resolved_depth(TrainConfig(policy="grow", max_depth=5), 9) == 5
    from paper_2305_00645_b200.shares import AVec

    vec = AVec(RING64, np.arange(7, dtype=np.uint64), np.zeros(7, dtype=np.uint64))
    assert [p.size for p in levels_of(vec, 3)] == [1, 2, 4]  # test_train.py:110-113


def test_share_conversion_and_consistency_check():
    rng = np.random.default_rng(0)
    comp = rng.integers(0, 1 << 63, (3, 11), dtype=np.uint64)
    pairs = pairs_from_components(comp)
    assert np.array_equal(components_from_pairs(pairs), comp)
    bad = [(pairs[0][0], pairs[0][1] ^ np.uint64(1)), pairs[1], pairs[2]]
    with pytest.raises(ShareError):
        components_from_pairs(bad)
    assert np.array_equal(reconstruct(comp, RING32), (comp[0] + comp[1] + comp[2]) & np.uint64(0xFFFFFFFF))


def test_native_host_staging_of_party_pairs():
    """gt_stage_pairs (host threads, no device work): the drop-in's pinned
    staging equals components_from_pairs, and an inconsistent pair raises
    ShareError like the reference's replication check (rss.py:222-228)."""
    from paper_2305_00645_b200.shares import stage_pairs

    rng = np.random.default_rng(1)
    comp = rng.integers(0, 1 << 63, (3, 300_001), dtype=np.uint64)  # several 1 MB slices per component
    pairs = pairs_from_components(comp)
    out = np.empty_like(comp)
    stage_pairs(pairs, out)
    assert np.array_equal(out, comp)
    bad = [pairs[0], (pairs[1][0], pairs[1][1].copy()), pairs[2]]
    bad[1][1][299_999] ^= np.uint64(1)
    with pytest.raises(ShareError):
        stage_pairs(bad, out)
    stage_pairs(bad, out, check=False)  # unchecked staging copies the lo components
    assert np.array_equal(out, comp)
    stage_pairs(pairs, None)  # the check alone (what the drop-in runs while the device trains)
    with pytest.raises(ShareError):
        stage_pairs(bad, None)


def test_run_local_party_threads_reused_errors_propagate():
    """run_local runs the three bodies on persistent party threads: results
    come back per party, a body's exception reaches the caller (the others
    see the broken rendezvous, as rss.py:518-541), the threads are reused by
    the next call, and a nested run_local gets fresh threads."""
    import threading

    from paper_2305_00645_b200 import engine

    names = []

    def ok(eng):
        names.append(threading.current_thread().name)
        return eng.party * 10

    run = engine.run_local(ok, seeds=5)
    assert run.results == [10, 20, 30] and sorted(names) == ["party1", "party2", "party3"]
    idents = {t.ident for t in threading.enumerate() if t.name.startswith("party")}

    def boom(eng):
        if eng.party == 2:
            raise ValueError("party 2 failed")
        return eng._bridge.call(eng.party, "x", None, lambda p: [0, 0, 0])

    with pytest.raises(ValueError, match="party 2 failed"):
        engine.run_local(boom, seeds=5)
    assert engine.run_local(ok, seeds=5).results == [10, 20, 30]
    assert idents <= {t.ident for t in threading.enumerate()}

    def nested(eng):
        return engine.run_local(ok, seeds=6).results[eng.party - 1]

    assert engine.run_local(nested, seeds=5).results == [10, 20, 30]


def test_division_params_match_reference():
    assert L.div_params(32, 10) == {"bound": 20, "ti": 14, "sigma": 7, "kf": 17, "iters": 6, "w0": 47746}
    with pytest.raises(ValueError):
        L.div_params(12, 10)  # test_gadgets.py:197-199


def test_native_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "gtree_b200.h")).read()
    declared = set(re.findall(r"\b(gt_[a-z0-9_]+)\s*\(", header)) - {"gt_allreduce_fn"}
    lib = ctypes.CDLL(_native.LIB_PATH)
    for sym in sorted(declared):
        assert hasattr(lib, sym), sym
    assert declared == set(_native.EXPORTS)
    assert lib.gt_abi_version() == _native.ABI_VERSION


def test_product_has_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2305_00645_b200.train import train_components

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        train_components(np.zeros((3, 4, 2), np.uint64), np.zeros((3, 4), np.uint64), TrainConfig(depth=2),
                         SeedSetup.from_int(1), b"\x00" * 16)


def test_trusted_helper_decisions_reproduce_reference_plaintext_trees():
    """enclave.split_decisions / majority_labels (the tee helper, host side)
    driven through the plaintext level loop (tree.py:289-325) reproduce the
    reference's plaintext_train trees (golden oT/oF) on every golden case."""
    from conftest import golden_npz
    from oracle import shadow
    from paper_2305_00645_b200 import enclave as E

    z, meta = golden_npz("trees_mpc.npz")
    for k, m in enumerate(meta):
        data, depth = z[f"data{k}"], m["depth"]
        X, y = data[:, :-1], data[:, -1]
        n, nf = X.shape
        setup = SeedSetup.from_master(derive_seed(bytes.fromhex(m["seed"]), "run"))
        fill = filler_values(setup.filler_seed, (1 << depth) - 1, data.shape[1])
        T = np.zeros((1 << depth) - 1, dtype=np.uint64)
        F = np.zeros_like(T)
        node = np.zeros(n, dtype=np.int64)
        types = np.array([E.F_LEAF])
        gam = np.ones((1, nf), dtype=bool)
        eff_prev = None
        for level in range(depth):
            nn, off = 1 << level, (1 << level) - 1
            C = shadow.node_counters(X, y, node, nn)
            eff = C.copy()
            if level:
                empty = (C[:, 0, 0] + C[:, 0, 1]) == 0
                eff[empty] = eff_prev[np.arange(nn)[empty] // 2]
            if level == depth - 1:
                T[off:off + nn] = E.majority_labels(eff)
                F[off:off + nn] = types
                break
            sd, new_f, is_int, new_g = E.split_decisions(C, gam, types)
            T[off:off + nn] = np.where(is_int, sd, fill[off:off + nn])
            F[off:off + nn] = new_f
            sf = np.where(node >= 0, np.where(is_int, sd.astype(np.int64), -1)[np.maximum(node, 0)], -1)
            go = np.where(sf >= 0, X[np.arange(n), np.maximum(sf, 0)], 0)
            node = np.where(sf >= 0, 2 * node + go, -1)
            types = np.repeat(np.where(is_int, E.F_LEAF, E.F_DUMMY), 2)
            gam = np.repeat(new_g, 2, axis=0)
            eff_prev = eff
        assert np.array_equal(T, z[f"oT{k}"]) and np.array_equal(F, z[f"oF{k}"]), m["name"]


def test_ledger_tee_transcripts_match_reference():
    g = golden_json("transcripts_tee.json")
    for name, v in g.items():
        led = L.Ledger()
        d = led.train(v["n"], v["d"] - 1, v["depth"], policy=v["policy"], heuristic="tee",
                      grow_stop_level=v["trained_depth"] - 1)
        assert d == v["trained_depth"]
        assert led.transcript.records == [tuple(r) for r in v["records"]], name
