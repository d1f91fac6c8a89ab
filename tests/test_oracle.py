"""Pin the oracle to the reference (CPU).  The oracle is trusted only because
these tests hold: Random123 KATs for the PRG, the reference's own frozen
gadget values (tests/golden/kats.json, test_gadgets.py / test_oaa.py), and
the revealed trees / predictions of reference runs (tests/golden/*.npz)."""

import numpy as np
import pytest

import oracle
from oracle import shadow
from conftest import KEYS, golden_json, golden_npz, opened, opened_bits, ref_cases, run_keys, share, share_bits


def test_philox_random123_kats():
    assert oracle.philox([0, 0, 0, 0], (0, 0)) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    m = 0xFFFFFFFF
    assert oracle.philox([m] * 4, (m, m)) == (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)
    assert oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], (0xA4093822, 0x299F31D0)) == (
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)


def test_exhaustive_width8_primitives():
    # test_acceptance.py:79-120 criterion 1: eq/lt/mul/b2a/select over all 2^16 pairs
    rng = np.random.default_rng(1)
    g = np.arange(256, dtype=np.uint64)
    xs, ys = [a.ravel() for a in np.meshgrid(g, g)]
    X, Y = share(xs, rng, 8), share(ys, rng, 8)
    e = oracle.eq(8, X, Y, k=KEYS, op=0x80000001)
    assert np.array_equal(opened_bits(e), (xs == ys).astype(np.uint8))
    assert np.array_equal(opened(oracle.mul(8, X, Y, KEYS, 0x80000002), 8), (xs * ys) % 256)
    assert np.array_equal(opened(oracle.b2a(8, e, KEYS, 0x80000003), 8), (xs == ys).astype(np.uint64))
    assert np.array_equal(opened_bits(oracle.lt(8, X, Y, k=KEYS, op=0x80000004)), (xs < ys).astype(np.uint8))
    cond = rng.integers(0, 2, xs.size, dtype=np.uint8)
    sel = oracle.select(8, X, Y, share_bits(cond, rng), KEYS, 0x80000005)
    assert np.array_equal(opened(sel, 8), np.where(cond == 1, ys, xs))


def test_division_matches_reference_kats():
    kat = golden_json("kats.json")["division_tau10_w32"]
    rng = np.random.default_rng(2)
    p = np.array(kat["p"], dtype=np.uint64)
    q = np.array(kat["q"], dtype=np.uint64)
    got = opened(oracle.division(32, share(p, rng, 32), share(q, rng, 32), 10, KEYS, 0x80000010), 32)
    assert got.tolist() == kat["out"]
    assert got[:5].tolist() == [3217, 1024, 512, 2000, 4096]  # test_gadgets.py:152-161


def test_truncate_argmin_oaa_kats():
    kats = golden_json("kats.json")
    rng = np.random.default_rng(3)
    for width, key in ((32, "truncate_w32"), (64, "truncate_w64")):
        x = np.array(kats[key]["x"], dtype=np.uint64)
        for k, want in kats[key]["out"].items():
            got = opened(oracle.truncate(width, share(x, rng, width), int(k), KEYS, 0x80000020 + int(k)), width)
            assert got.tolist() == want
            assert got.tolist() == (x >> np.uint64(int(k))).tolist()
    for case in kats["argmin_w32"]:
        sc = np.array(case["scores"], dtype=np.uint64)
        av = np.array(case["avail"], dtype=np.uint8)
        got = opened(oracle.argmin(32, share(sc, rng, 32), share_bits(av, rng), 1 << 11, KEYS, 0x80000030))
        assert got.tolist() == case["out"]
    o = kats["oaa_oob_w8"]
    got = oracle.oaa(8, share(np.array(o["table"], dtype=np.uint64), rng, 8),
                     share(np.array(o["idx"], dtype=np.uint64), rng, 8), KEYS, 0x80000040)
    assert opened(got, 8).tolist() == o["out"] == [5, 0, 0, 7]


def test_shadow_reproduces_reference_mpc_trees():
    from paper_2305_00645_b200.seeds import filler_values

    for m, data, T, F in ref_cases():
        setup, _, _ = run_keys(bytes.fromhex(m["seed"]))
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        t, f = shadow.mpc_train(data, m["depth"], fill)
        assert np.array_equal(t, T) and np.array_equal(f, F), m["name"]


def test_oracle_protocol_reproduces_reference_mpc_trees():
    from paper_2305_00645_b200.seeds import filler_values

    rng = np.random.default_rng(4)
    for m, data, T, F in ref_cases():
        setup, _, keys = run_keys(bytes.fromhex(m["seed"]))
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        t, f, d = oracle.train(share(data[:, :-1], rng), share(data[:, -1], rng), fill, m["depth"], keys)
        assert d == m["depth"]
        assert np.array_equal(opened(t), T) and np.array_equal(opened(f), F), m["name"]


def test_oracle_c2_adult_depth7_and_c3():
    from paper_2305_00645_b200.seeds import filler_values

    z, meta = golden_npz("c2c3.npz")
    data = np.random.default_rng(1011).integers(0, 2, size=(48842, 14), dtype=np.uint8)
    setup, _, keys = run_keys((11_000).to_bytes(16, "little"))
    fill = filler_values(setup.filler_seed, 127, 14)
    t, f = shadow.mpc_train(data, 7, fill)
    assert np.array_equal(t, z["T"]) and np.array_equal(f, z["F"])
    rng = np.random.default_rng(5)
    T, F, _ = oracle.train(share(data[:, :-1], rng), share(data[:, -1], rng), fill, 7, keys)
    assert np.array_equal(opened(T), z["T"]) and np.array_equal(opened(F), z["F"])
    q = np.random.default_rng(7).integers(0, 2, (10_000, 13), dtype=np.uint8)
    out, _ = oracle.infer(share(z["T"], rng), 7, share(q, rng), keys)
    assert np.array_equal(opened(out), z["preds"])
    assert np.array_equal(shadow.plaintext_infer(z["T"], 7, q), z["preds"])


def test_oracle_inference_matches_reference():
    z, meta = golden_npz("infer.npz")
    rng = np.random.default_rng(6)
    for k, m in enumerate(meta):
        T, q, p = z[f"T{k}"], z[f"q{k}"], z[f"p{k}"]
        out, _ = oracle.infer(share(T, rng), m["depth"], share(q, rng), KEYS)
        assert np.array_equal(opened(out), p)
        assert np.array_equal(shadow.plaintext_infer(T, m["depth"], q), p)


def test_oracle_shares_independent_of_input_sharing():
    # revealed outputs do not depend on how the inputs were shared
    m, data, T, F = next(iter(ref_cases()))
    from paper_2305_00645_b200.seeds import filler_values

    setup, _, keys = run_keys(bytes.fromhex(m["seed"]))
    fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
    outs = []
    for s in (10, 11):
        rng = np.random.default_rng(s)
        t, f, _ = oracle.train(share(data[:, :-1], rng), share(data[:, -1], rng), fill, m["depth"], keys)
        outs.append((opened(t), opened(f)))
    assert all(np.array_equal(a, b) for a, b in zip(outs[0], outs[1]))


def test_oracle_dot_reshare_same_revealed_trees():
    from paper_2305_00645_b200.seeds import filler_values

    rng = np.random.default_rng(13)
    for m, data, T, F in list(ref_cases())[:20]:
        setup, _, keys = run_keys(bytes.fromhex(m["seed"]))
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        t, f, _ = oracle.train(share(data[:, :-1], rng), share(data[:, -1], rng), fill, m["depth"], keys,
                               count_reshare=1)
        assert np.array_equal(opened(t), T) and np.array_equal(opened(f), F), m["name"]


def test_oracle_score_ring64_and_tau_variants_match_reference():
    from paper_2305_00645_b200.seeds import filler_values

    z, meta = golden_npz("trees_variants.npz")
    rng = np.random.default_rng(14)
    for k, m in enumerate(meta):
        data = z[f"data{k}"]
        setup, _, keys = run_keys(bytes.fromhex(m["seed"]))
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        t, f, _ = oracle.train(share(data[:, :-1], rng), share(data[:, -1], rng), fill, m["depth"], keys,
                               tau=m["tau"], score_width=m["width"])
        assert np.array_equal(opened(t), z[f"T{k}"]) and np.array_equal(opened(f), z[f"F{k}"]), m
