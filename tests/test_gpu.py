"""Device parity (B200): every kernel vs the oracle share-for-share (same
randomness schedule) and vs the reference's revealed outputs (golden
fixtures).  All calls go through the C ABI (libgtree_b200.so)."""

import numpy as np
import pytest
import torch

import oracle
from oracle import shadow
from conftest import KEYS, golden_npz, opened, opened_bits, ref_cases, run_keys, share, share_bits

pytestmark = pytest.mark.gpu

from paper_2305_00645_b200 import gadgets as G  # noqa: E402
from paper_2305_00645_b200.seeds import filler_values, make_keys  # noqa: E402
from paper_2305_00645_b200.shares import from_device, to_device  # noqa: E402


def _keys():
    from paper_2305_00645_b200._native import gt_keys

    k = gt_keys()
    k.dealer.k0, k.dealer.k1 = KEYS[0]
    for i in range(3):
        k.pair[i].k0, k.pair[i].k1 = KEYS[i + 1]
    return k


def _u8(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


def _b(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("width", [8, 32, 64])
def test_gadgets_share_exact_vs_oracle(width):
    rng = np.random.default_rng(width)
    n = 3001
    m = (1 << width) - 1 if width < 64 else (1 << 64) - 1
    xv = rng.integers(0, 1 << min(width, 63), n, dtype=np.uint64)
    yv = np.where(rng.random(n) < 0.3, xv, rng.integers(0, 1 << min(width, 63), n, dtype=np.uint64))
    X, Y = share(xv, rng, width), share(yv, rng, width)
    bits = share_bits(rng.integers(0, 2, n), rng)
    K = _keys()
    dX, dY, dB = to_device(X), to_device(Y), _u8(bits)
    op = 0x80000100
    assert np.array_equal(from_device(G.mul(width, dX, dY, K, op)), oracle.mul(width, X, Y, KEYS, op))
    assert np.array_equal(_b(G.eq(width, dX, dY, keys=K, op=op + 1)), oracle.eq(width, X, Y, k=KEYS, op=op + 1))
    pub = to_device(yv)
    assert np.array_equal(_b(G.eq(width, dX, None, pub, keys=K, op=op + 2)), oracle.eq(width, X, None, yv, k=KEYS, op=op + 2))
    got_lt = _b(G.lt(width, dX, dY, keys=K, op=op + 3))
    assert np.array_equal(got_lt, oracle.lt(width, X, Y, k=KEYS, op=op + 3))
    assert np.array_equal(opened_bits(got_lt), (xv < yv).astype(np.uint8))
    assert np.array_equal(from_device(G.b2a(width, dB, keys=K, op=op + 4)), oracle.b2a(width, bits, KEYS, op + 4))
    # grouped select: 3 payload elements per condition
    W1, W2 = share(np.repeat(xv, 3), rng, width), share(np.repeat(yv, 3), rng, width)
    got = from_device(G.select_share(width, to_device(W1), to_device(W2), dB, keys=K, op=op + 5))
    assert np.array_equal(got, oracle.select(width, W1, W2, bits, KEYS, op + 5))
    for k in (1, 3, width // 2, width - 1):
        got = from_device(G.truncate(width, dX, k, keys=K, op=op + 6 + k))
        assert np.array_equal(got, oracle.truncate(width, X, k, KEYS, op + 6 + k))
        assert np.array_equal(opened(got, width), xv >> np.uint64(k))


def test_exhaustive_width8_revealed_on_device():
    rng = np.random.default_rng(8)
    g = np.arange(256, dtype=np.uint64)
    xs, ys = [a.ravel() for a in np.meshgrid(g, g)]
    X, Y = to_device(share(xs, rng, 8)), to_device(share(ys, rng, 8))
    K = _keys()
    e = G.eq(8, X, Y, keys=K, op=0x80000200)
    assert np.array_equal(opened_bits(_b(e)), (xs == ys).astype(np.uint8))
    assert np.array_equal(opened(from_device(G.mul(8, X, Y, K, 0x80000201)), 8), (xs * ys) % 256)
    assert np.array_equal(opened(from_device(G.b2a(8, e, keys=K, op=0x80000202)), 8), (xs == ys).astype(np.uint64))
    assert np.array_equal(opened_bits(_b(G.lt(8, X, Y, keys=K, op=0x80000203))), (xs < ys).astype(np.uint8))


def test_division_argmin_oaa_kats_and_share_exact():
    from conftest import golden_json

    kats = golden_json("kats.json")
    rng = np.random.default_rng(9)
    K = _keys()
    d = kats["division_tau10_w32"]
    P, Q = share(np.array(d["p"], dtype=np.uint64), rng, 32), share(np.array(d["q"], dtype=np.uint64), rng, 32)
    got = from_device(G.division(32, to_device(P), to_device(Q), 10, keys=K, op=0x80000300))
    assert opened(got, 32).tolist() == d["out"]
    assert np.array_equal(got, oracle.division(32, P, Q, 10, KEYS, 0x80000300))
    for case in kats["argmin_w32"]:
        sc = share(np.array(case["scores"], dtype=np.uint64), rng, 32)
        av = share_bits(np.array(case["avail"], dtype=np.uint8), rng)
        got = from_device(G.argmin_masked(32, to_device(sc), _u8(av), 1 << 11, keys=K, op=0x80000301))
        assert opened(got).tolist() == case["out"]
        assert np.array_equal(got, oracle.argmin(32, sc, av, 1 << 11, KEYS, 0x80000301))
    o = kats["oaa_oob_w8"]
    t, i = share(np.array(o["table"], dtype=np.uint64), rng, 8), share(np.array(o["idx"], dtype=np.uint64), rng, 8)
    got = from_device(G.oaa(8, to_device(t), to_device(i), keys=K, op=0x80000302))
    assert opened(got, 8).tolist() == [5, 0, 0, 7]
    assert np.array_equal(got, oracle.oaa(8, t, i, KEYS, 0x80000302))
    rows = share(rng.integers(0, 1 << 40, (500, 13), dtype=np.uint64), rng)
    idx = share(rng.integers(0, 15, 500, dtype=np.uint64), rng)
    got = from_device(G.row_lookup(64, to_device(rows), to_device(idx), keys=K, op=0x80000303))
    assert np.array_equal(got, oracle.row_lookup(64, rows, idx, KEYS, 0x80000303))


def _device_train(data, depth, seed, rng, **cfgkw):
    from paper_2305_00645_b200.train import TrainConfig, train_components

    setup, k, keys = run_keys(seed)
    from paper_2305_00645_b200.seeds import derive_seed

    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    T, F, d = train_components(X, Y, TrainConfig(depth=depth, **cfgkw), setup, derive_seed(seed, "deal"))
    return X, Y, T, F, d, setup, keys


def test_training_matches_reference_trees_and_oracle_shares():
    rng = np.random.default_rng(10)
    for m, data, Tref, Fref in ref_cases():
        seed = bytes.fromhex(m["seed"])
        X, Y, T, F, d, setup, keys = _device_train(data, m["depth"], seed, rng)
        assert d == m["depth"]
        assert np.array_equal(opened(T), Tref) and np.array_equal(opened(F), Fref), m["name"]
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        To, Fo, _ = oracle.train(X, Y, fill, m["depth"], keys)
        assert np.array_equal(T, To) and np.array_equal(F, Fo), m["name"]


def test_training_c2_adult_depth7():
    z, meta = golden_npz("c2c3.npz")
    data = np.random.default_rng(1011).integers(0, 2, size=(48842, 14), dtype=np.uint8)
    rng = np.random.default_rng(11)
    X, Y, T, F, d, setup, keys = _device_train(data, 7, (11_000).to_bytes(16, "little"), rng)
    assert np.array_equal(opened(T), z["T"]) and np.array_equal(opened(F), z["F"])
    fill = filler_values(setup.filler_seed, 127, 14)
    To, Fo, _ = oracle.train(X, Y, fill, 7, keys)
    assert np.array_equal(T, To) and np.array_equal(F, Fo)


def test_grow_policy_matches_oracle():
    rng = np.random.default_rng(12)
    data = np.zeros((40, 4), dtype=np.uint8)
    data[:, 0] = np.arange(40) % 2  # features vary, label constant (test_train.py:65-71)
    X, Y, T, F, d, setup, keys = _device_train(data, 1, b"\x0c" * 16, rng, policy="grow", max_depth=3)
    assert d == 1 and opened(F).tolist() == [1] and opened(T).tolist() == [0]
    data = rng.integers(0, 2, (80, 4), dtype=np.uint8)
    X, Y, T, F, d, setup, keys = _device_train(data, 1, b"\x0d" * 16, rng, policy="grow", max_depth=3)
    fill = filler_values(setup.filler_seed, 7, 4)
    To, Fo, do = oracle.train(X, Y, fill, 3, keys, policy=1)
    assert d == do
    slots = (1 << d) - 1
    assert np.array_equal(T, To[:, :slots]) and np.array_equal(F, Fo[:, :slots])


def test_inference_matches_reference_and_oracle():
    from paper_2305_00645_b200.infer import infer_components

    z, meta = golden_npz("infer.npz")
    rng = np.random.default_rng(13)
    K = _keys()
    for k, m in enumerate(meta):
        T, q, p = share(z[f"T{k}"], rng), share(z[f"q{k}"], rng), z[f"p{k}"]
        out, slot = infer_components(T, m["depth"], q, K)
        assert np.array_equal(opened(out), p)
        oo, os_ = oracle.infer(T, m["depth"], q, KEYS)
        assert np.array_equal(out, oo) and np.array_equal(slot, os_)
    z, _ = golden_npz("c2c3.npz")
    q = np.random.default_rng(7).integers(0, 2, (10_000, 13), dtype=np.uint8)
    T, Q = share(z["T"], rng), share(q, rng)
    out, slot = infer_components(T, 7, Q, K, instance_base=0)
    assert np.array_equal(opened(out), z["preds"])
    oo, _ = oracle.infer(T, 7, Q, KEYS)
    assert np.array_equal(out, oo)
    # instance sharding: two halves keyed by global index == the whole batch
    a, _ = infer_components(T, 7, Q[:, :4000], K, instance_base=0)
    b, _ = infer_components(T, 7, Q[:, 4000:], K, instance_base=4000)
    assert np.array_equal(np.concatenate([a, b], axis=1), out)


def test_inference_large_random_tree_vs_plaintext():
    from paper_2305_00645_b200.infer import infer_components

    rng = np.random.default_rng(14)
    Tv, Fv = shadow.random_tree(np.random.default_rng(10), 10, 33)
    q = rng.integers(0, 2, (200_000, 32), dtype=np.uint8)
    out, _ = infer_components(share(Tv, rng), 10, share(q, rng), _keys())
    assert np.array_equal(opened(out), shadow.plaintext_infer(Tv, 10, q))


def test_dropin_run_local_train_and_infer():
    from conftest import golden_json
    from paper_2305_00645_b200 import TrainConfig, infer_batch, levels_of, run_local, train_tree
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from paper_2305_00645_b200.shares import AVec, RING64, pairs_from_components

    data = np.random.default_rng(60 + 4 + 3).integers(0, 2, (60, 4), dtype=np.uint8)
    seed = b"\x44" * 16
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    rng = np.random.default_rng(15)
    xp = pairs_from_components(share(data[:, :-1], rng))
    yp = pairs_from_components(share(data[:, -1], rng))

    def body(eng):
        X = AVec(RING64, *xp[eng.party - 1])
        y = AVec(RING64, *yp[eng.party - 1])
        r = train_tree(eng, X, y, TrainConfig(depth=3))
        return r

    run = run_local(body, seeds=setup, dealer_seed=derive_seed(seed, "deal"))
    T = sum(r.T.lo for r in run.results)
    ref = golden_json("transcripts.json")["train_n60_d4_h3_ll4194304"]
    assert run.transcript.records == [tuple(r) for r in ref["records"]]
    want_T, want_F = shadow.mpc_train(data, 3, filler_values(setup.filler_seed, 7, 4))
    assert np.array_equal(T, want_T)
    for r in run.results:  # replication consistency of the returned pairs
        assert r.T.lo.shape == (7,)
    q = rng.integers(0, 2, (50, 3), dtype=np.uint8)
    qp = pairs_from_components(share(q, rng))
    tp = [(r.T.lo, r.T.hi) for r in run.results]

    def body2(eng):
        t = AVec(RING64, *tp[eng.party - 1])
        return infer_batch(eng, levels_of(t, 3), AVec(RING64, *qp[eng.party - 1]))

    run2 = run_local(body2, seeds=setup)
    got = sum(r.lo for r in run2.results)
    assert np.array_equal(got, shadow.plaintext_infer(want_T, 3, q))


def test_dropin_run_local_c2_twice_equals_reference_tree():
    """The drop-in API at the C2 shape (48 842 x 13, depth 7): per-party host
    AVecs through run_local + train_tree, twice (the second call reuses the
    cached trainer and its pinned staging), both equal to the reference's C2
    tree (tests/golden/c2c3.npz)."""
    from paper_2305_00645_b200 import TrainConfig, run_local, train_tree
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from paper_2305_00645_b200.shares import AVec, RING64

    z, _ = golden_npz("c2c3.npz")
    data = np.random.default_rng(1011).integers(0, 2, size=(48842, 14), dtype=np.uint8)
    seed = (11_000).to_bytes(16, "little")
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    for it in range(2):
        rng = np.random.default_rng(70 + it)
        X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)

        def body(eng):
            p = eng.party
            return train_tree(eng, AVec(RING64, X[p - 1], X[p % 3]), AVec(RING64, Y[p - 1], Y[p % 3]),
                              TrainConfig(depth=7))

        run = run_local(body, seeds=setup, dealer_seed=derive_seed(seed, "deal"))
        assert np.array_equal(sum(r.T.lo for r in run.results), z["T"])
        assert np.array_equal(sum(r.F.lo for r in run.results), z["F"])


def test_dropin_inconsistent_pair_raises_after_the_device_run():
    """The drop-in's replication check (rss.py:222-228) runs on host threads
    while the device trains: a party whose hi disagrees with its neighbour's
    lo still gets ShareError, and the next call (same cached trainer) trains
    the reference tree."""
    from paper_2305_00645_b200 import TrainConfig, run_local, train_tree
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from paper_2305_00645_b200.shares import AVec, RING64, ShareError

    z, meta = golden_npz("trees_mpc.npz")
    k = next(i for i, m in enumerate(meta) if m["name"] == "spect_d4")
    data, seed = z[f"data{k}"], bytes.fromhex(meta[k]["seed"])
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    rng = np.random.default_rng(81)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    for bad in (True, False):
        def body(eng):
            p = eng.party
            hx = X[p % 3].copy()
            if bad and p == 2:
                hx[5, 1] ^= np.uint64(1)
            return train_tree(eng, AVec(RING64, X[p - 1], hx), AVec(RING64, Y[p - 1], Y[p % 3]),
                              TrainConfig(depth=meta[k]["depth"]))

        if bad:
            with pytest.raises(ShareError, match="replication"):
                run_local(body, seeds=setup, dealer_seed=derive_seed(seed, "deal"))
        else:
            run = run_local(body, seeds=setup, dealer_seed=derive_seed(seed, "deal"))
            assert np.array_equal(sum(r.T.lo for r in run.results), z[f"T{k}"])


def test_tee_heuristic_bit_identical_to_plaintext_trainer():
    # reference acceptance criterion 4 (test_acceptance.py:180-193): the trusted
    # path equals plaintext_train exactly; golden oT/oF are the reference's own
    # plaintext_train outputs
    from conftest import golden_npz
    from paper_2305_00645_b200.shares import AVec

    z, meta = golden_npz("trees_mpc.npz")
    rng = np.random.default_rng(40)
    for k, m in enumerate(meta):
        data, seed = z[f"data{k}"], bytes.fromhex(m["seed"])
        X, Y, T, F, d, setup, keys = _device_train(data, m["depth"], seed, rng, heuristic="tee")
        assert d == m["depth"]
        assert np.array_equal(opened(T), z[f"oT{k}"]) and np.array_equal(opened(F), z[f"oF{k}"]), m["name"]


def test_tee_transcripts_and_grow_match_reference():
    from conftest import golden_json
    from paper_2305_00645_b200 import TrainConfig, run_local, train_tree
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from paper_2305_00645_b200.shares import AVec, RING64, pairs_from_components

    g = golden_json("transcripts_tee.json")
    seed = b"\x45" * 16
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    rng = np.random.default_rng(41)
    for name, v in g.items():
        n, d, depth, policy = v["n"], v["d"], v["depth"], v["policy"]
        data = np.random.default_rng(n + d + depth).integers(0, 2, (n, d), dtype=np.uint8)
        xp = pairs_from_components(share(data[:, :-1], rng))
        yp = pairs_from_components(share(data[:, -1], rng))
        cfg = TrainConfig(depth=depth if policy == "fixed" else 1, heuristic="tee", policy=policy,
                          max_depth=depth if policy == "grow" else None)

        def body(eng):
            return train_tree(eng, AVec(RING64, *xp[eng.party - 1]), AVec(RING64, *yp[eng.party - 1]), cfg)

        run = run_local(body, seeds=setup, dealer_seed=derive_seed(seed, "deal"))
        assert run.results[0].depth == v["trained_depth"]
        T = sum(r.T.lo for r in run.results)
        F = sum(r.F.lo for r in run.results)
        assert T.tolist() == v["T"] and F.tolist() == v["F"], name
        assert run.transcript.records == [tuple(r) for r in v["records"]], name


def test_dot_product_count_reshare_same_tree_and_oracle_shares():
    rng = np.random.default_rng(42)
    cases = list(ref_cases())
    for m, data, Tref, Fref in cases[:12] + cases[-5:]:
        seed = bytes.fromhex(m["seed"])
        X, Y, T, F, d, setup, keys = _device_train(data, m["depth"], seed, rng, count_reshare="dot")
        assert np.array_equal(opened(T), Tref) and np.array_equal(opened(F), Fref), m["name"]
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        To, Fo, _ = oracle.train(X, Y, fill, m["depth"], keys, count_reshare=1)
        assert np.array_equal(T, To) and np.array_equal(F, Fo), m["name"]


def test_score_ring64_and_tau_variants_match_reference_and_oracle():
    from paper_2305_00645_b200.shares import Ring

    z, meta = golden_npz("trees_variants.npz")
    rng = np.random.default_rng(43)
    for k, m in enumerate(meta):
        data, seed = z[f"data{k}"], bytes.fromhex(m["seed"])
        X, Y, T, F, d, setup, keys = _device_train(data, m["depth"], seed, rng, tau=m["tau"],
                                                   score_ring=Ring(m["width"]))
        assert np.array_equal(opened(T), z[f"T{k}"]) and np.array_equal(opened(F), z[f"F{k}"]), m
        fill = filler_values(setup.filler_seed, (1 << m["depth"]) - 1, data.shape[1])
        To, Fo, _ = oracle.train(X, Y, fill, m["depth"], keys, tau=m["tau"], score_width=m["width"])
        assert np.array_equal(T, To) and np.array_equal(F, Fo), m


@pytest.mark.parametrize("nf,n,depth", [(13, 4000, 5), (20, 3001, 4), (33, 1500, 3), (64, 700, 2),
                                         (32, 60000, 8), (15, 3000, 4), (1, 5000, 3),
                                         (10, 2500, 6), (14, 4100, 7)])
def test_count_engines_share_exact_vs_oracle(nf, n, depth):
    """Tensor-core (tcgen05 kind::i8 limb) and CUDA-core count contractions
    give the oracle's shares, including several column blocks (nf > 15),
    partial sample blocks, (60000 x 32, depth 8) levels that take several
    lane chunks and K ranges, and the shallow levels' operand-swapped
    contraction at its column-block limits (16 columns: nf = 15; 4: nf = 1);
    the fused count's tensor-core mask sums over its whole range (nf = 10..14,
    the two constant columns beside the 2 nf + 1 feature/label columns)."""
    from paper_2305_00645_b200.seeds import derive_seed

    rng = np.random.default_rng(nf * 1000 + n)
    data = rng.integers(0, 2, size=(n, nf + 1), dtype=np.uint8)
    seed = (nf * 7 + n).to_bytes(16, "little")
    setup, k, keys = run_keys(seed)
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    To, Fo, _ = oracle.train(X, Y, fill, depth, keys)
    from paper_2305_00645_b200.train import TrainConfig, train_components

    for engine in ("tensor", "cuda"):
        T, F, d = train_components(X, Y, TrainConfig(depth=depth, count_engine=engine), setup, derive_seed(seed, "deal"))
        assert np.array_equal(T, To) and np.array_equal(F, Fo), engine


@pytest.mark.parametrize("engine,n,nf,depth", [("tensor", 3001, 12, 5), ("cuda", 3001, 12, 5),
                                                ("tensor", 300, 64, 3), ("tensor", 129, 5, 4)])
def test_host_operand_entry_equals_device_entry(engine, n, nf, depth):
    """gt_train_host (pinned host shares in, chunked 2-D uploads beside the
    prologue -- the last chunk small, down to one K block --, tree shares out)
    gives exactly the device entry's shares, also when captured in a CUDA
    graph and replayed; including the widest feature count."""
    from paper_2305_00645_b200._native import gt_keys
    from paper_2305_00645_b200.seeds import derive_seed
    from paper_2305_00645_b200.train import DeviceTrainer, TrainConfig, train_components

    rng = np.random.default_rng(77 + n + nf)
    data = rng.integers(0, 2, size=(n, nf + 1), dtype=np.uint8)
    seed = b"\x77" * 16
    setup, k, keys_t = run_keys(seed)
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    cfg = TrainConfig(depth=depth, count_engine=engine)
    T1, F1, _ = train_components(X, Y, cfg, setup, derive_seed(seed, "deal"))
    K = gt_keys()
    K.dealer.k0, K.dealer.k1 = keys_t[0]
    for i in range(3):
        K.pair[i].k0, K.pair[i].k1 = keys_t[i + 1]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).pin_memory()  # noqa: E731
    Xh, Yh, Fh = pin(X), pin(Y), pin(fill)
    Th = torch.empty((3, (1 << depth) - 1), dtype=torch.int64).pin_memory()
    Fo = torch.empty_like(Th).pin_memory()
    tr = DeviceTrainer(n, nf, cfg, host_io=True)
    tr.run_host(Xh, Yh, Fh, Th, Fo, K)
    torch.cuda.synchronize()
    assert np.array_equal(Th.numpy().view(np.uint64), T1) and np.array_equal(Fo.numpy().view(np.uint64), F1)
    Th.zero_()
    Fo.zero_()
    replay = tr.capture_host(Xh, Yh, Fh, Th, Fo, K)
    Th.zero_()
    Fo.zero_()
    replay()
    torch.cuda.synchronize()
    assert np.array_equal(Th.numpy().view(np.uint64), T1) and np.array_equal(Fo.numpy().view(np.uint64), F1)
