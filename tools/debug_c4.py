"""Debug: C4-shaped training parity vs the shadow oracle (revealed tree) and
the C oracle (shares, smaller N)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from oracle import shadow
from paper_2305_00645_b200 import TrainConfig
from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys, keys_tuple
from paper_2305_00645_b200.train import train_components

def share(v, rng):
    v = np.asarray(v, dtype=np.uint64)
    s1 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2)
    s2 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    return np.stack([s1, s2, v - s1 - s2])

for n, nf, depth, engine, check_shares in [(60000, 32, 8, "tensor", True), (60000, 32, 8, "cuda", False),
                                           (300000, 32, 8, "tensor", False), (10 ** 6, 32, 8, "tensor", False)]:
    data = np.random.default_rng(n).integers(0, 2, (n, nf + 1), dtype=np.uint8)
    seed = (40_000).to_bytes(16, "little")
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    dseed = derive_seed(seed, "deal")
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    rng = np.random.default_rng(5)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    T, F, d = train_components(X, Y, TrainConfig(depth=depth, count_engine=engine), setup, dseed)
    wT, wF = shadow.mpc_train(data, depth, fill)
    rT, rF = T.sum(axis=0), F.sum(axis=0)
    bad = np.nonzero((rT != wT) | (rF != wF))[0]
    print(n, nf, depth, engine, "revealed ok" if len(bad) == 0 else f"MISMATCH slots {bad[:10]} ({len(bad)})", flush=True)
    if check_shares:
        To, Fo, _ = oracle.train(X, Y, fill, depth, keys_tuple(make_keys(setup, dseed)))
        print("  shares == oracle:", np.array_equal(T, To) and np.array_equal(F, Fo),
              "oracle revealed == shadow:", np.array_equal(To.sum(axis=0), wT), flush=True)
