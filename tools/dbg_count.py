import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import *  # noqa
import test_gpu as tg
from paper_2305_00645_b200.seeds import derive_seed
from paper_2305_00645_b200.train import TrainConfig, train_components
cases = [tuple(int(v) for v in c.split(',')) for c in sys.argv[1:]]
for nf, n, depth in cases:
    rng = np.random.default_rng(nf * 1000 + n)
    data = rng.integers(0, 2, size=(n, nf + 1), dtype=np.uint8)
    seed = (nf * 7 + n).to_bytes(16, "little")
    setup, k, keys = tg.run_keys(seed)
    fill = tg.filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    X, Y = tg.share(data[:, :-1], rng), tg.share(data[:, -1], rng)
    To, Fo, _ = tg.oracle.train(X, Y, fill, depth, keys)
    res = []
    for engine in ("tensor",):
        T, F, d = train_components(X, Y, TrainConfig(depth=depth, count_engine=engine), setup, derive_seed(seed, "deal"))
        res.append(bool(np.array_equal(T, To) and np.array_equal(F, Fo)))
    print(nf, n, depth, res, flush=True)
