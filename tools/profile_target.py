"""Short driver for ncu captures: `train` runs the C2 tree N times, `infer`
runs C3 (10^4 x 7 levels) N times, `infer5` a C5 slice (10^6 x 10 levels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2305_00645_b200 import TrainConfig
from paper_2305_00645_b200.train import DeviceTrainer
from paper_2305_00645_b200.infer import infer_device

what = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
setup, keys, fill = bench._keys_and_filler()
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
if what == "train":
    data, X, Y = bench._c2_inputs()
    tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2))
    X, Y, F = t(X), t(Y), t(fill)
    for _ in range(reps):
        tr.run(X, Y, F, keys)
else:
    rng = np.random.default_rng(1)
    depth, nf, n = (7, 13, 10_000) if what == "infer" else (10, 32, 1_000_000)
    T = t(bench._share(rng.integers(0, nf, (1 << depth) - 1), rng))
    Q = t(bench._share(rng.integers(0, 2, (n, nf)), rng))
    for _ in range(reps):
        infer_device(T, depth, Q, keys)
torch.cuda.synchronize()
print("done", what)
