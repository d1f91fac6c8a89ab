"""Dev timing probe: device time of C2 training / C3 + C5-slice inference."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_00645_b200 import TrainConfig
from paper_2305_00645_b200.train import DeviceTrainer
from paper_2305_00645_b200.infer import infer_device
from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys
from paper_2305_00645_b200.shares import to_device

def share(v, rng):
    v = np.asarray(v, dtype=np.uint64)
    s1 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2)
    s2 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    return np.stack([s1, s2, v - s1 - s2])

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts), sorted(ts)[len(ts)//2]

rng = np.random.default_rng(0)
data = np.random.default_rng(1011).integers(0, 2, size=(48842, 14), dtype=np.uint8)
seed = (11_000).to_bytes(16, "little")
setup = SeedSetup.from_master(derive_seed(seed, "run")); keys = make_keys(setup, derive_seed(seed, "deal"))
tr = DeviceTrainer(48842, 13, TrainConfig(depth=7))
X = to_device(share(data[:, :-1], rng)); Y = to_device(share(data[:, -1], rng))
fill = to_device(filler_values(setup.filler_seed, 127, 14))
print("C2 train ms (min, med):", timed(lambda: tr.run(X, Y, fill, keys)), flush=True)
from paper_2305_00645_b200 import _native as _nv
pr = _nv.gt_train_profile()
tr.run(X, Y, fill, keys, profile=pr); torch.cuda.synchronize()
print("C2 per-kernel ms:", {k: round(getattr(pr, "ms_" + k), 4) for k in ("prods", "partition", "count_lanes", "count_contract", "node_hc", "node_finish")}, flush=True)
tr_dot = DeviceTrainer(48842, 13, TrainConfig(depth=7, count_reshare="dot"))
print("C2 dot ms (min, med):", timed(lambda: tr_dot.run(X, Y, fill, keys)), flush=True)
if os.environ.get("QT_TRAIN_ONLY"):
    sys.exit(0)
for depth, nf, n in ((7, 13, 10_000), (10, 32, 1_000_000)):
    T = to_device(share(rng.integers(0, nf, (1 << depth) - 1), rng)); Q = to_device(share(rng.integers(0, 2, (n, nf)), rng))
    ms = timed(lambda: infer_device(T, depth, Q, keys))
    print(f"infer depth {depth} nf {nf} n {n} ms:", ms, "inst/s:", n / ms[0] * 1e3, flush=True)

# Philox block throughput (integer-ALU roof of the share kernels)
from paper_2305_00645_b200 import _native
lib = _native.load()
import ctypes
grid, iters = 148 * 8 * 4, 4096
out = torch.empty(grid * 256, dtype=torch.int64, device="cuda")
def run():
    _native.check(lib.gt_diag_philox(grid, iters, out.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
ms = timed(run)
print("philox blocks/s:", grid * 256 * iters / (ms[0] / 1e3), flush=True)
