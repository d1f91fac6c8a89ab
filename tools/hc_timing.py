"""Per-level heuristic phase timings (GT_HC_TIMING=1): post-finish kernel of
node 0: scores, argmin rounds, budget clear, split."""
import ctypes, os, sys
os.environ["GT_HC_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2305_00645_b200 import TrainConfig, _native
from paper_2305_00645_b200.train import DeviceTrainer
setup, keys, fill = bench._keys_and_filler()
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
data, X, Y = bench._c2_inputs()
tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2))
X, Y, F = t(X), t(Y), t(fill)
for _ in range(3):
    tr.run(X, Y, F, keys)
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_ulonglong * 128)()
_native.check(lib.gt_diag_hc_timestamps(buf, 128))
for lv in range(bench.DEPTH_C2 - 1):
    ts = [buf[8 * lv + k] for k in range(7)]
    d = lambda a, b: (ts[b] - ts[a]) / 1e3
    print(f"level {lv}: scores {d(0, 1):.2f} us, argmin {d(1, 2):.2f} us, budget {d(2, 3):.2f} us, "
          f"split: keys {d(3, 5):.2f} chains {d(5, 6):.2f} counters {d(6, 4):.2f} us")
print("timeline per level (us from the control CTA's start): ctrl tapes/end, feat start/tape/end, div start/end, post start/end")
for lv in range(bench.DEPTH_C2 - 1):
    q = [buf[64 + 8 * lv + k] for k in range(8)]
    t0 = q[0]
    r = lambda v: (v - t0) / 1e3
    print(f"level {lv}: ctrl {r(q[1]):.2f}/{r(q[2]):.2f}  feat {r(q[3]):.2f}/{r(q[4]):.2f}/{r(q[5]):.2f}  "
          f"div {r(q[6]):.2f}/ladder {r(buf[8 * lv + 7]):.2f}/{r(q[7]):.2f}  post {r(buf[8 * lv]):.2f}/{r(buf[8 * lv + 4]):.2f}")
