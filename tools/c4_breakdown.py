"""Per-kernel-class device time of one C4-shaped tree (10^6 x 32, depth 8)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_00645_b200 import TrainConfig, _native
from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys
from paper_2305_00645_b200.train import DeviceTrainer
n, nf, depth = 10 ** 6, 32, 8
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
X = torch.randint(-2**62, 2**62, (3, n, nf), generator=g, device=dev, dtype=torch.int64)
Y = torch.randint(-2**62, 2**62, (3, n), generator=g, device=dev, dtype=torch.int64)
seed = (40_000).to_bytes(16, "little")
setup = SeedSetup.from_master(derive_seed(seed, "run")); keys = make_keys(setup, derive_seed(seed, "deal"))
FL = torch.from_numpy(filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1).view(np.int64)).to(dev)
tr = DeviceTrainer(n, nf, TrainConfig(depth=depth))
tr.run(X, Y, FL, keys)
for _ in range(2):
    p = _native.gt_train_profile(); tr.run(X, Y, FL, keys, profile=p); torch.cuda.synchronize()
print({k: round(getattr(p, "ms_" + k), 3) for k in ("prods", "partition", "count_lanes", "count_contract", "node_hc", "node_finish", "total")})
