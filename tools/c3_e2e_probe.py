import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2305_00645_b200.infer import infer_device
setup, keys, fill = bench._keys_and_filler()
dev = torch.device("cuda", 0)
z = np.load(os.path.join(bench.ROOT, "tests", "golden", "c2c3.npz")) if False else None
data, Xh, Yh = bench._c2_inputs()
rng = np.random.default_rng(1)
Tv = rng.integers(0, 13, 127)
T = torch.from_numpy(bench._share(Tv, rng).view(np.int64)).to(dev)
q = np.random.default_rng(7).integers(0, 2, (10000, 13), dtype=np.uint8)
Qp = torch.from_numpy(np.ascontiguousarray(bench._share(q, rng)).view(np.int64)).pin_memory()
Q = Qp.to(dev); out = torch.empty((3, 10000), dtype=torch.int64, device=dev)
Oh = torch.empty((3, 10000), dtype=torch.int64).pin_memory()
def step():
    Q.copy_(Qp, non_blocking=True); infer_device(T, 7, Q, keys, out=out); Oh.copy_(out, non_blocking=True)
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s): step()
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s): step()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for mode in ("graph", "graph-noflush", "h2d-only"):
    ts = []
    for i in range(12):
        if mode != "graph-noflush": flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        if mode == "h2d-only": Q.copy_(Qp, non_blocking=True)
        else: g.replay()
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    print(mode, " ".join(f"{t:.0f}" for t in ts))
