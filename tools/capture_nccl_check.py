"""CUDA-graph capture of a sharded training run with its NCCL count allreduce
(run under torchrun; a 1-rank NCCL group still issues real NCCL calls here):
the replayed tree must equal the eager one."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import bench
from paper_2305_00645_b200 import TrainConfig, _native
from paper_2305_00645_b200.train import DeviceTrainer
from paper_2305_00645_b200.shares import from_device

dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
setup, keys, fill = bench._keys_and_filler()
data, Xh, Yh = bench._c2_inputs()
t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
X, Y, F = t(Xh), t(Yh), t(fill)
tr = DeviceTrainer(bench.N_C2, bench.NF_C2, TrainConfig(depth=bench.DEPTH_C2), device=dev)

def _cb(buf, count, stream, user):
    try:
        dist.all_reduce(tr.workspace_view(buf, int(count)), op=dist.ReduceOp.SUM)  # real NCCL even at world 1
        return 0
    except Exception as e:  # noqa: BLE001
        print("cb error", e, flush=True)
        return 1
cb = _native.ALLREDUCE_FN(_cb)
tr.run(X, Y, F, keys, allreduce=cb); torch.cuda.synchronize()
T0, F0 = from_device(tr.T).copy(), from_device(tr.F).copy()
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
eager = timeit(lambda: tr.run(X, Y, F, keys, allreduce=cb))
try:
    replay = tr.capture(X, Y, F, keys, allreduce=cb)
    g = timeit(replay)
    replay(); torch.cuda.synchronize()
    same = np.array_equal(from_device(tr.T), T0) and np.array_equal(from_device(tr.F), F0)
    print(f"rank {rank}: eager {eager:.3f} ms, graph {g:.3f} ms, graph tree == eager tree: {same}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: eager {eager:.3f} ms, capture failed: {e}", flush=True)
dist.destroy_process_group()
