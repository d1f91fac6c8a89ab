"""Sample-sharded device training across ranks (B200).  The GPU box gives
one GPU, so two ranks share cuda:0 and reduce over gloo (NCCL refuses two
ranks on one device); this drives the real multi-rank device path --
DeviceTrainer with n_total/sample_base, the gt_train allreduce callback and
dist.allreduce_u64_ -- and requires the tree SHARES to equal the
single-device run bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, opened, run_keys, share

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, Y, fill, depth, keys_t, out_dir, side_stream=False):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2305_00645_b200 import TrainConfig
    from paper_2305_00645_b200._native import gt_keys
    from paper_2305_00645_b200.dist import shard_range, train_sharded
    from paper_2305_00645_b200.shares import from_device, to_device

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    k = gt_keys()
    k.dealer.k0, k.dealer.k1 = keys_t[0]
    for i in range(3):
        k.pair[i].k0, k.pair[i].k1 = keys_t[i + 1]
    n = X.shape[1]
    start, cnt = shard_range(n, world, rank)
    Xd = to_device(np.ascontiguousarray(X[:, start:start + cnt]))
    Yd = to_device(np.ascontiguousarray(Y[:, start:start + cnt]))
    Fd = to_device(fill)
    s = None
    if side_stream:  # a stream that is NOT torch's current one: the allreduce must follow it
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        torch.cuda.current_stream().synchronize()
    tr, d = train_sharded(Xd, Yd, Fd, TrainConfig(depth=depth), k, n_total=n, sample_base=start, stream=s)
    if s is not None:
        s.synchronize()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), T=from_device(tr.T), F=from_device(tr.F), d=d)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,world,side", [(5003, 2, False), (4999, 3, False), (5003, 2, True)])
def test_sharded_device_training_equals_single_device(tmp_path, n, world, side):
    """(4999, 3) gives odd shard bases (1667, 3333): the count lanes' zero
    words then straddle shard boundaries (count_lane_pair's unaligned path).
    side=True runs every rank on a non-current stream: the allreduce callback
    must enqueue on the stream gt_train hands it."""
    from paper_2305_00645_b200 import TrainConfig
    from paper_2305_00645_b200.seeds import derive_seed, filler_values
    from paper_2305_00645_b200.train import train_components

    rng = np.random.default_rng(31)
    data = rng.integers(0, 2, (n, 10), dtype=np.uint8)
    depth = 5
    seed = b"\x52" * 16
    setup, k, keys_t = run_keys(seed)
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, 10)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    T1, F1, _ = train_components(X, Y, TrainConfig(depth=depth), setup, derive_seed(seed, "deal"))
    mp.spawn(_worker, args=(world, _port(), X, Y, fill, depth, keys_t, str(tmp_path), side), nprocs=world,
             join=True)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert int(z["d"]) == depth
        assert np.array_equal(z["T"], T1) and np.array_equal(z["F"], F1)


def test_graph_captured_nccl_allreduce_equals_eager():
    """The sharded run's count allreduce captured in the CUDA graph with the
    level kernels (bench N > 1): a 1-rank NCCL group still issues real NCCL
    calls; the replayed C2 tree must equal the eager one."""
    import subprocess
    import sys

    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "capture_nccl_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "graph tree == eager tree: True" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
