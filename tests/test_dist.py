"""Multi-process (gloo, world_size 2, CPU) coverage of the sharded paths:
sample-sharded training with a per-level count allreduce must give the SAME
share components as the unsharded run (randomness keyed by global index,
share addition linear), and instance sharding must tile the batch."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, opened, run_keys, share
from paper_2305_00645_b200.dist import allreduce_u64_, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, data, depth, keys, fill, X, Y, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = X.shape[1]
    start, cnt = shard_range(n, world, rank)

    def ar(buf):
        t = torch.from_numpy(buf.view(np.int64))
        allreduce_u64_(t)

    T, F, d = oracle.train(X[:, start:start + cnt], Y[:, start:start + cnt], fill, depth, keys, n_total=n,
                           sample_base=start, allreduce=ar)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), T=T, F=F)
    # exact u64 wraparound through the limb-split allreduce
    t = torch.tensor([-1, 2 ** 62, -(2 ** 63)], dtype=torch.int64)
    allreduce_u64_(t)
    np.save(os.path.join(out_dir, f"w{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_tiles():
    for n in (0, 1, 7, 48842, 10 ** 6):
        for w in (1, 2, 4, 8):
            parts = [shard_range(n, w, r) for r in range(w)]
            assert sum(c for _, c in parts) == n
            assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(w - 1))


def test_sharded_training_equals_single_device_shares(tmp_path):
    import oracle
    from paper_2305_00645_b200.seeds import filler_values

    rng = np.random.default_rng(12)
    data = rng.integers(0, 2, (301, 6), dtype=np.uint8)
    depth = 4
    setup, _, keys = run_keys(b"\x21" * 16)
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, 6)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    T1, F1, _ = oracle.train(X, Y, fill, depth, keys)
    port = _free_port()
    mp.spawn(_worker, args=(2, port, data, depth, keys, fill, X, Y, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["T"], T1) and np.array_equal(z["F"], F1)
        w = np.load(tmp_path / f"w{r}.npy").view(np.uint64)
        want = (np.array([-1, 2 ** 62, -(2 ** 63)], dtype=np.int64).view(np.uint64) * np.uint64(2))
        assert np.array_equal(w, want)
