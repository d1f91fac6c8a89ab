"""Multi-GPU plumbing: sample-sharded training, instance-sharded inference.

Training: samples are split contiguously over the ranks of
one box; features, labels and node indices never leave their GPU.  Every
level produces count partials ``S[3][n_h][W+1]`` on each rank, and because
share addition is linear the ranks simply sum them (one allreduce of a few
hundred KB per level over NVLink) before the per-node heuristic, which every
rank then runs redundantly with identical counter-keyed randomness -- so all
ranks hold bit-identical tree shares and no broadcast is needed.  Randomness
is keyed by GLOBAL sample index, so the shares equal the single-GPU run's.

Inference: queries are independent; each rank walks its contiguous slice
(keyed by global instance index) with no collective at all.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Tuple

from . import _native


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous split of n items: (start, count) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n), world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def allreduce_u64_(t, group=None) -> None:
    """In-place SUM mod 2^64 of an int64 tensor holding uint64 bits.

    NCCL adds int64 with two's-complement wraparound, which is exactly Z_2^64
    addition.  Other backends (gloo on CPU) get an overflow-free 16-bit limb
    split so the result is exact independent of the backend's integer
    semantics."""
    import torch
    import torch.distributed as dist

    if dist.get_world_size(group) == 1:
        return
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return
    u = t.view(torch.int64)
    limbs = torch.stack([(u >> (16 * k)) & 0xFFFF for k in range(4)]).cpu()  # gloo: host tensors
    dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)
    acc = torch.zeros_like(limbs[0])
    for k in range(4):
        acc = acc + (limbs[k] << (16 * k))  # wraps mod 2^64
    u.copy_(acc.to(u.device))


def make_allreduce(trainer, group=None):
    """gt_allreduce_fn for DeviceTrainer.run: sums the level's count partials
    (a slice of the trainer's workspace) across `group`."""

    def _cb(buf, count, stream, user):
        try:
            import torch

            # enqueue on the stream gt_train passes (its count kernels' stream), not
            # torch's current one: the collective must be ordered after the partials
            s = torch.cuda.ExternalStream(int(stream), device=trainer.device) if stream else \
                torch.cuda.current_stream(trainer.device)
            with torch.cuda.stream(s):
                allreduce_u64_(trainer.workspace_view(buf, int(count)), group)
            return 0
        except Exception:  # noqa: BLE001 - reported to the C side as failure
            return 1

    return _native.ALLREDUCE_FN(_cb)


def train_sharded(X_local, Y_local, filler, cfg, keys, *, n_total: int, sample_base: int, group=None,
                  trainer=None, stream=None):
    """Run one sample-sharded training step on this rank.  X_local
    [3, n_local, nf], Y_local [3, n_local] device tensors; `stream` (default:
    torch's current stream) orders the kernels and the allreduce.  Returns the
    trainer (T/F on trainer.T / trainer.F) and the trained depth."""
    from .train import DeviceTrainer

    if trainer is None:
        trainer = DeviceTrainer(int(X_local.shape[1]), int(X_local.shape[2]), cfg, n_total=n_total,
                                sample_base=sample_base, device=X_local.device)
    cb = make_allreduce(trainer, group)
    depth = trainer.run(X_local, Y_local, filler, keys, allreduce=cb, stream=stream)
    return trainer, depth
