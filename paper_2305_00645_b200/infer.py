"""Secure batch inference on B200 (reference pkg/src/obtree/infer.py).

The whole always-descend walk (``infer_batch``, infer.py:20-35) is one fused
sm_100a kernel (``gt_infer``): the encoded tree stays in shared memory, each
query's level payload and feature bit are fetched with oblivious full-scan
lookups, and no collective is needed -- instances are independent, so a
multi-GPU run shards them by global index (``instance_base``).
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _native
from .shares import RING64, components_from_pairs, from_device, pairs_from_components, ptr, to_device


def inference_needs(n_queries: int, depth: int, n_columns: int) -> dict:
    """Lane counts of the walk per gadget (infer.py:38-43): eq / select
    lanes of the oblivious lookups, for reporting."""
    lanes = n_queries * (((1 << depth) - 1) + depth * (n_columns - 1))
    return {("edabit", 64): lanes, ("dabit", 64): lanes}


def infer_device(tree, depth: int, queries, keys, *, instance_base: int = 0, out=None, slot_out=None, stream=None):
    """tree [3, 2^H - 1], queries [3, n, nf] device int64 tensors -> out
    [3, n] label shares (and final slot shares in slot_out if given)."""
    torch = _native.require_cuda()
    lib = _native.load()
    n, nf = int(queries.shape[1]), int(queries.shape[2])
    if tuple(tree.shape) != (3, (1 << depth) - 1):
        raise ValueError("tree must be [3, 2^depth - 1] heap-ordered payload shares")
    if out is None:
        out = torch.empty((3, n), dtype=torch.int64, device=queries.device)
    s = stream if stream is not None else torch.cuda.current_stream(queries.device)
    rc = lib.gt_infer(depth, ptr(tree), ptr(queries), n, nf, int(instance_base), ptr(out), ptr(slot_out),
                      ctypes.byref(keys), ctypes.c_void_p(s.cuda_stream))
    _native.check(rc)
    return out


def infer_components(tree: np.ndarray, depth: int, queries: np.ndarray, keys, *, instance_base: int = 0,
                     device=None) -> Tuple[np.ndarray, np.ndarray]:
    """Host component arrays in, host component arrays out (predictions, final slots)."""
    torch = _native.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    q = np.asarray(queries, dtype=np.uint64)
    if q.ndim != 3 or q.shape[0] != 3:
        raise ValueError("queries must be [3, n, nf] component shares")
    tq = to_device(q, dev)
    slot = torch.empty((3, q.shape[1]), dtype=torch.int64, device=dev)
    out = infer_device(to_device(tree, dev), depth, tq, keys, instance_base=instance_base, slot_out=slot)
    return from_device(out), from_device(slot)


def infer_3pc(level_pairs: Sequence, query_pairs: Sequence, keys, *, check: bool = True, device=None):
    """level_pairs: per party, the concatenated heap payload (lo, hi) of all
    levels; query_pairs: per party (lo, hi) shaped (n, nf).  Returns the
    per-party (lo, hi) label shares."""
    tree = components_from_pairs(level_pairs, RING64, check)
    q = components_from_pairs(query_pairs, RING64, check)
    slots = tree.shape[1]
    depth = int(slots + 1).bit_length() - 1
    if (1 << depth) - 1 != slots:
        raise ValueError("tree payload must hold 2^depth - 1 slots")
    out, _ = infer_components(tree, depth, q, keys, device=device)
    return pairs_from_components(out)
