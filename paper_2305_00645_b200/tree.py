"""Tree data model and host-side plaintext evaluator (reference tree.py).

Used by the CLI around the B200 path: CSV datasets (tree.py:52-96), the
complete-tree state and its validator (tree.py:104-157), and the exact
plaintext trainer / always-descend walk that ``compare`` checks the secure
tree against (tree.py:272-336).  The trainer shares its split rule with the
trusted helper (enclave.split_decisions), exactly as the reference's
plaintext trainer and EnclaveService share tree.split_decisions.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .enclave import F_DUMMY, F_INTERNAL, F_LEAF, majority_labels, split_decisions
from .seeds import derive_seed, filler_values


class DataError(ValueError):
    """tree.py:32-33."""


class TreeError(ValueError):
    """tree.py:36-37."""


def load_csv(path, min_columns: int = 2) -> np.ndarray:
    """Binary matrix, one sample per line, label last (tree.py:52-79)."""
    rows: List[List[int]] = []
    width: Optional[int] = None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            cells = [c.strip() for c in line.split(",")]
            if width is None:
                width = len(cells)
                if width < min_columns:
                    raise DataError(f"line {lineno}: need at least one feature and the label")
            elif len(cells) != width:
                raise DataError(f"line {lineno}: expected {width} columns, found {len(cells)}")
            row = []
            for col, cell in enumerate(cells):
                if cell not in ("0", "1"):
                    raise DataError(f"line {lineno}, column {col + 1}: {cell!r} is not a binary value")
                row.append(int(cell))
            rows.append(row)
    if not rows:
        raise DataError("dataset is empty")
    return np.array(rows, dtype=np.uint8)


def save_csv(path, data: np.ndarray) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for row in np.asarray(data, dtype=np.uint8):
            fh.write(",".join(str(int(v)) for v in row) + "\n")


def check_dataset(data: np.ndarray) -> np.ndarray:
    data = np.asarray(data)
    if data.ndim != 2 or data.shape[1] < 2:
        raise DataError("dataset must be samples x (features + label) with at least one feature")
    bad = np.argwhere(data > 1)
    if bad.size:
        r, c = bad[0]
        raise DataError(f"row {int(r) + 1}, column {int(c) + 1}: value is not binary")
    return data.astype(np.uint8)


@dataclass
class TreeState:
    """Complete-tree payloads: depth levels, 2^depth - 1 slots (tree.py:104-157)."""

    depth: int
    T: np.ndarray
    F: np.ndarray

    def __post_init__(self) -> None:
        self.T = np.asarray(self.T, dtype=np.uint64)
        self.F = np.asarray(self.F, dtype=np.uint64)

    @property
    def slots(self) -> int:
        return (1 << self.depth) - 1

    def validate(self, n_columns: Optional[int] = None, filler: Optional[np.ndarray] = None) -> None:
        if self.depth < 1:
            raise TreeError("depth must be at least 1")
        if self.T.shape != (self.slots,) or self.F.shape != (self.slots,):
            raise TreeError(f"payload arrays must have {self.slots} slots")
        if not np.isin(self.F, (F_INTERNAL, F_LEAF, F_DUMMY)).all():
            raise TreeError("node types must be 0, 1, or 2")
        last = (1 << (self.depth - 1)) - 1
        for i in range(self.slots):
            if i >= last:
                if self.F[i] == F_INTERNAL:
                    raise TreeError(f"slot {i}: internal node at the last level")
                if self.T[i] > 1:
                    raise TreeError(f"slot {i}: label {int(self.T[i])} is not binary")
            else:
                left, right = 2 * i + 1, 2 * i + 2
                if self.F[i] == F_INTERNAL:
                    if n_columns is not None and self.T[i] > n_columns - 2:
                        raise TreeError(f"slot {i}: split feature {int(self.T[i])} out of range")
                else:
                    if self.F[left] != F_DUMMY or self.F[right] != F_DUMMY:
                        raise TreeError(f"slot {i}: non-internal node has non-dummy children")
                    if filler is not None and self.T[i] != filler[i]:
                        raise TreeError(f"slot {i}: placeholder payload does not match the public stream")
        if self.F[0] == F_DUMMY:
            raise TreeError("root cannot be a dummy")

    def to_json(self) -> str:
        return json.dumps({"depth": self.depth, "T": [int(v) for v in self.T], "F": [int(v) for v in self.F]})

    @classmethod
    def from_json(cls, text: str) -> "TreeState":
        doc = json.loads(text)
        return cls(depth=int(doc["depth"]), T=np.array(doc["T"], dtype=np.uint64),
                   F=np.array(doc["F"], dtype=np.uint64))


def _level_counters(X: np.ndarray, y: np.ndarray, node: np.ndarray, n_nodes: int) -> np.ndarray:
    """(n_nodes, 3, 2nf) node counters for a whole level (tree.py:177-197)."""
    nf = X.shape[1]
    out = np.zeros((n_nodes, 3, 2 * nf), dtype=np.int64)
    keep = node >= 0
    nd, yy = node[keep], y[keep].astype(np.int64)
    for f in range(nf):
        x = X[keep, f].astype(np.int64)
        cnt = np.bincount(nd * 4 + x * 2 + yy, minlength=4 * n_nodes).reshape(n_nodes, 2, 2)
        out[:, 0, 2 * f:2 * f + 2] = cnt.sum(axis=2)
        out[:, 1, 2 * f:2 * f + 2] = cnt[:, :, 0]
        out[:, 2, 2 * f:2 * f + 2] = cnt[:, :, 1]
    return out


def plaintext_train(data: np.ndarray, depth: int, seed: bytes) -> TreeState:
    """Exact plaintext trainer (tree.py:272-326), level-vectorised."""
    data = check_dataset(data)
    if depth < 1:
        raise TreeError("depth must be at least 1")
    X, y = data[:, :-1], data[:, -1]
    n, nf = X.shape
    fill = filler_values(derive_seed(seed, "filler"), (1 << depth) - 1, data.shape[1])
    T = np.zeros((1 << depth) - 1, dtype=np.uint64)
    F = np.zeros_like(T)
    node = np.zeros(n, dtype=np.int64)
    types = np.array([F_LEAF], dtype=np.uint64)
    gam = np.ones((1, nf), dtype=bool)
    eff_prev = None
    for level in range(depth):
        nn, off = 1 << level, (1 << level) - 1
        C = _level_counters(X, y, node, nn)
        eff = C.copy()
        if level:
            empty = (C[:, 0, 0] + C[:, 0, 1]) == 0
            eff[empty] = eff_prev[np.arange(nn)[empty] // 2]
        if level == depth - 1:
            T[off:off + nn] = majority_labels(eff)
            F[off:off + nn] = types
            break
        sd, new_f, is_int, new_g = split_decisions(C, gam, types)
        T[off:off + nn] = np.where(is_int, sd, fill[off:off + nn])
        F[off:off + nn] = new_f
        sf = np.where(node >= 0, np.where(is_int, sd.astype(np.int64), -1)[np.maximum(node, 0)], -1)
        go = np.where(sf >= 0, X[np.arange(n), np.maximum(sf, 0)], 0)
        node = np.where(sf >= 0, 2 * node + go, -1)
        types = np.repeat(np.where(is_int, F_LEAF, F_DUMMY), 2).astype(np.uint64)
        gam = np.repeat(new_g, 2, axis=0)
        eff_prev = eff
    return TreeState(depth=depth, T=T, F=F)


def plaintext_infer(tree: TreeState, queries: np.ndarray) -> np.ndarray:
    """Always-descend walk for a batch (tree.py:329-336)."""
    q = np.atleast_2d(np.asarray(queries))
    node = np.zeros(q.shape[0], dtype=np.int64)
    for _ in range(tree.depth - 1):
        feat = tree.T[node].astype(np.int64)
        node = 2 * node + 1 + q[np.arange(q.shape[0]), feat].astype(np.int64)
    return tree.T[node]
