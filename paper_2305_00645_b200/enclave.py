"""Trusted split helper for heuristic "tee" (reference enclave.py:94-185,
_heuristic_tee / _labels_tee train.py:277-301).

The parties hand the helper their shares of a level's node state; it
reconstructs them, decides every node's split exactly, and hands back fresh
shares of the decisions.  On B200 the three parties' shares already sit in
one device buffer, so the "upload" is a device-to-host copy of the component
arrays at the helper's call from ``gt_train`` (``gt_heuristic_fn``) -- made
on the stream ``gt_train`` passes -- and the "download" a host-to-device copy
of freshly drawn components.

The split rule is the reference's (tree.py:200-264: additive Gini
sum_j (a_j^2 - m0_j^2 - m1_j^2) / (a_j * tot) over the non-empty branches,
an empty node or a spent feature scores 2, leftmost strict minimum; split
iff the node is a live leaf, impure and has features left; majority label
with ties to 0) evaluated as whole-level integer arrays: every score is a
fraction num/den with den > 0, and candidates are compared by exact
cross-multiplication on Python integers (object arrays), so there is no
rounding and no per-node loop.
"""

from __future__ import annotations

import hashlib
from typing import Tuple

import numpy as np

from . import _native

F_INTERNAL, F_LEAF, F_DUMMY = 0, 1, 2  # node types, tree.py:40-42


class EnclaveError(RuntimeError):
    """enclave.py:43-44."""


def score_fractions(C: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Exact per-(node, feature) impurity as (numerator, denominator) object
    arrays.  C: (n, 3, 2nf) exact counters, rows = all / label 0 / label 1,
    columns (2i + j) = feature i takes value j."""
    C = np.asarray(C).astype(object)
    a, m0, m1 = C[:, 0, 0::2], C[:, 1, 0::2], C[:, 2, 0::2]  # branch j = 0
    b, n0, n1 = C[:, 0, 1::2], C[:, 1, 1::2], C[:, 2, 1::2]  # branch j = 1
    tot = a + b
    pa = np.where(a > 0, a * a - m0 * m0 - m1 * m1, 0)
    pb = np.where(b > 0, b * b - n0 * n0 - n1 * n1, 0)
    da, db = np.where(a > 0, a, 1), np.where(b > 0, b, 1)
    num, den = pa * db + pb * da, da * db * tot
    empty = tot == 0
    return np.where(empty, 2, num), np.where(empty, 1, den)


def best_features(C: np.ndarray, gammas: np.ndarray) -> np.ndarray:
    """Leftmost strict argmin of the scores over the features still in each
    node's budget (spent features score 2, like an empty node)."""
    num, den = score_fractions(C)
    gam = np.asarray(gammas, dtype=bool)
    num, den = np.where(gam, num, 2), np.where(gam, den, 1)
    n, nf = num.shape
    best = np.zeros(n, dtype=np.int64)
    bn, bd = np.full(n, 2, dtype=object), np.ones(n, dtype=object)
    for i in range(nf):
        win = (num[:, i] * bd) < (bn * den[:, i])
        best = np.where(win, i, best)
        bn, bd = np.where(win, num[:, i], bn), np.where(win, den[:, i], bd)
    return best


def label_totals(C: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """(psi0, psi1): samples of label 0 / label 1 at each node (feature 0's
    two cells of rows 1 and 2 partition the node)."""
    C = np.asarray(C).astype(object)
    return C[:, 1, 0] + C[:, 1, 1], C[:, 2, 0] + C[:, 2, 1]


def split_decisions(C: np.ndarray, gammas: np.ndarray, types: np.ndarray):
    """Whole-level split decisions -> (sd, new_type, is_internal, new_gammas)."""
    gam = np.array(gammas, dtype=bool)
    kinds = np.asarray(types, dtype=np.uint64)
    psi0, psi1 = label_totals(C)
    sd = best_features(C, gam)
    grow = (kinds == F_LEAF) & (psi0 != 0) & (psi1 != 0) & gam.any(axis=1)
    rows = np.nonzero(grow)[0]
    gam[rows, sd[rows]] = False
    new_f = np.where(grow, np.uint64(F_INTERNAL), kinds).astype(np.uint64)
    return sd.astype(np.uint64), new_f, grow, gam


def majority_labels(C: np.ndarray) -> np.ndarray:
    """1 where label-1 samples strictly outnumber label-0 samples, else 0."""
    psi0, psi1 = label_totals(C)
    return (psi1 > psi0).astype(np.uint64)


class DeviceEnclave:
    """The helper as seen by ``gt_train``: reconstructs the uploaded
    component arrays, decides, reshares with its own seeded stream."""

    def __init__(self, seed: bytes, trainer):
        self.trainer = trainer
        digest = hashlib.sha256(seed + b"/b200-enclave").digest()
        self.rng = np.random.Generator(np.random.PCG64(int.from_bytes(digest[:16], "little")))
        self.calls = 0
        self.error = None
        self._fn = _native.HEURISTIC_FN(self._call)

    @property
    def fn(self):
        return self._fn

    def _random(self, shape, mask=None) -> np.ndarray:
        w = self.rng.integers(0, 1 << 63, shape, dtype=np.uint64) * np.uint64(2) + \
            self.rng.integers(0, 2, shape, dtype=np.uint64)
        return w if mask is None else w & np.uint64(mask)

    def _arith(self, values) -> np.ndarray:
        v = np.asarray(values, dtype=np.uint64)
        r1, r2 = self._random(v.shape), self._random(v.shape)
        return np.stack([r1, r2, v - r1 - r2])

    def _xor(self, words, mask: int) -> np.ndarray:
        w = np.asarray(words, dtype=np.uint64)
        r1, r2 = self._random(w.shape, mask), self._random(w.shape, mask)
        return np.stack([r1, r2, w ^ r1 ^ r2])

    def _fetch(self, addr: int, count: int, stream) -> np.ndarray:
        torch = _native.require_cuda()
        with torch.cuda.stream(stream):
            host = self.trainer.workspace_view(addr, count).to("cpu")  # synchronous on `stream`
        return host.numpy().view(np.uint64)

    def _store(self, addr: int, arr: np.ndarray, stream) -> None:
        torch = _native.require_cuda()
        src = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1)).view(np.int64))
        with torch.cuda.stream(stream):
            self.trainer.workspace_view(addr, src.numel()).copy_(src)
        stream.synchronize()

    # gt_heuristic_fn(op, level, n, nf, counters, gamma, types, out, stream, user)
    def _call(self, op, level, n, nf, counters, gamma, types, out, stream, user):
        try:
            torch = _native.require_cuda()
            s = torch.cuda.ExternalStream(int(stream or 0), device=self.trainer.device) if stream else \
                torch.cuda.current_stream(self.trainer.device)
            self.calls += 1
            cells = n * 3 * 2 * nf
            C = self._fetch(counters, 3 * cells, s).reshape(3, n, 3, 2 * nf).sum(axis=0, dtype=np.uint64)
            if op == 1:  # split decisions (enclave.py:161-180)
                gw = np.bitwise_xor.reduce(self._fetch(gamma, 3 * n, s).reshape(3, n), axis=0)
                kinds = self._fetch(types, 3 * n, s).reshape(3, n).sum(axis=0, dtype=np.uint64)
                bits = np.arange(nf, dtype=np.uint64)
                gammas = ((gw[:, None] >> bits[None, :]) & np.uint64(1)).astype(bool)
                sd, new_f, is_int, new_g = split_decisions(C, gammas, kinds)
                gword = np.bitwise_or.reduce(new_g.astype(np.uint64) << bits[None, :], axis=1) if nf else \
                    np.zeros(n, dtype=np.uint64)
                res = np.stack([self._xor(is_int.astype(np.uint64), 1), self._arith(sd), self._arith(new_f),
                                self._xor(gword, (1 << nf) - 1)])
            elif op == 2:  # leaf labels (enclave.py:182-186)
                res = self._arith(majority_labels(C))
            else:
                raise EnclaveError(f"unknown enclave op {op}")
            self._store(out, res, s)
            return 0
        except Exception as e:  # noqa: BLE001 - surfaced as a failed call
            self.error = e
            return 1
