"""ORACLE (test infrastructure only): plain-integer shadow of the reference's
revealed arithmetic.

The reference MPC trainer's revealed tree is an exact function of the
plaintext data: every gadget is exact (gadgets.py:3-10), so the opened tree
equals ``plaintext_train`` (tree.py:272-326) with the rational impurity
replaced by the fixed-point pipeline the MPC path evaluates on shares
(train.py:232-274, gadgets.py:297-401).  This module restates that pipeline
on plain integers so revealed trees can be checked at
10^6 samples in seconds; it is pinned to reference runs by the golden
fixtures (tests/golden/trees_mpc.npz, c2c3.npz).
"""

from __future__ import annotations

import math

import numpy as np

F_INTERNAL, F_LEAF, F_DUMMY = 0, 1, 2  # tree.py:40-42
M32 = np.uint64(0xFFFFFFFF)


def counter_shift(n_samples: int, score_width: int = 32, tau: int = 10) -> int:
    """train.py:75-78."""
    return max(0, int(n_samples).bit_length() - (score_width - tau - 2) // 2)


def _div_params(width: int, tau: int):
    bound = width - tau - 2
    ti = tau + 4
    sigma = max(0, bound + ti + 5 - width)
    kf = bound + ti - sigma - tau
    iters = math.ceil(math.log2(tau)) + 2 if tau > 1 else 2
    return bound, ti, sigma, kf, iters, round(2.9142 * (1 << ti))


def fx_div(p: np.ndarray, q: np.ndarray, tau: int = 10) -> np.ndarray:
    """division() on revealed values, all unsigned mod 2^32 with floor shifts
    (gadgets.py:310-349).  p, q uint64 arrays holding 32-bit values."""
    bound, ti, sigma, kf, iters, w0 = _div_params(32, tau)
    p = p.astype(np.uint64) & M32
    q = q.astype(np.uint64) & M32
    tsum = np.zeros_like(q)
    for j in range(1, bound):
        tsum += (q >= np.uint64(1 << j)).astype(np.uint64) << np.uint64(bound - 1 - j)
    v = (np.uint64(1 << (bound - 1)) - tsum) & M32
    qnorm = ((q * v) & M32) >> np.uint64(bound - ti)
    w = (np.uint64(w0) - np.uint64(2) * qnorm) & M32
    for _ in range(iters):
        e = (np.uint64(1 << (ti + 1)) - (((qnorm * w) & M32) >> np.uint64(ti))) & M32
        w = ((w * e) & M32) >> np.uint64(ti)
    pn = ((p * v) & M32) >> np.uint64(sigma)
    return ((((pn * w) & M32) + np.uint64(1 << (kf - 1))) & M32) >> np.uint64(kf)


def fx_scores(C: np.ndarray, shift: int, tau: int = 10) -> np.ndarray:
    """Per-feature fixed-point scores of one node (train.py:252-269).
    C: (3, 2nf) exact counters (python ints or uint64)."""
    c = (np.asarray(C, dtype=np.uint64) >> np.uint64(shift)) & M32
    nf = c.shape[1] // 2
    a = c[0]
    tot = (a[0::2] + a[1::2]) & M32
    tot_rep = np.repeat(tot, 2)
    P = (a * a - c[1] * c[1] - c[2] * c[2]) & M32
    Q = (a * tot_rep) & M32
    Q = Q + (Q == 0).astype(np.uint64)
    terms = fx_div(P, Q, tau)
    return ((terms[0::2] + terms[1::2]) & M32).reshape(nf)


def node_counters(features: np.ndarray, labels: np.ndarray, node: np.ndarray, n_nodes: int) -> np.ndarray:
    """(n_nodes, 3, 2nf) counters for all nodes of a level at once
    (vectorised tree.node_counters, tree.py:177-197); node = -1 for samples
    outside every candidate."""
    nf = features.shape[1]
    out = np.zeros((n_nodes, 3, 2 * nf), dtype=np.int64)
    keep = node >= 0
    nd = node[keep].astype(np.int64)
    y = labels[keep].astype(np.int64)
    for f in range(nf):
        x = features[keep, f].astype(np.int64)
        cnt = np.bincount(nd * 4 + x * 2 + y, minlength=4 * n_nodes).reshape(n_nodes, 2, 2)  # [n, x, y]
        out[:, 0, 2 * f:2 * f + 2] = cnt.sum(axis=2)
        out[:, 1, 2 * f:2 * f + 2] = cnt[:, :, 0]
        out[:, 2, 2 * f:2 * f + 2] = cnt[:, :, 1]
    return out


def mpc_train(data: np.ndarray, depth: int, filler: np.ndarray, tau: int = 10, n_total: int | None = None):
    """Revealed (T, F) of the reference MPC trainer (fixed policy)."""
    data = np.asarray(data, dtype=np.uint8)
    X, y = data[:, :-1], data[:, -1]
    n, nf = X.shape
    shift = counter_shift(n if n_total is None else n_total, 32, tau)
    worst = 1 << (tau + 1)
    total = (1 << depth) - 1
    T = np.zeros(total, dtype=np.uint64)
    F = np.zeros(total, dtype=np.uint64)
    node = np.zeros(n, dtype=np.int64)  # current node index within level, -1 = dropped out
    types = np.array([F_LEAF], dtype=np.int64)
    gammas = np.ones((1, nf), dtype=bool)
    eff_prev = None
    for level in range(depth):
        nn = 1 << level
        off = nn - 1
        C = node_counters(X, y, node, nn)
        tot = C[:, 0, 0] + C[:, 0, 1]
        eff = C.copy()
        if level > 0:
            empty = tot == 0
            eff[empty] = eff_prev[np.arange(nn)[empty] // 2]
        if level == depth - 1:
            psi0 = eff[:, 1, 0] + eff[:, 1, 1]
            psi1 = eff[:, 2, 0] + eff[:, 2, 1]
            T[off:off + nn] = (psi1 > psi0).astype(np.uint64)
            F[off:off + nn] = types.astype(np.uint64)
            break
        new_types = np.full(2 * nn, F_DUMMY, dtype=np.int64)
        new_g = np.zeros((2 * nn, nf), dtype=bool)
        split_feat = np.full(nn, -1, dtype=np.int64)
        for k in range(nn):
            c = C[k]
            psi0 = int(c[1, 0]) + int(c[1, 1])
            psi1 = int(c[2, 0]) + int(c[2, 1])
            sc = fx_scores(c, shift, tau).astype(np.int64)
            sc = np.where(gammas[k], sc, worst)
            sd = int(np.argmin(sc))  # leftmost minimum (gadgets.py:366-401)
            split = types[k] == F_LEAF and psi0 != 0 and psi1 != 0 and gammas[k].any()
            g = gammas[k].copy()
            g[sd] = False  # cleared for every node (train.py:272-273)
            new_g[2 * k] = new_g[2 * k + 1] = g
            if split:
                T[off + k] = sd
                F[off + k] = F_INTERNAL
                new_types[2 * k] = new_types[2 * k + 1] = F_LEAF
                split_feat[k] = sd
            else:
                T[off + k] = filler[off + k]
                F[off + k] = types[k]
        # descend: members of split nodes go left/right, the rest drop out
        valid = node >= 0
        sf = np.where(valid, split_feat[np.maximum(node, 0)], -1)
        go = np.where(sf >= 0, X[np.arange(n), np.maximum(sf, 0)], 0).astype(np.int64)
        node = np.where(sf >= 0, 2 * node + go, -1)
        # dummies inherit c_eff: their counters come from eff_prev via replace
        eff_prev = eff
        types = new_types
        gammas = new_g
    return T, F


def plaintext_infer(T: np.ndarray, depth: int, queries: np.ndarray) -> np.ndarray:
    """Vectorised always-descend walk (tree.py:329-336)."""
    q = np.asarray(queries)
    node = np.zeros(q.shape[0], dtype=np.int64)
    T = np.asarray(T, dtype=np.uint64)
    for _ in range(depth - 1):
        feat = T[node].astype(np.int64)
        node = 2 * node + 1 + q[np.arange(q.shape[0]), feat].astype(np.int64)
    return T[node]


def random_tree(rng: np.random.Generator, depth: int, n_columns: int):
    """tree.py:339-360 restated (structurally valid random tree)."""
    nf = n_columns - 1
    total = (1 << depth) - 1
    T = np.zeros(total, dtype=np.uint64)
    F = np.full(total, F_DUMMY, dtype=np.uint64)
    F[0] = F_INTERNAL if (depth > 1 and rng.integers(0, 4) > 0) else F_LEAF
    last = (1 << (depth - 1)) - 1
    for i in range(total):
        if i >= last:
            if F[i] == F_INTERNAL:
                F[i] = F_LEAF
            T[i] = rng.integers(0, 2)
            continue
        T[i] = rng.integers(0, nf)
        if F[i] == F_INTERNAL:
            for child in (2 * i + 1, 2 * i + 2):
                F[child] = F_INTERNAL if rng.integers(0, 3) > 0 else F_LEAF
    return T, F
