"""Secure level-wise training on B200 (reference pkg/src/obtree/train.py).

``TrainConfig`` / ``TrainResult`` / ``counter_shift`` / ``resolved_depth`` /
``levels_of`` keep the reference's names and meaning (train.py:57-90).
The level loop itself (partition -> count -> heuristic -> replace -> split /
labels, train.py:108-197) runs natively: ``gt_train`` in the C ABI drives the
sm_100a kernels level by level on one CUDA stream, calling back only for the
per-level count allreduce of a sample-sharded run.
"""

from __future__ import annotations

import collections
import ctypes
import threading
from collections import OrderedDict
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .seeds import SeedSetup, filler_values, make_keys
from .shares import RING32, RING64, AVec, Ring, components_from_pairs, from_device, ptr, to_device


@dataclass
class TrainConfig:
    """train.py:57-65."""

    depth: int = 4
    tau: int = 10
    heuristic: str = "mpc"  # "mpc" | "tee"
    policy: str = "fixed"  # "fixed" | "grow" | "feature_cap"
    max_depth: Optional[int] = None
    score_ring: Ring = RING32
    count_ring: Ring = RING64
    # B200 extension: "elementwise" reshares every count product like the
    # reference (train.py:219); "dot" sums the local products over samples
    # first and reshares each counter cell once (ABY3-style dot product) --
    # same revealed tree, a fraction of the reshared words.
    count_reshare: str = "elementwise"
    # B200 extension: which unit runs the count contraction -- "tensor"
    # (tcgen05.mma kind::i8 over INT8 limbs of the Z_2^64 shares) or "cuda"
    # (64-bit IMAD on the CUDA cores).  Both produce identical shares.
    count_engine: str = "tensor"


@dataclass
class TrainResult:
    """train.py:68-72 (T, F per party as AVec in the drop-in path)."""

    T: object
    F: object
    depth: int


def as_config(cfg) -> TrainConfig:
    """Accept the reference's own TrainConfig (train.py:57-65) -- or any
    object with its fields -- where a TrainConfig is expected; the B200-only
    knobs take their defaults."""
    if isinstance(cfg, TrainConfig):
        return cfg
    out = TrainConfig()
    for name in ("depth", "tau", "heuristic", "policy", "max_depth", "count_reshare", "count_engine"):
        if hasattr(cfg, name):
            setattr(out, name, getattr(cfg, name))
    for name in ("score_ring", "count_ring"):
        if hasattr(cfg, name):
            setattr(out, name, Ring(int(getattr(cfg, name).width)))
    return out


def counter_shift(n_samples: int, cfg: TrainConfig) -> int:
    """Public scale-down so squared counters fit the division domain (train.py:75-78)."""
    headroom = (cfg.score_ring.width - cfg.tau - 2) // 2
    return max(0, int(n_samples).bit_length() - headroom)


def resolved_depth(cfg: TrainConfig, n_columns: int) -> int:
    """train.py:81-86."""
    if cfg.policy == "feature_cap":
        return n_columns
    if cfg.policy == "grow":
        return cfg.max_depth if cfg.max_depth is not None else n_columns
    return cfg.depth


def levels_of(vec, depth: int) -> List:
    """Heap-level slices of a payload vector (train.py:89-90)."""
    return [vec.take(slice((1 << t) - 1, (1 << (t + 1)) - 1)) for t in range(depth)]


def _validate(cfg: TrainConfig, nf: int) -> int:
    if cfg.heuristic not in ("mpc", "tee"):
        raise ValueError(f"unknown heuristic {cfg.heuristic!r}")
    if cfg.policy not in ("fixed", "grow", "feature_cap"):
        raise ValueError(f"unknown depth policy {cfg.policy!r}")
    if cfg.count_reshare not in ("elementwise", "dot"):
        raise ValueError(f"unknown count_reshare {cfg.count_reshare!r}")
    if cfg.count_engine not in ("tensor", "cuda"):
        raise ValueError(f"unknown count_engine {cfg.count_engine!r}")
    if cfg.count_ring.width != 64:
        raise ValueError("counters live in Z_2^64 on the B200 path")
    depth = resolved_depth(cfg, nf + 1)
    if depth < 1:
        raise ValueError("depth must be at least 1")
    if depth > 16:
        raise ValueError(f"depth {depth} exceeds the B200 trainer's 16 levels (heap slots and node "
                         "indices are sized for 2^16 - 1); pass an explicit depth / max_depth")
    if not 1 <= nf <= 64:
        raise ValueError(f"{nf} features: the B200 trainer supports 1..64 (a node's feature budget "
                         "gamma is one 64-bit word of bit shares)")
    if cfg.score_ring.width not in (32, 64):
        raise ValueError("score ring must be Z_2^32 or Z_2^64")
    if not 0 <= cfg.tau < cfg.score_ring.width - 2:
        raise ValueError(f"fixed-point precision tau={cfg.tau} must satisfy 0 <= tau < {cfg.score_ring.width - 2}")
    return depth


class DeviceTrainer:
    """One training shape (samples on this device, features, depth) with its
    device workspace; ``run`` can be called repeatedly (bench steps)."""

    def __init__(self, n_local: int, nf: int, cfg: TrainConfig, *, n_total: Optional[int] = None,
                 sample_base: int = 0, device=None, host_io: bool = False):
        torch = _native.require_cuda()
        self.lib = _native.load()
        self.depth = _validate(cfg, nf)
        self.cfg = cfg
        self.nf = nf
        self.n_local = int(n_local)
        self.n_total = int(n_total if n_total is not None else n_local)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        c = _native.gt_train_cfg()
        c.depth = self.depth
        c.tau = cfg.tau
        c.score_width = cfg.score_ring.width
        c.nf = nf
        c.policy = 1 if cfg.policy == "grow" else 0
        c.heuristic = 1 if cfg.heuristic == "tee" else 0
        c.count_reshare = 1 if cfg.count_reshare == "dot" else 0
        c.count_engine = 1 if cfg.count_engine == "cuda" else 0
        c.n_total = self.n_total
        c.n_local = self.n_local
        c.sample_base = int(sample_base)
        self.c = c
        self.host_io = bool(host_io)
        nbytes = (self.lib.gt_train_host_workspace_bytes if self.host_io else self.lib.gt_train_workspace_bytes)(
            ctypes.byref(c))
        if nbytes == 0:
            raise ValueError("unsupported training shape (depth 1..16, 1..64 features)")
        self.workspace = torch.empty(nbytes // 8, dtype=torch.int64, device=self.device)
        slots = (1 << self.depth) - 1
        self.T = torch.empty((3, slots), dtype=torch.int64, device=self.device)
        self.F = torch.empty((3, slots), dtype=torch.int64, device=self.device)

    def workspace_view(self, addr: int, count: int):
        """Tensor view of `count` words of the workspace at device address `addr`."""
        off = (addr - self.workspace.data_ptr()) // 8
        return self.workspace[off:off + count]

    def run(self, X, Y, filler, keys, *, allreduce=None, stream=None, profile=None, enclave_seed=None) -> int:
        """X [3, n_local, nf], Y [3, n_local], filler [2^H - 1] device int64
        tensors (uint64 bits).  Results land in self.T / self.F; returns the
        trained depth.  `profile` (a _native.gt_train_profile) receives the
        CUDA-event device time per kernel class.  Heuristic "tee" calls the
        trusted helper (enclave.DeviceEnclave, seeded by `enclave_seed`, the
        reference's SeedSetup.enclave_seed) once per level."""
        torch = _native.require_cuda()
        if tuple(X.shape) != (3, self.n_local, self.nf) or tuple(Y.shape) != (3, self.n_local):
            raise ValueError("features must be [3, n, nf] and labels [3, n] component shares")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        d = ctypes.c_int32(0)
        cb = _native.ALLREDUCE_FN(0) if allreduce is None else allreduce
        prof = ctypes.byref(profile) if profile is not None else None
        helper = None
        hfn = _native.HEURISTIC_FN(0)
        if self.cfg.heuristic == "tee":
            from .enclave import DeviceEnclave

            helper = DeviceEnclave(enclave_seed if enclave_seed is not None else b"\x00" * 16, self)
            hfn = helper.fn
        rc = self.lib.gt_train_ex(ctypes.byref(self.c), ptr(X), ptr(Y), ptr(filler), ptr(self.T), ptr(self.F),
                                  ctypes.byref(d), ptr(self.workspace), self.workspace.numel() * 8,
                                  ctypes.byref(keys), cb, None, hfn, None, ctypes.c_void_p(s.cuda_stream), prof)
        if rc and helper is not None and getattr(helper, "error", None) is not None:
            raise helper.error
        _native.check(rc)
        return int(d.value)


    def run_host(self, Xh, Yh, filler_h, T_h, F_h, keys, *, allreduce=None, stream=None) -> int:
        """Training from HOST operands (pinned int64 CPU tensors, same shapes as
        `run`; results into the pinned host tensors T_h / F_h [3, 2^H - 1]):
        gt_train_host uploads the sample shares in chunks beside the prologue
        and reads the tree back, all ordered on `stream`.  Needs a trainer built
        with host_io=True; synchronise the stream before reading T_h / F_h."""
        torch = _native.require_cuda()
        if not self.host_io:
            raise ValueError("construct the DeviceTrainer with host_io=True for run_host")
        if tuple(Xh.shape) != (3, self.n_local, self.nf) or tuple(Yh.shape) != (3, self.n_local):
            raise ValueError("features must be [3, n, nf] and labels [3, n] component shares")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        d = ctypes.c_int32(0)
        cb = _native.ALLREDUCE_FN(0) if allreduce is None else allreduce
        rc = self.lib.gt_train_host(ctypes.byref(self.c), Xh.data_ptr(), Yh.data_ptr(), filler_h.data_ptr(),
                                    T_h.data_ptr(), F_h.data_ptr(), ctypes.byref(d), ptr(self.workspace),
                                    self.workspace.numel() * 8, ctypes.byref(keys), cb, None,
                                    ctypes.c_void_p(s.cuda_stream))
        _native.check(rc)
        return int(d.value)

    def capture_host(self, Xh, Yh, filler_h, T_h, F_h, keys, allreduce=None):
        """CUDA graph of one whole host-operand run (uploads, kernels, the
        sharded run's count allreduce if capturable, readback).  Fixed policy,
        mpc heuristic only (as ``capture``)."""
        torch = _native.require_cuda()
        if self.cfg.policy == "grow" or self.cfg.heuristic == "tee":
            raise ValueError("grow / tee synchronise with the host per level; they cannot be captured")
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.run_host(Xh, Yh, filler_h, T_h, F_h, keys, stream=s, allreduce=allreduce)
        s.synchronize()
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.run_host(Xh, Yh, filler_h, T_h, F_h, keys, stream=s, allreduce=allreduce)
        self._graph_host_refs = (Xh, Yh, filler_h, T_h, F_h, keys, allreduce)
        return g.replay

    def host_graph(self, keys):
        """Replay of a captured whole host-operand run on this trainer's pinned
        staging buffers for these keys (the drop-in path: the graph is
        captured on a key set's first use, then replayed), or None where the
        run cannot be captured (grow, tee).  A few key sets are kept."""
        if self.cfg.policy == "grow" or self.cfg.heuristic == "tee" or not getattr(self, "staging", None):
            return None
        graphs = self.__dict__.setdefault("_host_graphs", collections.OrderedDict())
        kb = bytes(keys)
        g = graphs.pop(kb, None)
        if g is None:
            st = self.staging
            while len(graphs) >= 4:
                graphs.popitem(last=False)
            g = self.capture_host(st["X"], st["Y"], st["fill"], st["T"], st["F"], keys)
        graphs[kb] = g
        return g

    def capture(self, X, Y, filler, keys, allreduce=None):
        """Capture one whole training run (every level's kernels, and the
        per-level count allreduce of a sharded run when `allreduce` enqueues
        a graph-capturable collective such as NCCL's) into a CUDA graph;
        returns a callable that replays it on the current stream.  Fixed
        policy only (grow opens a stop bit on the host mid-run)."""
        torch = _native.require_cuda()
        if self.cfg.policy == "grow" or self.cfg.heuristic == "tee":
            raise ValueError("grow / tee synchronise with the host per level; they cannot be captured")
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.run(X, Y, filler, keys, stream=s, allreduce=allreduce)  # warm: kernel attributes outside capture
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.run(X, Y, filler, keys, stream=s, allreduce=allreduce)
        self._graph_refs = (X, Y, filler, keys, allreduce)  # keep the captured buffers alive
        return g.replay


# Host-operand entry points reuse one trainer (workspace + pinned staging) per
# training shape: repeated calls of the drop-in API (bench steps, CLI runs,
# cross-validation loops) pay no allocation.  A lock serialises the cached
# trainers' use across host threads (one rendezvous thread per run_local).
_TRAINERS: "OrderedDict" = OrderedDict()
_TRAINER_CACHE_MAX = 2
_TRAIN_LOCK = threading.Lock()


def _cached_trainer(n: int, nf: int, cfg: TrainConfig, device, host_io: bool) -> "DeviceTrainer":
    torch = _native.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (n, nf, repr(cfg), str(dev), host_io)
    tr = _TRAINERS.pop(key, None)
    if tr is None:
        while len(_TRAINERS) >= _TRAINER_CACHE_MAX:
            _TRAINERS.popitem(last=False)
        tr = DeviceTrainer(n, nf, cfg, device=dev, host_io=host_io)
        if host_io:
            slots = (1 << tr.depth) - 1
            pin = lambda *shape: torch.empty(shape, dtype=torch.int64).pin_memory()  # noqa: E731
            tr.staging = {"X": pin(3, n, nf), "Y": pin(3, n), "fill": pin(slots), "T": pin(3, slots),
                          "F": pin(3, slots)}
    _TRAINERS[key] = tr
    return tr


def train_pairs(x_pairs: Sequence, y_pairs: Sequence, cfg: TrainConfig, seeds: SeedSetup, dealer_seed: bytes,
                *, device=None, check: bool = True) -> Tuple[np.ndarray, np.ndarray, int]:
    """train_components on the three parties' (lo, hi) pairs (x: (N, nf), y:
    (N,) per party): heuristic mpc stages the pairs straight into the cached
    trainer's pinned buffers (replication check on the way), no intermediate
    component array."""
    from .shares import ShareError, components_from_pairs, stage_pairs

    cfg = as_config(cfg)
    lo0 = np.asarray(x_pairs[0][0])
    if lo0.ndim != 2 or np.asarray(y_pairs[0][0]).shape != (lo0.shape[0],):
        raise ValueError("features must be (n, nf) and labels (n,) per party")
    n, nf = lo0.shape
    if n == 0:
        raise ValueError("dataset is empty")
    if cfg.heuristic != "mpc":
        X = components_from_pairs(x_pairs, RING64, check)
        Y = components_from_pairs(y_pairs, RING64, check)
        return train_components(X, Y, cfg, seeds, dealer_seed, device=device)
    keys = make_keys(seeds, dealer_seed)
    torch = _native.require_cuda()
    with _TRAIN_LOCK:
        tr = _cached_trainer(n, nf, cfg, device, True)
        st = tr.staging
        stage_pairs(x_pairs, st["X"].numpy().view(np.uint64), False)
        stage_pairs(y_pairs, st["Y"].numpy().view(np.uint64), False)
        st["fill"].numpy().view(np.uint64)[:] = filler_values(seeds.filler_seed, (1 << tr.depth) - 1, nf + 1)
        s = torch.cuda.current_stream(tr.device)
        replay = tr.host_graph(keys)
        if replay is not None:  # one graph launch instead of ~370 eager launches per tree
            with torch.cuda.device(tr.device):
                replay()
            depth = tr.depth
        else:
            depth = tr.run_host(st["X"], st["Y"], st["fill"], st["T"], st["F"], keys, stream=s)
        # the replication check (rss.py:222-228) runs on host threads while the
        # device trains; an inconsistent pair still raises, after the run
        try:
            if check:
                stage_pairs(x_pairs, None, True)
                stage_pairs(y_pairs, None, True)
        finally:
            s.synchronize()
        slots = (1 << depth) - 1
        return (st["T"].numpy().view(np.uint64)[:, :slots].copy(),
                st["F"].numpy().view(np.uint64)[:, :slots].copy(), depth)


def train_components(X: np.ndarray, Y: np.ndarray, cfg: TrainConfig, seeds: SeedSetup, dealer_seed: bytes,
                     *, device=None) -> Tuple[np.ndarray, np.ndarray, int]:
    """Whole-run entry on component-major shares: X [3, N, nf], Y [3, N]
    uint64 -> (T [3, slots], F [3, slots], depth) component shares.
    Heuristic mpc goes through gt_train_host (pinned staging, chunked upload
    beside the prologue); tee through gt_train_ex (its helper callback)."""
    X = np.asarray(X, dtype=np.uint64)
    Y = np.asarray(Y, dtype=np.uint64)
    if X.ndim != 3 or X.shape[0] != 3 or Y.shape != (3, X.shape[1]):
        raise ValueError("features must be [3, n, nf] and labels [3, n]")
    n, nf = X.shape[1], X.shape[2]
    if n == 0:
        raise ValueError("dataset is empty")
    cfg = as_config(cfg)
    keys = make_keys(seeds, dealer_seed)
    with _TRAIN_LOCK:
        if cfg.heuristic == "mpc":
            torch = _native.require_cuda()
            tr = _cached_trainer(n, nf, cfg, device, True)
            st = tr.staging
            np.copyto(st["X"].numpy().view(np.uint64), X)
            np.copyto(st["Y"].numpy().view(np.uint64), Y)
            st["fill"].numpy().view(np.uint64)[:] = filler_values(seeds.filler_seed, (1 << tr.depth) - 1, nf + 1)
            s = torch.cuda.current_stream(tr.device)
            depth = tr.run_host(st["X"], st["Y"], st["fill"], st["T"], st["F"], keys, stream=s)
            s.synchronize()
            slots = (1 << depth) - 1
            return (st["T"].numpy().view(np.uint64)[:, :slots].copy(),
                    st["F"].numpy().view(np.uint64)[:, :slots].copy(), depth)
        tr = _cached_trainer(n, nf, cfg, device, False)
        fill = filler_values(seeds.filler_seed, (1 << tr.depth) - 1, nf + 1)
        depth = tr.run(to_device(X, tr.device), to_device(Y, tr.device), to_device(fill, tr.device), keys,
                       enclave_seed=seeds.enclave_seed)
        slots = (1 << depth) - 1
        return from_device(tr.T)[:, :slots].copy(), from_device(tr.F)[:, :slots].copy(), depth


def train_3pc(x_pairs: Sequence, y_pairs: Sequence, cfg: TrainConfig, seeds: SeedSetup, dealer_seed: bytes,
              *, device=None, check: bool = True):
    """Whole-run entry on the three parties' replicated pairs (the form
    ``share_values`` returns, dealer.py:259-263): x_pairs[i] = (lo, hi) of
    party i+1, lo/hi shaped (N, nf); y_pairs[i] shaped (N,).  Returns
    (T_pairs, F_pairs, depth) in the same per-party form."""
    X = components_from_pairs(x_pairs, RING64, check)
    Y = components_from_pairs(y_pairs, RING64, check)
    if X.ndim != 3:
        raise ValueError("features must be (n, nf) per party")
    T, F, depth = train_components(X, Y.reshape(3, -1), cfg, seeds, dealer_seed, device=device)
    from .shares import pairs_from_components

    return pairs_from_components(T), pairs_from_components(F), depth
