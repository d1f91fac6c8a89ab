"""Drop-in per-party API: ``run_local`` / ``train_tree`` / ``infer_batch``.

The reference runs the same protocol body on three party threads
(``run_local``, rss.py:496-542) and each body calls ``train_tree(eng, X, y,
cfg)`` (train.py:108) or ``infer_batch(eng, levels, queries)``
(infer.py:20) on its own share pair.  Here the three co-resident parties meet
at a rendezvous -- the pattern of the reference's ``EnclaveBridge``
(transport.py:304-342): the three engines hand in their pairs, the last one
to arrive checks replication consistency, runs ONE device call for all three
parties, and every engine gets its own pair of the result back.  The
run's transcript is the analytic ledger of exactly that protocol
(ledger.py), so ``LocalRun.metrics`` reads like the reference's.
"""

from __future__ import annotations

import queue
import threading
import time
from typing import Callable, List, Optional, Sequence, Union

import numpy as np

from .ledger import REF_LANE_LIMIT, Ledger, Metrics, Transcript
from .seeds import PARTIES, SeedSetup, derive_seed, filler_values, make_keys
from .shares import RING64, AVec, ShareError, avecs_from_components, components_from_avecs, ring_of
from .train import TrainConfig, TrainResult, as_config, resolved_depth, train_pairs


class TransportError(RuntimeError):
    """transport.py:40-41."""


class _Rendezvous:
    """Gather one request per party, compute once, scatter (EnclaveBridge)."""

    def __init__(self, timeout: float):
        self.timeout = timeout
        self._cv = threading.Condition()
        self._requests = {}
        self._responses = {}
        self._error: Optional[BaseException] = None
        self._generation = 0
        self.aborted = False

    def abort(self) -> None:
        with self._cv:
            self.aborted = True
            self._cv.notify_all()

    def call(self, party: int, name: str, payload, compute: Callable[[List], List]):
        with self._cv:
            if self.aborted:
                raise TransportError("round barrier broken (peer died or deadlock timeout)")
            gen = self._generation
            self._requests[party] = (name, payload)
            if len(self._requests) == 3:
                names = {self._requests[p][0] for p in PARTIES}
                try:
                    if len(names) != 1:
                        raise TransportError(f"parties diverged: round tags {sorted(names)}")
                    outs = compute([self._requests[p][1] for p in PARTIES])
                    self._responses = {p: outs[p - 1] for p in PARTIES}
                    self._error = None
                except BaseException as e:  # noqa: BLE001 - re-raised on every party
                    self._responses = {}
                    self._error = e
                self._requests = {}
                self._generation += 1
                self._cv.notify_all()
            else:
                deadline = time.monotonic() + self.timeout
                while self._generation == gen and not self.aborted:
                    left = deadline - time.monotonic()
                    if left <= 0:
                        raise TransportError("rendezvous timed out")
                    self._cv.wait(timeout=left)
                if self.aborted and self._generation == gen:
                    raise TransportError("round barrier broken (peer died or deadlock timeout)")
            if self._error is not None:
                raise self._error
            return self._responses[party]


class PartyEngine:
    """One party's handle (rss.py:270-298).  Protocol bodies written for the
    reference receive this object; its device work happens at rendezvous."""

    def __init__(self, party: int, seeds: SeedSetup, bridge: _Rendezvous, ledger: Ledger, dealer_seed: bytes,
                 material=None, lane_limit: int = REF_LANE_LIMIT, device=None):
        if party not in PARTIES:
            raise ShareError(f"invalid party id {party}")
        self.party = party
        self.seeds = seeds
        self.material = material
        self.lane_limit = lane_limit
        self.dealer_seed = dealer_seed
        self.device = device
        self._bridge = bridge
        self._ledger = ledger
        self._phase: List[str] = []

    def phase(self, label: str):
        return _Phase(self, label)

    def tag(self, fallback: str) -> str:
        return self._phase[-1] if self._phase else fallback


class _Phase:
    def __init__(self, eng: PartyEngine, label: str):
        self.eng, self.label = eng, label

    def __enter__(self):
        self.eng._phase.append(self.label)
        return self

    def __exit__(self, *exc):
        self.eng._phase.pop()
        return False


def _own(eng) -> "PartyEngine":
    if not isinstance(eng, PartyEngine):
        raise TransportError("the B200 drop-ins run the three parties co-resident on the device: call them "
                             "from a body executed by this package's run_local (the reference's TCP seats "
                             "are not a B200 transport)")
    return eng


class LocalRun:
    """rss.py:489-493: results per party, the transcript and its metrics
    (summarised from the transcript on first access)."""

    def __init__(self, results: List, transcript: Transcript, metrics: Optional[Metrics] = None):
        self.results = results
        self.transcript = transcript
        self._metrics = metrics

    @property
    def metrics(self) -> Metrics:
        if self._metrics is None:
            self._metrics = Metrics.from_transcript(self.transcript)
        return self._metrics


class _PartyPool:
    """Three persistent party threads (party1..party3) that run_local hands
    its bodies to: starting three fresh threads per call costs ~0.5 ms of
    thread start-up on the host path of every tree.  A call that times out
    leaves its stuck threads behind and retires the pool (the next call
    starts a new one)."""

    def __init__(self):
        self.tasks = [queue.SimpleQueue() for _ in PARTIES]
        self.broken = False
        for i in range(3):
            threading.Thread(target=self._worker, args=(i,), name=f"party{i + 1}", daemon=True).start()

    def _worker(self, i: int) -> None:
        while True:
            job, done = self.tasks[i].get()
            try:
                job()
            finally:
                done.release()

    def run(self, jobs: Sequence[Callable[[], None]], timeout: float) -> bool:
        """Run the three jobs on the party threads; False if they did not all
        finish within `timeout` seconds."""
        done = threading.Semaphore(0)
        for i, job in enumerate(jobs):
            self.tasks[i].put((job, done))
        deadline = time.monotonic() + timeout
        for _ in jobs:
            if not done.acquire(timeout=max(0.0, deadline - time.monotonic())):
                self.broken = True
                return False
        return True


_POOL: Optional[_PartyPool] = None
_POOL_LOCK = threading.Lock()


def _party_pool() -> Optional[_PartyPool]:
    """The process's party threads, or None when a run_local call is already
    using them (a nested or concurrent call gets fresh threads)."""
    global _POOL
    if not _POOL_LOCK.acquire(blocking=False):
        return None
    if _POOL is None or _POOL.broken:
        _POOL = _PartyPool()
    return _POOL


def run_local(fn: Callable[[PartyEngine], object], *, seeds: Union[SeedSetup, int], materials: Optional[Sequence] = None,
              enclave_handler=None, lane_limit: int = REF_LANE_LIMIT, timeout: float = 300.0,
              dealer_seed: Optional[bytes] = None, device=None) -> LocalRun:
    """rss.py:496-542 with the three engines meeting on the device.
    `materials` / `enclave_handler` are accepted for signature compatibility:
    correlated material is generated in-kernel from `dealer_seed`
    (default derive_seed(master, "live-dealer"), as cli.cmd_train)."""
    if isinstance(seeds, int):
        seeds = SeedSetup.from_int(seeds)
    if dealer_seed is None:
        dealer_seed = derive_seed(seeds.master, "live-dealer")
    bridge = _Rendezvous(timeout)
    ledger = Ledger(lane_limit)
    engines = [PartyEngine(i, seeds, bridge, ledger, dealer_seed, materials[i - 1] if materials else None, lane_limit,
                           device) for i in PARTIES]
    results: List = [None, None, None]
    errors: List = [None, None, None]

    def body(idx: int) -> None:
        try:
            results[idx] = fn(engines[idx])
        except BaseException as e:  # noqa: BLE001 - propagated below
            errors[idx] = e
            bridge.abort()

    pool = _party_pool()
    if pool is not None:
        try:
            finished = pool.run([lambda i=i: body(i) for i in range(3)], timeout * 4)
        finally:
            _POOL_LOCK.release()
        if not finished:
            bridge.abort()
            raise TransportError("party thread failed to finish")
    else:
        threads = [threading.Thread(target=body, args=(i,), name=f"party{i + 1}", daemon=True) for i in range(3)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=timeout * 4)
            if t.is_alive():
                bridge.abort()
                raise TransportError("party thread failed to finish")
    for e in errors:
        if e is not None and not isinstance(e, TransportError):
            raise e
    for e in errors:
        if e is not None:
            raise e
    return LocalRun(results=results, transcript=ledger.transcript)


def train_tree(eng: PartyEngine, features, labels, cfg: TrainConfig) -> TrainResult:
    """Per-party drop-in for train.py:108 (SPMD; all three parties call it).
    `cfg` may be this package's TrainConfig or the reference's own."""
    _own(eng)
    n_samples, nf = features.shape
    cfg = as_config(cfg)

    def compute(payloads):
        T, F, depth = train_pairs([(p[0].lo, p[0].hi) for p in payloads],
                                  [(p[1].lo.reshape(-1), p[1].hi.reshape(-1)) for p in payloads], cfg, eng.seeds,
                                  eng.dealer_seed, device=eng.device)
        eng._ledger.train(n_samples, nf, resolved_depth(cfg, nf + 1), cfg.tau, cfg.score_ring.width,
                          grow_stop_level=depth - 1, policy=cfg.policy, heuristic=cfg.heuristic,
                          count_reshare=cfg.count_reshare)
        tv, fv = avecs_from_components(T, RING64), avecs_from_components(F, RING64)
        return [TrainResult(T=tv[i], F=fv[i], depth=depth) for i in range(3)]

    return eng._bridge.call(eng.party, "train_tree", (features, labels), compute)


def infer_batch(eng: PartyEngine, levels: List, queries) -> AVec:
    """Per-party drop-in for infer.py:20 (levels sizes 1, 2, 4, ...)."""
    _own(eng)
    n_queries, nf = queries.shape
    depth = len(levels)

    def compute(payloads):
        from .infer import infer_components

        tree = np.concatenate([components_from_avecs([p[0][t] for p in payloads]) for t in range(depth)], axis=1)
        Q = components_from_avecs([p[1] for p in payloads])
        keys = make_keys(eng.seeds, eng.dealer_seed)
        out, _ = infer_components(tree, depth, Q, keys, device=eng.device)
        eng._ledger.infer(n_queries, nf, depth)
        return avecs_from_components(out, ring_of(levels[0]))

    return eng._bridge.call(eng.party, "infer_batch", (levels, queries), compute)


def _lookup(eng: PartyEngine, name: str, table, idx, per_row: bool):
    _own(eng)
    ring = ring_of(table)
    shape = tuple(idx.shape)

    def compute(payloads):
        from . import gadgets as G
        from .shares import from_device, to_device

        tab = components_from_avecs([p[0] for p in payloads])
        ix = components_from_avecs([p[1] for p in payloads]).reshape(3, -1)
        keys = make_keys(eng.seeds, eng.dealer_seed)
        op = 0x40000000 | eng._ledger.round_no  # fresh randomness per call site
        dev = eng.device if eng.device is not None else "cuda"
        if per_row:
            out = G.row_lookup(ring.width, to_device(tab, dev), to_device(ix, dev), keys=keys, op=op)
        else:
            out = G.oaa(ring.width, to_device(tab.reshape(3, -1), dev), to_device(ix, dev), keys=keys, op=op)
        if eng._phase:  # the caller's phase tags the records, as in the reference transcript
            with eng._ledger.phase(eng._phase[-1]):
                eng._ledger.oaa(ix.shape[1], tab.shape[-1], ring.width)
        else:
            eng._ledger.oaa(ix.shape[1], tab.shape[-1], ring.width)
        return avecs_from_components(from_device(out).reshape((3,) + shape), ring)

    return eng._bridge.call(eng.party, name, (table, idx), compute)


def oaa(eng: PartyEngine, table, idx) -> AVec:
    """Per-party drop-in for oaa.py:20-35: shares of table[idx], zero where
    idx is out of range (ValueError unless `table` is one-dimensional)."""
    _own(eng)
    if len(table.shape) != 1:
        raise ValueError("table must be one-dimensional")
    return _lookup(eng, "oaa", table, idx, per_row=False)


def row_lookup(eng: PartyEngine, rows, idx) -> AVec:
    """Per-party drop-in for oaa.py:38-55: out[i] = rows[i][idx[i]]."""
    _own(eng)
    if len(rows.shape) != 2:
        raise ValueError("rows must be two-dimensional")
    if idx.size != rows.shape[0]:
        raise ValueError("one index per row required")
    return _lookup(eng, "row_lookup", rows, idx, per_row=True)


def open_results(run: LocalRun, pick=lambda r: r) -> np.ndarray:
    """Reconstruct a vector from the three parties' returned AVecs."""
    return components_from_avecs([pick(r) for r in run.results]).sum(axis=0, dtype=np.uint64)
