"""Analytic inter-party message ledger.

On the device the three parties share one register file, so an ``open`` or a
reshare is an algebraic identity, not a message.  The protocol still has a
definite communication pattern -- it is what a three-host deployment would
send -- and it depends only on public shapes (the reference's obliviousness
property, test_acceptance.py:255-306).  This module restates that pattern:
for every gadget call of the training / inference schedule it appends the
same (round, sender, receiver, nbytes, tag) records the reference's
``InprocRouter`` commits (transport.py:131-286), so the bytes and rounds a
B200 run reports sit next to the reference's like for like.

``lane_limit`` reproduces the reference's chunking of wide lane batches
(oaa.py:58-63, train.py:207-221); ``lane_limit=None`` is the device schedule
(every gadget call is a single batch, so fewer rounds, same bytes up to the
bit-packing of partial bytes).
"""

from __future__ import annotations

import json
import math
from contextlib import contextmanager
from typing import Dict, Iterable, List, Optional, Tuple

PARTIES = (1, 2, 3)
REF_LANE_LIMIT = 1 << 22  # PartyEngine default, rss.py:277

Record = Tuple[int, int, int, int, str]


def next_party(i: int) -> int:
    return i % 3 + 1


def prev_party(i: int) -> int:
    return (i - 2) % 3 + 1


class Transcript:
    """transport.py:136-161."""

    def __init__(self) -> None:
        self.records: List[Record] = []

    def append(self, round_no: int, sender: int, receiver: int, nbytes: int, tag: str) -> None:
        self.records.append((round_no, sender, receiver, nbytes, tag))

    def shape(self) -> Tuple[Record, ...]:
        return tuple(self.records)

    def total_bytes(self, sender: Optional[int] = None) -> int:
        return sum(r[3] for r in self.records if sender is None or r[1] == sender)

    def rounds(self) -> int:
        return max((r[0] for r in self.records), default=0)


class Metrics:
    """transport.py:164-202."""

    def __init__(self, rounds: int, bytes_by_pair: Dict[str, int], bytes_by_tag: Dict[str, int],
                 rounds_by_tag: Dict[str, int]):
        self.rounds = rounds
        self.bytes_by_pair = bytes_by_pair
        self.bytes_by_tag = bytes_by_tag
        self.rounds_by_tag = rounds_by_tag

    @classmethod
    def from_transcript(cls, transcript: Transcript) -> "Metrics":
        pair: Dict[str, int] = {}
        tagb: Dict[str, int] = {}
        tag_rounds: Dict[str, set] = {}
        for rnd, s, r, n, tag in transcript.records:
            key = f"{s}->{r}"
            pair[key] = pair.get(key, 0) + n
            tagb[tag] = tagb.get(tag, 0) + n
            tag_rounds.setdefault(tag, set()).add(rnd)
        return cls(rounds=transcript.rounds(), bytes_by_pair=dict(sorted(pair.items())),
                   bytes_by_tag=dict(sorted(tagb.items())),
                   rounds_by_tag={k: len(v) for k, v in sorted(tag_rounds.items())})

    def total_bytes(self) -> int:
        return sum(self.bytes_by_pair.values())

    def sent_by_party(self, party: int) -> int:
        return sum(v for k, v in self.bytes_by_pair.items() if k.startswith(f"{party}->"))

    def to_dict(self) -> dict:
        return {"rounds": self.rounds, "total_bytes": self.total_bytes(), "bytes_by_pair": self.bytes_by_pair,
                "bytes_by_phase": self.bytes_by_tag, "rounds_by_phase": self.rounds_by_tag}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)


def _packed(nbits: int) -> int:
    return (nbits + 7) // 8  # np.packbits, rss.py:255-256


class Ledger:
    """Shape-only replay of the reference's communication."""

    def __init__(self, lane_limit: Optional[int] = REF_LANE_LIMIT) -> None:
        self.transcript = Transcript()
        self.round_no = 0
        self.lane_limit = lane_limit
        self._phase: List[str] = []

    # -- bookkeeping ---------------------------------------------------------
    @contextmanager
    def phase(self, label: str):
        self._phase.append(label)
        try:
            yield self
        finally:
            self._phase.pop()

    def tag(self, fallback: str) -> str:
        return self._phase[-1] if self._phase else fallback

    def _round(self, msgs: Iterable[Tuple[int, int, int]], tag: str) -> None:
        msgs = sorted(msgs)  # canonical (sender, receiver) order, transport.py:253-270
        if not msgs:
            return
        self.round_no += 1
        for s, r, n in msgs:
            self.transcript.append(self.round_no, s, r, n, tag)

    def metrics(self) -> Metrics:
        return Metrics.from_transcript(self.transcript)

    # -- communicating primitives (rss.py:371-412) ---------------------------
    def open_a(self, n: int, width: int, tag: str = "open") -> None:
        self._round(((p, next_party(p), n * (width // 8)) for p in PARTIES), self.tag(tag))

    def open_bits(self, n: int, tag: str = "open_bits") -> None:
        self._round(((p, next_party(p), _packed(n)) for p in PARTIES), self.tag(tag))

    def mul(self, n: int, width: int, tag: str = "mul") -> None:
        self._round(((p, prev_party(p), n * (width // 8)) for p in PARTIES), self.tag(tag))

    def and_bits(self, n: int, tag: str = "and") -> None:
        self._round(((p, prev_party(p), _packed(n)) for p in PARTIES), self.tag(tag))

    def or_bits(self, n: int) -> None:
        self.and_bits(n, "or")

    def enclave_call(self, up: int, down: int, tag: str) -> None:
        """EnclaveBridge.call (transport.py:316-342): one request up from every
        party, one response down; two rounds, records interleaved per party."""
        tag = self.tag(tag)
        up_r, down_r = self.round_no + 1, self.round_no + 2
        self.round_no = down_r
        for p in PARTIES:
            self.transcript.append(up_r, p, 0, up, tag)
            self.transcript.append(down_r, 0, p, down, tag)

    # -- gadgets (gadgets.py) -------------------------------------------------
    def and_reduce(self, k: int, n: int) -> None:  # gadgets.py:94-109
        while k > 1:
            half = k // 2
            self.and_bits(half * n)
            k = half + k % 2

    def eq(self, n: int, width: int) -> None:  # gadgets.py:120-130
        self.open_a(n, width, "eq.open")
        self.and_reduce(width, n)

    def prefix_borrow(self, width: int, n: int) -> None:  # gadgets.py:137-160
        shift = 1
        while shift < width:
            self.and_bits(2 * (width - shift) * n)
            shift *= 2

    def lt(self, n: int, width: int) -> None:  # gadgets.py:188-216
        self.open_a(2 * n, width, "lt.open")
        self.prefix_borrow(width, 2 * n)
        self.and_bits(width * n, "lt.gen")
        self.prefix_borrow(width, n)

    def b2a(self, n: int) -> None:  # gadgets.py:223-231
        self.open_bits(n, "b2a.open")

    def select(self, n_cond: int, n_payload: int, width: int) -> None:  # gadgets.py:238-253
        self.b2a(n_cond)
        self.mul(n_payload, width, "select.mul")

    def truncate(self, n: int, width: int, k: int) -> None:  # gadgets.py:260-288
        if k == 0:
            return
        self.open_a(n, width, "trunc.open")
        self.prefix_borrow(width, n)
        self.b2a(2 * n)

    def division(self, n: int, width: int, tau: int) -> None:  # gadgets.py:310-349
        d = div_params(width, tau)
        ladder = d["bound"] - 1
        self.lt(ladder * n, width)
        self.b2a(ladder * n)
        self.mul(n, width, "div.mul")
        self.truncate(n, width, d["bound"] - d["ti"])
        for _ in range(d["iters"]):
            self.mul(n, width, "div.mul")
            self.truncate(n, width, d["ti"])
            self.mul(n, width, "div.mul")
            self.truncate(n, width, d["ti"])
        self.mul(n, width, "div.mul")
        if d["sigma"]:
            self.truncate(n, width, d["sigma"])
        self.mul(n, width, "div.mul")
        self.truncate(n, width, d["kf"])

    def argmin(self, n: int, m: int, score_width: int, idx_width: int = 64) -> None:  # gadgets.py:366-401
        self.select(n * m, n * m, score_width)
        while m > 1:
            pairs = m // 2
            self.lt(n * pairs, score_width)
            self.select(n * pairs, n * pairs, score_width)
            self.select(n * pairs, n * pairs, idx_width)
            m = pairs + m % 2

    # -- oblivious lookup (oaa.py) -------------------------------------------
    def _chunks(self, n: int, m: int):
        if self.lane_limit is None:
            if n:
                yield n
            return
        step = max(1, self.lane_limit // max(m, 1))
        for lo in range(0, n, step):
            yield min(lo + step, n) - lo

    def oaa(self, n: int, m: int, width: int) -> None:  # oaa.py:20-35
        for span in self._chunks(n, m):
            self.eq(span * m, width)
            self.select(span * m, span * m, width)

    row_lookup = oaa  # oaa.py:38-55 has the identical message pattern

    # -- protocols ------------------------------------------------------------
    def count_level(self, n: int, n_nodes: int, nf: int, dot: bool = False) -> None:  # train.py:201-229
        width = 2 * nf + 1
        self.eq(n_nodes, 64)
        if self.lane_limit is None:
            spans = [n] if n else []
        else:
            step = max(1, self.lane_limit // max(n_nodes * width, 1))
            spans = [min(lo + step, n) - lo for lo in range(0, n, step)]
        for span in spans:
            self.eq(span * n_nodes, 64)
            self.and_bits(span * n_nodes)
            self.b2a(span * n_nodes)
            if not dot:
                self.mul(span * n_nodes * width, 64, "count.mul")
        if dot and spans:  # one reshare of the summed cells (count_reshare="dot")
            self.mul(n_nodes * width, 64, "count.mul")

    def heuristic_mpc(self, n_nodes: int, nf: int, n_samples: int, tau: int, score_width: int) -> None:
        cols = 2 * nf  # train.py:232-274
        self.eq(3 * n_nodes, 64)
        self.and_reduce(nf, n_nodes)
        self.or_bits(n_nodes)
        self.or_bits(n_nodes)
        self.and_bits(n_nodes)
        self.select(n_nodes, n_nodes, 64)
        shift = counter_shift(n_samples, score_width, tau)
        if shift:
            self.truncate(n_nodes * 3 * cols, 64, shift)
        self.mul(4 * n_nodes * cols, score_width, "hc.mul")
        self.eq(n_nodes * cols, score_width)
        self.b2a(n_nodes * cols)
        self.division(n_nodes * cols, score_width, tau)
        self.argmin(n_nodes, nf, score_width, 64)
        self.eq(n_nodes * nf, 64)
        self.and_bits(n_nodes * nf)

    def heuristic_tee(self, n_nodes: int, nf: int) -> None:  # train.py:277-292, enclave.py:60-86
        cells = n_nodes * 3 * 2 * nf
        up = 16 + 16 * cells + 2 * n_nodes * nf + 16 * n_nodes
        down = 16 * n_nodes + 16 * n_nodes + 2 * n_nodes + 2 * n_nodes * nf
        self.enclave_call(up, down, "hc_tee")

    def labels_tee(self, n_nodes: int, nf: int) -> None:  # train.py:295-301
        self.enclave_call(16 + 16 * n_nodes * 3 * 2 * nf, 16 * n_nodes, "labels_tee")

    # -- whole-call replays, memoised per shape --------------------------------
    # The records of one train / infer call depend only on public shapes, so a
    # repeated call (the drop-in API run per tree) replays its records from a
    # cache, shifted to the ledger's current round.
    _MEMO: Dict[tuple, Tuple[List[Record], int, object]] = {}

    def _memo(self, key: tuple, build):
        key = (key, self.lane_limit, tuple(self._phase))
        hit = Ledger._MEMO.get(key)
        r0 = self.round_no
        if hit is None:
            start = len(self.transcript.records)
            ret = build()
            recs = [(r - r0, s, t, n, tag) for r, s, t, n, tag in self.transcript.records[start:]]
            if len(Ledger._MEMO) > 64:
                Ledger._MEMO.clear()
            Ledger._MEMO[key] = (recs, self.round_no - r0, ret)
            return ret
        recs, nrounds, ret = hit
        if r0 == 0:  # a fresh ledger (one run_local call): the cached records as they are
            self.transcript.records.extend(recs)
        else:
            self.transcript.records.extend((r + r0, s, t, n, tag) for r, s, t, n, tag in recs)
        self.round_no = r0 + nrounds
        return ret

    def train(self, n: int, nf: int, depth: int, tau: int = 10, score_width: int = 32,
              grow_stop_level: Optional[int] = None, policy: str = "fixed", heuristic: str = "mpc",
              count_reshare: str = "elementwise") -> int:
        """train_tree (train.py:108-197).  Under the grow policy the opened
        stop bit is data dependent; pass the level the run stopped at."""
        args = (n, nf, depth, tau, score_width, grow_stop_level, policy, heuristic, count_reshare)
        return self._memo(("train",) + args, lambda: self._train(*args))

    def _train(self, n: int, nf: int, depth: int, tau: int, score_width: int, grow_stop_level: Optional[int],
               policy: str, heuristic: str, count_reshare: str) -> int:
        with self.phase("count:0"):
            self.mul(n * nf, 64, "count.mul")
        for level in range(depth):
            n_nodes = 1 << level
            if level > 0:
                with self.phase(f"partition:{level}"):
                    self.oaa(n, 1 << (level - 1), 64)
                    self.row_lookup(n, nf, 64)
            with self.phase(f"count:{level}"):
                self.count_level(n, n_nodes, nf, dot=count_reshare == "dot")
            last = level == depth - 1
            if not last:
                if heuristic == "tee":
                    with self.phase(f"hc_tee:{level}"):
                        self.heuristic_tee(n_nodes, nf)
                else:
                    with self.phase(f"hc_mpc:{level}"):
                        self.heuristic_mpc(n_nodes, nf, n, tau, score_width)
            with self.phase(f"replace:{level}"):
                if level > 0:
                    self.eq(n_nodes, 64)
                    self.select(n_nodes, n_nodes * 3 * 2 * nf, 64)
            do_labels = last
            if not last and policy == "grow":
                with self.phase(f"stop:{level}"):
                    self.and_reduce(n_nodes, 1)
                    self.open_bits(1, "stop")
                do_labels = grow_stop_level == level
            if not do_labels:
                with self.phase(f"split:{level}"):
                    self.select(n_nodes, n_nodes, 64)
                    self.select(n_nodes, n_nodes, 64)
                    self.select(n_nodes, n_nodes * 3 * 2 * nf, 64)
                continue
            with self.phase(f"labels:{level}"):
                if heuristic == "tee":
                    self.labels_tee(n_nodes, nf)
                else:
                    self.lt(n_nodes, 64)
                    self.b2a(n_nodes)
            return level + 1
        raise AssertionError("unreachable")

    def infer(self, n: int, nf: int, depth: int) -> None:  # infer.py:20-35
        self._memo(("infer", n, nf, depth), lambda: self._infer(n, nf, depth))

    def _infer(self, n: int, nf: int, depth: int) -> None:
        for t in range(depth):
            with self.phase(f"walk:{t}"):
                self.oaa(n, 1 << t, 64)
                self.row_lookup(n, nf, 64)


def div_params(width: int, tau: int) -> Dict[str, int]:
    """gadgets.py:297-307."""
    bound = width - tau - 2
    ti = tau + 4
    sigma = max(0, bound + ti + 5 - width)
    kf = bound + ti - sigma - tau
    iters = math.ceil(math.log2(tau)) + 2 if tau > 1 else 2
    if ti >= bound or kf < 1:
        raise ValueError(f"division unsupported at width {width}, tau {tau}")
    w0 = round(2.9142 * (1 << ti))
    return {"bound": bound, "ti": ti, "sigma": sigma, "kf": kf, "iters": iters, "w0": w0}


def counter_shift(n_samples: int, score_width: int = 32, tau: int = 10) -> int:
    """train.py:75-78."""
    headroom = (score_width - tau - 2) // 2
    return max(0, int(n_samples).bit_length() - headroom)


def train_metrics(n: int, nf: int, depth: int, tau: int = 10, score_width: int = 32,
                  lane_limit: Optional[int] = REF_LANE_LIMIT) -> Metrics:
    led = Ledger(lane_limit)
    led.train(n, nf, depth, tau, score_width)
    return led.metrics()


def infer_metrics(n: int, nf: int, depth: int, lane_limit: Optional[int] = REF_LANE_LIMIT) -> Metrics:
    led = Ledger(lane_limit)
    led.infer(n, nf, depth)
    return led.metrics()
