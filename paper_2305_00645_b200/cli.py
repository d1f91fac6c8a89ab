"""Command line for the B200 path (reference pkg/src/obtree/cli.py).

``python -m paper_2305_00645_b200.cli {train,infer,compare,bench}`` with the
reference's flags, config-file precedence (cli.py:161-222), exit codes
(cli.py:53-56) and output files: per-party ``tree_T.shr`` / ``tree_F.shr`` /
``predictions.shr`` in the reference's OBS1 share-file format (rss.py:452-481,
so shares move between the two implementations), ``tree_meta.json``,
``metrics.json`` (the ledger's transcript, identical to the reference's for
the same run), and ``tree.json`` / ``predictions.csv`` under
``--profile test --reveal``.  Inputs are shared exactly as the reference CLI
shares them (share_values over derive_seed(seed, "deal/...")); every share
computation runs on the device.  ``--deal-dir`` reads a directory written by
the reference's ``obtree deal`` (features.shr / labels.shr / seeds.json /
enclave.json; the correlated-material bank is regenerated in-kernel).
Out of scope: material.bin, binarize, the enclave server, TCP seats.
"""

from __future__ import annotations

import argparse
import json
import logging
import os
import sys
import time
from dataclasses import dataclass
from pathlib import Path
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import tree as tree_mod
from ._native import ProtocolError
from .enclave import EnclaveError
from .engine import TransportError
from .ledger import Ledger, Metrics
from .seeds import PARTIES, SeedSetup, derive_seed, make_keys, share_values
from .shares import RING64, Ring, RingError, ShareError, components_from_pairs, pairs_from_components, \
    read_share_file, write_share_file

log = logging.getLogger("gtree_b200")

EXIT_OK, EXIT_USAGE, EXIT_PROTOCOL, EXIT_MISMATCH = 0, 1, 2, 3
TREE_T_NAME, TREE_F_NAME = "tree_T.shr", "tree_F.shr"
TREE_META_NAME, METRICS_NAME, META_NAME = "tree_meta.json", "metrics.json", "meta.json"


class UsageError(Exception):
    """cli.py:61-62."""


class CompareMismatch(Exception):
    """cli.py:65-66."""


@dataclass
class RunConfig:
    """cli.py:74-123 (in-process subset) + the B200 count_reshare option."""

    width: int = 32
    tau: int = 10
    depth: int = 4
    policy: str = "fixed"
    max_depth: Optional[int] = None
    heuristic: str = "mpc"
    seed: bytes = bytes(16)
    reveal: bool = False
    profile: str = "prod"
    lane_limit: int = 1 << 22
    timeout: float = 300.0
    count_reshare: str = "elementwise"

    def validate(self) -> None:
        if self.width < 8 or self.width > 64:
            raise UsageError("score ring width must be between 8 and 64")
        if not 0 < self.tau < self.width - 2:
            raise UsageError("tau must satisfy 0 < tau < width - 2")
        if self.depth < 1:
            raise UsageError("depth must be at least 1")
        if self.policy not in ("fixed", "grow", "feature_cap"):
            raise UsageError(f"unknown depth policy {self.policy!r}")
        if self.heuristic not in ("mpc", "tee"):
            raise UsageError(f"unknown heuristic path {self.heuristic!r}")
        if self.reveal and self.profile != "test":
            raise UsageError("--reveal is only honored in the test profile")

    def train_config(self):
        from .train import TrainConfig

        return TrainConfig(depth=self.depth, tau=self.tau, heuristic=self.heuristic, policy=self.policy,
                           max_depth=self.max_depth, score_ring=Ring(self.width), count_reshare=self.count_reshare)


def parse_seed(text: str) -> bytes:
    """Decimal integer or hex string (cli.py:126-140)."""
    s = text.strip()
    try:
        return int(s, 10).to_bytes(16, "little", signed=False)
    except (ValueError, OverflowError):
        pass
    s = s[2:] if s.lower().startswith("0x") else s
    try:
        raw = bytes.fromhex(s)
    except ValueError as e:
        raise UsageError(f"seed must be an integer or hex string, got {text!r}") from e
    if not raw:
        raise UsageError("seed must not be empty")
    return raw


def load_config_file(path: str) -> Dict[str, str]:
    """Flat key = value file (cli.py:161-180)."""
    out: Dict[str, str] = {}
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise UsageError(f"cannot read config file {path}: {e}") from e
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, sep, value = line.partition("=")
        if not sep:
            raise UsageError(f"{path}:{lineno}: expected key = value")
        out[key.strip().replace("-", "_")] = value.strip()
    return out


_BOOL = {"true": True, "yes": True, "on": True, "1": True, "false": False, "no": False, "off": False, "0": False}
_COERCE = {"width": int, "tau": int, "depth": int, "max_depth": int, "lane_limit": int, "rows": str, "seed": str,
           "reveal": bool, "timeout": float, "split": float, "tolerance": float}


def apply_config(args: argparse.Namespace, cfg: Dict[str, str]) -> None:
    """Config supplies defaults; explicit flags win (cli.py:183-208)."""
    for key, value in cfg.items():
        if not hasattr(args, key):
            raise UsageError(f"config key {key!r} does not match any option")
        if getattr(args, key) is not None:
            continue
        kind = _COERCE.get(key, str)
        if kind is bool:
            if value.lower() not in _BOOL:
                raise UsageError(f"config key {key!r} needs a boolean, got {value!r}")
            setattr(args, key, _BOOL[value.lower()])
        else:
            try:
                setattr(args, key, kind(value))
            except (ValueError, UsageError) as e:
                raise UsageError(f"config key {key!r}: {e}") from e


def build_run_config(args: argparse.Namespace) -> RunConfig:
    rc = RunConfig()
    for name in ("width", "tau", "depth", "policy", "max_depth", "heuristic", "profile", "lane_limit", "timeout",
                 "count_reshare"):
        v = getattr(args, name, None)
        if v is not None:
            setattr(rc, name, v)
    if getattr(args, "seed", None) is not None:
        rc.seed = parse_seed(args.seed)
    if getattr(args, "reveal", None):
        rc.reveal = True
    rc.validate()
    return rc


def party_dir(base: Path, party: int) -> Path:
    return base / f"party{party}"


def _pairs_from_files(base: Path, name: str, shape) -> List:
    out = []
    for i in PARTIES:
        lo, hi, ring, _ = read_share_file(str(party_dir(base, i) / name))
        out.append((lo.reshape(shape), hi.reshape(shape)))
    return out


def _open(comp: np.ndarray) -> np.ndarray:
    return np.asarray(comp, dtype=np.uint64).sum(axis=0, dtype=np.uint64)


def _seeds_from_deal_dir(base: Path) -> SeedSetup:
    """assemble_seeds (cli.py:316-334)."""
    pair, local, filler = {}, {}, b""
    for i in PARTIES:
        doc = json.loads((party_dir(base, i) / "seeds.json").read_text())
        pair[i] = bytes.fromhex(doc["pair_next"])
        local[i] = bytes.fromhex(doc["local"])
        filler = bytes.fromhex(doc["filler"])
    enc = json.loads((base / "enclave.json").read_text())
    return SeedSetup(master=b"", pair_seeds=pair, local_seeds=local, enclave_seed=bytes.fromhex(enc["seed"]),
                     filler_seed=filler, enclave_channel_keys={i: bytes.fromhex(enc["keys"][str(i)]) for i in PARTIES})


def write_party_seeds(base: Path, setup: SeedSetup) -> None:
    """cli.py:281-299 (same files, same bytes)."""
    for i in PARTIES:
        prev = PARTIES[(i - 2) % 3]
        doc = {"party": i, "pair_next": setup.pair_seeds[i].hex(), "pair_prev": setup.pair_seeds[prev].hex(),
               "local": setup.local_seeds[i].hex(), "filler": setup.filler_seed.hex(),
               "enclave_key": setup.enclave_channel_keys[i].hex()}
        (party_dir(base, i) / "seeds.json").write_text(json.dumps(doc, indent=2, sort_keys=True))
    enc = {"seed": setup.enclave_seed.hex(), "keys": {str(i): setup.enclave_channel_keys[i].hex() for i in PARTIES}}
    (base / "enclave.json").write_text(json.dumps(enc, indent=2, sort_keys=True))


def write_shared(base: Path, name: str, values: np.ndarray, seed: bytes, label: str) -> None:
    pairs = share_values(values, 64, derive_seed(seed, label))
    for i in PARTIES:
        write_share_file(str(party_dir(base, i) / name), *pairs[i - 1], RING64, i)


def cmd_deal(args: argparse.Namespace) -> int:
    """cli.py:354-411.  Writes the same share, seed and meta files as the
    reference; no material.bin -- the B200 path derives its correlated
    randomness in-kernel from Philox keys (randomness)."""
    from .train import resolved_depth

    rc = build_run_config(args)
    if (args.data is None) == (args.queries is None):
        raise UsageError("deal needs exactly one of --data or --queries")
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    for i in PARTIES:
        party_dir(out, i).mkdir(exist_ok=True)
    write_party_seeds(out, SeedSetup.from_master(rc.seed))
    meta: Dict[str, object] = {"width": rc.width, "tau": rc.tau, "policy": rc.policy, "heuristic": rc.heuristic}
    if args.data is not None:
        data = tree_mod.load_csv(args.data)
        n, d = data.shape
        write_shared(out, "features.shr", data[:, :-1], rc.seed, "deal/features")
        write_shared(out, "labels.shr", data[:, -1], rc.seed, "deal/labels")
        meta.update({"kind": "train", "n_rows": n, "n_columns": d, "depth": resolved_depth(rc.train_config(), d)})
    else:
        queries = tree_mod.load_csv(args.queries, min_columns=1)
        if args.depth is None:
            raise UsageError("dealing queries needs --depth of the target tree")
        n, nf = queries.shape
        write_shared(out, "queries.shr", queries, rc.seed, "deal/queries")
        meta.update({"kind": "infer", "n_rows": n, "n_columns": nf + 1, "depth": rc.depth})
        if args.tree is not None:
            state = tree_mod.TreeState.from_json(Path(args.tree).read_text())
            state.validate(n_columns=nf + 1)
            if state.depth != rc.depth:
                raise UsageError("--depth does not match the tree file")
            write_shared(out, TREE_T_NAME, state.T, rc.seed, "deal/tree")
    (out / META_NAME).write_text(json.dumps(meta, indent=2, sort_keys=True))
    print(f"dealt {meta['kind']} shares for {meta['n_rows']} rows into {out}")
    return EXIT_OK


# ---------------------------------------------------------------------------
# train / infer / compare
# ---------------------------------------------------------------------------

def _train_device(setup: SeedSetup, dealer_seed: bytes, x_pairs, y_pairs, rc: RunConfig, n: int, d: int):
    from .train import train_components

    X = components_from_pairs(x_pairs, RING64).reshape(3, n, d - 1)
    Y = components_from_pairs(y_pairs, RING64).reshape(3, n)
    T, F, depth = train_components(X, Y, rc.train_config(), setup, dealer_seed)
    led = Ledger(rc.lane_limit)
    from .train import resolved_depth

    led.train(n, d - 1, resolved_depth(rc.train_config(), d), rc.tau, rc.width, grow_stop_level=depth - 1,
              policy=rc.policy, heuristic=rc.heuristic, count_reshare=rc.count_reshare)
    return T, F, depth, led.metrics()


def cmd_train(args: argparse.Namespace) -> int:
    """cli.py:419-483 (in-process)."""
    rc = build_run_config(args)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    if args.deal_dir is not None:
        base = Path(args.deal_dir)
        meta = json.loads((base / META_NAME).read_text())
        if meta.get("kind") != "train":
            raise UsageError(f"{base} was not dealt for training")
        n, d = int(meta["n_rows"]), int(meta["n_columns"])
        setup = _seeds_from_deal_dir(base)
        dealer_seed = derive_seed(setup.enclave_seed, "b200-dealer")
        x_pairs = _pairs_from_files(base, "features.shr", (n, d - 1))
        y_pairs = _pairs_from_files(base, "labels.shr", (n,))
    elif args.data is not None:
        data = tree_mod.load_csv(args.data)
        n, d = data.shape
        setup = SeedSetup.from_master(rc.seed)
        dealer_seed = derive_seed(rc.seed, "live-dealer")
        x_pairs = share_values(data[:, :-1], 64, derive_seed(rc.seed, "deal/features"))
        y_pairs = share_values(data[:, -1], 64, derive_seed(rc.seed, "deal/labels"))
    else:
        raise UsageError("train needs --data (live dealing) or --deal-dir")
    T, F, depth, metrics = _train_device(setup, dealer_seed, x_pairs, y_pairs, rc, n, d)
    tp, fp = pairs_from_components(T), pairs_from_components(F)
    for i in PARTIES:
        party_dir(out, i).mkdir(parents=True, exist_ok=True)
        write_share_file(str(party_dir(out, i) / TREE_T_NAME), *tp[i - 1], RING64, i)
        write_share_file(str(party_dir(out, i) / TREE_F_NAME), *fp[i - 1], RING64, i)
    (out / TREE_META_NAME).write_text(json.dumps({"depth": depth, "n_columns": d, "heuristic": rc.heuristic},
                                                 indent=2, sort_keys=True))
    (out / METRICS_NAME).write_text(metrics.to_json())
    if rc.reveal:
        state = tree_mod.TreeState(depth, _open(T), _open(F))
        state.validate(n_columns=d)
        (out / "tree.json").write_text(state.to_json())
    print(f"trained depth-{depth} tree shares into {out} ({metrics.total_bytes()} bytes, {metrics.rounds} rounds)")
    return EXIT_OK


def cmd_infer(args: argparse.Namespace) -> int:
    """cli.py:531-577 (in-process)."""
    from .infer import infer_components

    rc = build_run_config(args)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    if args.queries is None:
        raise UsageError("infer needs --queries")
    queries = tree_mod.load_csv(args.queries, min_columns=1)
    n, nf = queries.shape
    if args.tree_dir is not None:
        tdir = Path(args.tree_dir)
        meta = json.loads((tdir / TREE_META_NAME).read_text())
        depth, d = int(meta["depth"]), int(meta["n_columns"])
        if d != nf + 1:
            raise UsageError(f"tree expects {d - 1} features, queries have {nf}")
        t_pairs = _pairs_from_files(tdir, TREE_T_NAME, ((1 << depth) - 1,))
    elif args.tree is not None:
        state = tree_mod.TreeState.from_json(Path(args.tree).read_text())
        state.validate(n_columns=nf + 1)
        depth = state.depth
        t_pairs = share_values(state.T, 64, derive_seed(rc.seed, "deal/tree"))
    else:
        raise UsageError("infer needs --tree-dir (shares) or --tree (plaintext)")
    q_pairs = share_values(queries, 64, derive_seed(rc.seed, "deal/queries"))
    setup = SeedSetup.from_master(rc.seed)
    keys = make_keys(setup, derive_seed(rc.seed, "live-dealer"))
    tree = components_from_pairs(t_pairs, RING64)
    Q = components_from_pairs(q_pairs, RING64).reshape(3, n, nf)
    preds, _ = infer_components(tree, depth, Q, keys)
    led = Ledger(rc.lane_limit)
    led.infer(n, nf, depth)
    metrics = led.metrics()
    pp = pairs_from_components(preds)
    for i in PARTIES:
        party_dir(out, i).mkdir(exist_ok=True)
        write_share_file(str(party_dir(out, i) / "predictions.shr"), *pp[i - 1], RING64, i)
    (out / METRICS_NAME).write_text(metrics.to_json())
    if rc.reveal:
        tree_mod.save_csv(out / "predictions.csv", _open(preds).reshape(-1, 1))
    print(f"classified {n} queries into {out} ({metrics.total_bytes()} bytes, {metrics.rounds} rounds)")
    return EXIT_OK


def cmd_compare(args: argparse.Namespace) -> int:
    """cli.py:617-688."""
    if args.profile is None:
        args.profile = "test"
    rc = build_run_config(args)
    if rc.profile != "test":
        raise UsageError("compare reveals the trained tree and needs the test profile")
    from .train import resolved_depth

    data = tree_mod.load_csv(args.data)
    n, d = data.shape
    split = args.split if args.split is not None else (0.8 if rc.heuristic == "mpc" else 1.0)
    if not 0.0 < split <= 1.0:
        raise UsageError("--split must be in (0, 1]")
    tolerance = args.tolerance if args.tolerance is not None else 4.0
    rng = np.random.default_rng(int.from_bytes(derive_seed(rc.seed, "compare/split")[:8], "little"))
    order = rng.permutation(n)
    n_train = max(1, int(round(n * split)))
    train_rows = data[np.sort(order[:n_train])]
    test_rows = data[np.sort(order[n_train:])] if n_train < n else data
    oracle = tree_mod.plaintext_train(train_rows, resolved_depth(rc.train_config(), d), rc.seed)
    setup = SeedSetup.from_master(rc.seed)
    x_pairs = share_values(train_rows[:, :-1], 64, derive_seed(rc.seed, "deal/features"))
    y_pairs = share_values(train_rows[:, -1], 64, derive_seed(rc.seed, "deal/labels"))
    T, F, depth, metrics = _train_device(setup, derive_seed(rc.seed, "live-dealer"), x_pairs, y_pairs, rc,
                                         n_train, d)
    secure = tree_mod.TreeState(depth, _open(T), _open(F))
    secure.validate(n_columns=d)
    identical = bool(np.array_equal(secure.T, oracle.T) and np.array_equal(secure.F, oracle.F))

    def accuracy(state) -> float:
        return float(np.mean(tree_mod.plaintext_infer(state, test_rows[:, :-1]) == test_rows[:, -1]))

    acc_oracle, acc_secure = accuracy(oracle), accuracy(secure)
    delta_pp = abs(acc_oracle - acc_secure) * 100.0
    print(f"trees identical: {'true' if identical else 'false'}")
    print(f"oracle accuracy: {acc_oracle:.4f}")
    print(f"secure accuracy: {acc_secure:.4f}")
    print(f"accuracy delta: {delta_pp:.2f} pp (tolerance {tolerance:.2f})")
    if args.out is not None:
        Path(args.out).write_text(json.dumps({
            "identical": identical, "oracle_accuracy": acc_oracle, "secure_accuracy": acc_secure,
            "delta_pp": delta_pp, "heuristic": rc.heuristic, "depth": depth,
            "metrics": json.loads(metrics.to_json())}, indent=2, sort_keys=True))
    if rc.heuristic == "tee" and not identical:
        raise CompareMismatch("trusted-path tree differs from the plaintext oracle")
    if delta_pp > tolerance:
        raise CompareMismatch(f"accuracy delta {delta_pp:.2f} pp exceeds tolerance {tolerance:.2f}")
    return EXIT_OK


# ---------------------------------------------------------------------------
# bench: the reference's communication tables (cli.py:696-841) + device time
# ---------------------------------------------------------------------------

def bench_rows(suite: str, args: argparse.Namespace, rc: RunConfig, run: bool = True) -> List[Dict[str, object]]:
    rows: List[Dict[str, object]] = []
    if suite == "oaa":
        width = rc.width
        lookups = args.lookups if args.lookups is not None else 1000
        for m in [int(s) for s in (args.sizes or "1,8,64").split(",")]:
            led = Ledger(rc.lane_limit)
            with led.phase("oaa"):
                led.oaa(lookups, m, width)
            met = led.metrics()
            party_bits = max(met.sent_by_party(i) for i in PARTIES) * 8
            reference = (4 * width - 1) * m
            row = {"table_size": m, "lookups": lookups, "party_bits": party_bits,
                   "bits_per_lookup": party_bits / lookups, "reference_bits": reference,
                   "ratio": party_bits / lookups / reference, "rounds": met.rounds}
            if run:
                row["seconds"] = _time_oaa(width, m, lookups, rc)
            rows.append(row)
    elif suite == "train":
        from .train import TrainConfig, resolved_depth

        for n in [int(s) for s in (args.rows or "128,512").split(",")]:
            for d in [int(s) for s in (args.cols or "8").split(",")]:
                for h in [int(s) for s in (args.depths or "3,5").split(",")]:
                    for heu in ("tee", "mpc"):
                        cfg = TrainConfig(depth=h, heuristic=heu, tau=rc.tau, score_ring=Ring(rc.width))
                        led = Ledger(rc.lane_limit)
                        led.train(n, d - 1, resolved_depth(cfg, d), rc.tau, rc.width, heuristic=heu)
                        met = led.metrics()
                        row = {"rows": n, "columns": d, "depth": h, "heuristic": heu,
                               "total_bytes": met.total_bytes(), "rounds": met.rounds}
                        if run:
                            row["seconds"] = _time_train(n, d, cfg, rc)
                        rows.append(row)
    elif suite == "infer":
        d = (args.cols and int(args.cols.split(",")[0])) or 8
        for nq in [int(s) for s in (args.rows or "1000").split(",")]:
            for h in [int(s) for s in (args.depths or "4,8").split(",")]:
                led = Ledger(rc.lane_limit)
                led.infer(nq, d - 1, h)
                met = led.metrics()
                row = {"queries": nq, "depth": h, "columns": d, "total_bytes": met.total_bytes(),
                       "rounds": met.rounds}
                if run:
                    row["seconds"] = _time_infer(nq, h, d, rc)
                rows.append(row)
    else:
        raise UsageError(f"unknown bench suite {suite!r}")
    return rows


def _keys(rc: RunConfig, label: str):
    return make_keys(SeedSetup.from_master(derive_seed(rc.seed, label)), derive_seed(rc.seed, label + "/deal"))


def _time_oaa(width, m, lookups, rc) -> float:
    from . import gadgets as G
    from .shares import share_values as comp_share, to_device
    import torch

    rng = np.random.default_rng(1234 + m)
    ring = Ring(width)
    t = to_device(comp_share(rng.integers(0, 1 << min(width, 32), m, dtype=np.uint64), ring, rng))
    i = to_device(comp_share(rng.integers(0, m, lookups, dtype=np.uint64), ring, rng))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.oaa(width, t, i, keys=_keys(rc, f"bench/{m}"), op=0x80000000)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def _time_train(n, d, cfg, rc) -> float:
    from .train import train_components

    data = np.random.default_rng(n * 31 + d * 7 + cfg.depth).integers(0, 2, (n, d), dtype=np.uint8)
    setup = SeedSetup.from_master(derive_seed(rc.seed, f"bench/{n}/{d}/{cfg.depth}"))
    X = components_from_pairs(share_values(data[:, :-1], 64, derive_seed(rc.seed, "bx")), RING64).reshape(3, n, d - 1)
    Y = components_from_pairs(share_values(data[:, -1], 64, derive_seed(rc.seed, "by")), RING64).reshape(3, n)
    t0 = time.perf_counter()
    train_components(X, Y, cfg, setup, derive_seed(rc.seed, f"bench-deal/{n}/{d}/{cfg.depth}"))
    return time.perf_counter() - t0


def _time_infer(nq, h, d, rc) -> float:
    from .infer import infer_components

    rng = np.random.default_rng(nq + h)
    T = rng.integers(0, d - 1, (1 << h) - 1).astype(np.uint64)
    q = rng.integers(0, 2, (nq, d - 1), dtype=np.uint8)
    tree = components_from_pairs(share_values(T, 64, derive_seed(rc.seed, "bt")), RING64)
    Q = components_from_pairs(share_values(q, 64, derive_seed(rc.seed, "bq")), RING64).reshape(3, nq, d - 1)
    t0 = time.perf_counter()
    infer_components(tree, h, Q, _keys(rc, f"bi/{nq}/{h}"))
    return time.perf_counter() - t0


def cmd_bench(args: argparse.Namespace) -> int:
    rc = build_run_config(args)
    rows = bench_rows(args.suite, args, rc, run=True)
    if rows:
        cols = list(rows[0].keys())
        fmt = lambda v: f"{v:.3f}" if isinstance(v, float) else str(v)  # noqa: E731
        widths = {c: max(len(c), *(len(fmt(r[c])) for r in rows)) for c in cols}
        print("  ".join(c.rjust(widths[c]) for c in cols))
        for r in rows:
            print("  ".join(fmt(r[c]).rjust(widths[c]) for c in cols))
    if args.out is not None:
        clean = [{k: v for k, v in r.items() if k != "seconds"} for r in rows]
        Path(args.out).write_text(json.dumps(clean, indent=2, sort_keys=True))
    return EXIT_OK


# ---------------------------------------------------------------------------
# parser
# ---------------------------------------------------------------------------

def _run_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--config", help="key = value file supplying flag defaults")
    p.add_argument("--width", type=int, help="score ring bit width (default 32)")
    p.add_argument("--tau", type=int, help="fixed-point fractional bits (default 10)")
    p.add_argument("--depth", type=int, help="tree depth H (default 4)")
    p.add_argument("--policy", choices=("fixed", "grow", "feature_cap"), help="depth policy (default fixed)")
    p.add_argument("--max-depth", type=int, dest="max_depth", help="cap for the grow policy")
    p.add_argument("--heuristic", choices=("mpc", "tee"), help="split scoring path (default mpc)")
    p.add_argument("--seed", help="master seed: integer or hex string (default 0)")
    p.add_argument("--lane-limit", type=int, dest="lane_limit", help="reference batch ceiling (ledger chunking)")
    p.add_argument("--timeout", type=float, help="accepted for compatibility")
    p.add_argument("--profile", choices=("prod", "test"), help="prod (default) or test")
    p.add_argument("--reveal", action="store_true", default=None, help="write plaintext outputs (test profile)")
    p.add_argument("--count-reshare", dest="count_reshare", choices=("elementwise", "dot"),
                   help="B200 option: per-product (default, as the reference) or dot-product reshare")


def build_parser() -> argparse.ArgumentParser:
    top = argparse.ArgumentParser(prog="gtree-b200", description="Three-party decision trees on B200.")
    sub = top.add_subparsers(dest="command", required=True)
    p = sub.add_parser("deal", help="split a dataset into shares (no material file: randomness is in-kernel)")
    _run_flags(p)
    p.add_argument("--data", help="binary CSV with the label in the last column")
    p.add_argument("--queries", help="binary CSV of feature rows (inference dealing)")
    p.add_argument("--tree", help="plaintext tree JSON to share alongside queries")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_deal)
    p = sub.add_parser("train", help="train a tree on shared data")
    _run_flags(p)
    p.add_argument("--data", help="binary CSV (in-process live dealing)")
    p.add_argument("--deal-dir", dest="deal_dir", help="directory produced by obtree deal")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_train)
    p = sub.add_parser("infer", help="classify shared queries with a shared tree")
    _run_flags(p)
    p.add_argument("--queries", help="binary CSV of feature rows")
    p.add_argument("--tree-dir", dest="tree_dir", help="directory produced by train")
    p.add_argument("--tree", help="plaintext tree JSON")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_infer)
    p = sub.add_parser("compare", help="train both oracle and secure paths and compare")
    _run_flags(p)
    p.add_argument("--data", required=True)
    p.add_argument("--split", type=float)
    p.add_argument("--tolerance", type=float)
    p.add_argument("--out")
    p.set_defaults(func=cmd_compare)
    p = sub.add_parser("bench", help="communication tables + device time over a parameter grid")
    _run_flags(p)
    p.add_argument("--suite", choices=("oaa", "train", "infer"), default="oaa")
    p.add_argument("--lookups", type=int)
    p.add_argument("--sizes")
    p.add_argument("--rows")
    p.add_argument("--cols")
    p.add_argument("--depths")
    p.add_argument("--out")
    p.set_defaults(func=cmd_bench)
    return top


def main(argv: Optional[Sequence[str]] = None) -> int:
    """cli.py:1040-1064: exit 1 usage/data, 2 protocol, 3 mismatch."""
    logging.basicConfig(level=getattr(logging, os.environ.get("OBTREE_LOG", "WARNING").upper(), logging.WARNING))
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code in (0, None) else EXIT_USAGE
    try:
        if getattr(args, "config", None):
            apply_config(args, load_config_file(args.config))
        return args.func(args)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except (tree_mod.DataError, tree_mod.TreeError, RingError, FileNotFoundError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except (TransportError, ShareError, EnclaveError, ProtocolError) as e:
        print(f"protocol failure: {e}", file=sys.stderr)
        return EXIT_PROTOCOL
    except CompareMismatch as e:
        print(f"verification mismatch: {e}", file=sys.stderr)
        return EXIT_MISMATCH


if __name__ == "__main__":
    sys.exit(main())
