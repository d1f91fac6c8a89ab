"""Correlated-material banks and deal directories, loaded straight to the device.

SURVEY.md 8(f)3: the step before the hot path (dealt inputs) and after it
(tree shares).  Three pieces, each readable by the reference and by this
package:

* Material needs (reference train.py:309-346, infer.py:38-43, gadgets.py
  needs_*): how many edabits / dabits / truncation pairs a training or
  inference run consumes, restated as per-gadget tallies.
* OBD1 material banks (dealer.py:87-193): per party, sections of
  (kind, width, k, count) with the banked arrays, and the reference dealer's
  deterministic generation (AES-128-CTR per material key), byte for byte.
* Deal directories (cli.py:260-400: partyN/{seeds.json, features.shr,
  labels.shr, queries.shr, tree_T.shr, material.bin}, meta.json,
  enclave.json): the three parties' OBS1 share files are read into ONE pinned
  host buffer and copied to the device once; ``gt_unpack_pairs`` widens the
  little-endian ring words into the component-major ``[3, ...]`` layout and
  counts replication mismatches on the device (no numpy staging).

The device hot path draws its material in-kernel (Philox, DESIGN.md section
4), so banks loaded here are for dealer-provisioned deployments and for
checking a deal; revealed outputs never depend on them.
"""

from __future__ import annotations

import ctypes
import json
import os
import struct
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .seeds import PARTIES, SeedSetup, derive_seed
from .shares import RING64, Ring, ShareError

MaterialKey = tuple  # ("edabit", w) | ("dabit", w) | ("trunc", w, k)


class MaterialError(RuntimeError):
    """A bank ran out of a material kind (gadgets.py MaterialError)."""

# ---------------------------------------------------------------------------
# material needs
# ---------------------------------------------------------------------------


class Needs(dict):
    """key -> element count (gadgets.py:55-72 semantics)."""

    def add(self, key: MaterialKey, n: int) -> "Needs":
        if n:
            self[key] = self.get(key, 0) + int(n)
        return self


def _eq(nd: Needs, n: int, w: int) -> None:  # one edabit per eq lane
    nd.add(("edabit", w), n)


def _lt(nd: Needs, n: int, w: int) -> None:  # both operands masked
    nd.add(("edabit", w), 2 * n)


def _b2a(nd: Needs, n: int, w: int) -> None:  # one dabit per bit
    nd.add(("dabit", w), n)


def _trunc(nd: Needs, n: int, w: int, k: int) -> None:  # pair + wrap / low-borrow dabits
    if k:
        nd.add(("trunc", w, k), n)
        nd.add(("dabit", w), 2 * n)


def _division(nd: Needs, n: int, w: int, tau: int) -> None:
    from .ledger import div_params

    d = div_params(w, tau)
    ladder = d["bound"] - 1
    _lt(nd, ladder * n, w)
    _b2a(nd, ladder * n, w)
    _trunc(nd, n, w, d["bound"] - d["ti"])
    _trunc(nd, 2 * d["iters"] * n, w, d["ti"])
    _trunc(nd, n, w, d["sigma"])
    _trunc(nd, n, w, d["kf"])


def _argmin(nd: Needs, rows: int, m: int, sw: int, iw: int) -> None:
    _b2a(nd, rows * m, sw)  # masking selects
    while m > 1:
        pairs = m // 2
        _lt(nd, rows * pairs, sw)
        _b2a(nd, rows * pairs, sw)
        _b2a(nd, rows * pairs, iw)
        m = pairs + (m & 1)


def _oaa(nd: Needs, lookups: int, m: int, w: int) -> None:  # eq + select per entry
    _eq(nd, lookups * m, w)
    _b2a(nd, lookups * m, w)


def training_needs(n_samples: int, n_columns: int, cfg) -> Needs:
    """Material a training run consumes (train.py:309-346)."""
    from .train import as_config, counter_shift, resolved_depth

    cfg = as_config(cfg)
    nf = n_columns - 1
    depth = resolved_depth(cfg, n_columns)
    w, sw = cfg.count_ring.width, cfg.score_ring.width
    nd = Needs()
    for level in range(depth):
        nodes, cols, last = 1 << level, 2 * nf, level == depth - 1
        if level:
            _oaa(nd, n_samples, 1 << (level - 1), w)  # partition: level payloads
            _oaa(nd, n_samples, nf, w)  # row fetch
        _eq(nd, nodes, w)  # is_leaf
        _eq(nd, n_samples * nodes, w)  # count lanes
        _b2a(nd, n_samples * nodes, w)
        if not last and cfg.heuristic == "mpc":
            _eq(nd, 3 * nodes, w)  # probe / featureless / should-split
            _b2a(nd, nodes, w)  # new type
            _trunc(nd, nodes * 3 * cols, w, counter_shift(n_samples, cfg))
            _eq(nd, nodes * cols, sw)  # Q == 0
            _b2a(nd, nodes * cols, sw)
            _division(nd, nodes * cols, sw, cfg.tau)
            _argmin(nd, nodes, nf, sw, w)
            _eq(nd, nodes * nf, w)  # budget clear
        if level:
            _eq(nd, nodes, w)  # empty node
            _b2a(nd, nodes, w)  # inherit counters
        if not last:
            _b2a(nd, 3 * nodes, w)  # split: payload, child type, child counters
        elif cfg.heuristic == "mpc":
            _lt(nd, nodes, w)  # labels
            _b2a(nd, nodes, w)
    return nd


def inference_needs(n_queries: int, depth: int, n_columns: int, width: int = 64) -> Needs:
    """Material an inference batch consumes (infer.py:38-43)."""
    nd = Needs()
    for t in range(depth):
        _oaa(nd, n_queries, 1 << t, width)
        _oaa(nd, n_queries, n_columns - 1, width)
    return nd


# ---------------------------------------------------------------------------
# OBD1 banks and the reference dealer's generation
# ---------------------------------------------------------------------------

MATERIAL_MAGIC = b"OBD1"
_KINDS = ("edabit", "dabit", "trunc")
_SECTION = struct.Struct("<BBBxQ")  # kind code, width, k, pad, count
# per kind: the bank's arrays, "w" = ring words, "b" = one byte per bit
_FIELDS = {"edabit": "wwww", "dabit": "wwbb", "trunc": "wwwwww"}


def _word_bytes(width: int) -> int:
    return 8 if width == 64 else 4 if width == 32 else 1


def _pack(a: np.ndarray, width: int) -> bytes:
    return np.ascontiguousarray(a, dtype=np.uint64).astype({8: "<u8", 4: "<u4", 1: "u1"}[_word_bytes(width)]).tobytes()


class _Aes:
    """The reference dealer's AES-128-CTR keystream (transport.py:63-94)."""

    def __init__(self, seed: bytes):
        from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes

        self._enc = Cipher(algorithms.AES(seed), modes.CTR(b"\x00" * 16)).encryptor()

    def words(self, count: int, width: int) -> np.ndarray:
        wb = width // 8
        raw = self._enc.update(b"\x00" * (count * wb))
        return np.frombuffer(raw, dtype={8: "<u8", 4: "<u4", 1: "u1"}[wb]).astype(np.uint64)

    def bits(self, count: int) -> np.ndarray:
        raw = self._enc.update(b"\x00" * ((count + 7) // 8))
        return np.unpackbits(np.frombuffer(raw, dtype=np.uint8))[:count]


def _replicate(v, s1, s2, minus, mask):
    """Three replicated pairs (s_i, s_{i+1}) of v: s3 = v - s1 - s2 (or xor)."""
    s3 = ((v - s1 - s2) & mask) if minus else (v ^ s1 ^ s2)
    return [(s1, s2), (s2, s3), (s3, s1)]


def _generate_key(key: MaterialKey, count: int, prg: _Aes) -> List[Tuple[np.ndarray, ...]]:
    """One key's banks for the three parties (dealer.py:43-84)."""
    kind, w = key[0], key[1]
    mask = np.uint64((1 << w) - 1) if w < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)

    def arith(v):
        s1, s2 = prg.words(count, w) & mask, prg.words(count, w) & mask
        return _replicate(v & mask, s1, s2, True, mask)

    def planes(v):
        t1, t2 = prg.words(count, w), prg.words(count, w)
        return _replicate(v, t1, t2, False, mask)

    if kind == "dabit":
        b = prg.bits(count)
        a = arith(b.astype(np.uint64))
        u1, u2 = prg.bits(count).astype(np.uint8), prg.bits(count).astype(np.uint8)
        bb = _replicate(b.astype(np.uint8) & 1, u1, u2, False, None)
        return [a[i] + bb[i] for i in range(3)]
    r = prg.words(count, w)
    parts = [arith(r), planes(r)]
    if kind == "trunc":
        parts.append(arith(r >> np.uint64(key[2])))
    return [tuple(x for part in parts for x in part[i]) for i in range(3)]


@dataclass
class MaterialBank:
    """One party's banked material: key -> arrays (dealer.py:87-185)."""

    sections: Dict[MaterialKey, Tuple[np.ndarray, ...]]

    @staticmethod
    def _order(keys):
        return sorted(keys, key=repr)

    def to_bytes(self) -> bytes:
        out = [MATERIAL_MAGIC, struct.pack("<I", len(self.sections))]
        for key in self._order(self.sections):
            arrays = self.sections[key]
            out.append(_SECTION.pack(_KINDS.index(key[0]), key[1], key[2] if key[0] == "trunc" else 0,
                                     int(arrays[0].shape[0])))
            for spec, a in zip(_FIELDS[key[0]], arrays):
                out.append(_pack(a, key[1]) if spec == "w" else np.ascontiguousarray(a, dtype=np.uint8).tobytes())
        return b"".join(out)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "MaterialBank":
        if raw[:4] != MATERIAL_MAGIC:
            raise ValueError("not a material file")
        (nsec,) = struct.unpack_from("<I", raw, 4)
        at, sections = 8, {}
        for _ in range(nsec):
            code, w, k, count = _SECTION.unpack_from(raw, at)
            at += _SECTION.size
            kind = _KINDS[code]
            arrays = []
            for spec in _FIELDS[kind]:
                nb = count * (_word_bytes(w) if spec == "w" else 1)
                dt = {8: "<u8", 4: "<u4", 1: "u1"}[_word_bytes(w)] if spec == "w" else np.uint8
                a = np.frombuffer(raw, dtype=dt, count=count, offset=at)
                arrays.append(a.astype(np.uint64) if spec == "w" else a.copy())
                at += nb
            key = (kind, w, k) if kind == "trunc" else (kind, w)
            if key in sections:  # a repeated key appends (MaterialStore.add_bank)
                arrays = [np.concatenate([o, n]) for o, n in zip(sections[key], arrays)]
            sections[key] = tuple(arrays)
        return cls(sections)

    def to_file(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.to_bytes())

    @classmethod
    def from_file(cls, path) -> "MaterialBank":
        with open(path, "rb") as fh:
            return cls.from_bytes(fh.read())


def generate_material(needs: Dict[MaterialKey, int], seed: bytes) -> List[MaterialBank]:
    """The three parties' banks, deterministically from `seed`
    (dealer.py:178-190: one AES stream per key, derive_seed(seed,
    "material/<repr(key)>"))."""
    banks = [MaterialBank({}) for _ in PARTIES]
    for key in MaterialBank._order(needs):
        count = int(needs[key])
        if count <= 0:
            continue
        per_party = _generate_key(tuple(key), count, _Aes(derive_seed(seed, f"material/{tuple(key)!r}")))
        for bank, arrays in zip(banks, per_party):
            bank.sections[tuple(key)] = arrays
    return banks


# ---------------------------------------------------------------------------
# device loading (one pinned read per file set, one H2D copy, gt_unpack_pairs)
# ---------------------------------------------------------------------------

_SHARE_HEADER = struct.Struct("<4sBBBxQ")  # OBS1: magic, width, kind, party, count (rss.py:452-481)


def _lib():
    from . import _native

    return _native.load()


def _unpack_device(raw_dev, lo_offs: Sequence[int], hi_offs: Sequence[int], stride: int, wbytes: int, n: int,
                   out, check: bool, stream) -> int:
    """gt_unpack_pairs on a device byte buffer: component i = the words at
    raw + lo_offs[i] (stride bytes apart), checked against the next party's hi."""
    import torch

    from . import _native

    base = raw_dev.data_ptr()
    arr = ctypes.c_void_p * 3
    bad = torch.zeros(1, dtype=torch.int64, device=out.device) if check else None
    _native.check(_lib().gt_unpack_pairs(arr(*[base + o for o in lo_offs]), arr(*[base + o for o in hi_offs]),
                                         stride, wbytes, n, out.data_ptr(), bad.data_ptr() if check else None,
                                         ctypes.c_void_p(stream.cuda_stream)))
    return int(bad.item()) if check else 0


def load_share_files(paths: Sequence[str], shape: Tuple[int, ...], device=None, check: bool = True):
    """The three parties' OBS1 files of one vector -> component-major device
    tensor [3, *shape] (int64 holding the ring words), read into one pinned
    buffer, copied once, unpacked on the device.  ShareError on a bad header,
    a shape mismatch or a replication inconsistency."""
    from . import _native

    torch = _native.require_cuda()
    if len(paths) != 3:
        raise ShareError("need the share files of exactly three parties")
    heads = []
    for p in paths:
        with open(p, "rb") as fh:
            magic, width, kind, party, count = _SHARE_HEADER.unpack(fh.read(_SHARE_HEADER.size))
        if magic != b"OBS1":
            raise ShareError(f"{p}: not a share file")
        heads.append((width, kind, party, count))
    widths = {h[0] for h in heads}
    counts = {h[3] for h in heads}
    if len(widths) != 1 or len(counts) != 1:
        raise ShareError("party share files disagree on ring or length")
    width, n = widths.pop(), counts.pop()
    if int(np.prod(shape, dtype=np.int64)) != n:
        raise ShareError(f"share files hold {n} elements, expected shape {tuple(shape)}")
    if sorted(h[2] for h in heads) != [1, 2, 3]:
        raise ShareError("share files must be those of parties 1, 2, 3")
    wb = _word_bytes(width)
    nbytes = 2 * n * wb
    pinned = torch.empty(3 * nbytes, dtype=torch.uint8).pin_memory()
    host = pinned.numpy()
    for p, (_, _, party, _) in zip(paths, heads):
        with open(p, "rb") as fh:
            fh.seek(_SHARE_HEADER.size)
            if fh.readinto(memoryview(host[(party - 1) * nbytes:party * nbytes])) != nbytes:
                raise ShareError(f"{p}: truncated share file")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    raw = pinned.to(dev, non_blocking=True)
    out = torch.empty((3,) + tuple(shape), dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev)
    # interleaved (lo, hi) words: party p's lo at p*nbytes, its hi one word later
    bad = _unpack_device(raw, [i * nbytes for i in range(3)], [i * nbytes + wb for i in range(3)], 2 * wb, wb, n,
                         out, check, s)
    if bad:
        raise ShareError(f"replication inconsistency between party pairs ({bad} words)")
    return out


def material_to_device(banks: Sequence[MaterialBank], device=None, check: bool = True):
    """The three parties' banks -> {key: tuple of component-major device
    tensors [3, count], one per field pair} (edabit: r, bits; dabit: a, bit;
    trunc: r, bits, r >> k): one pinned buffer, one copy, gt_unpack_pairs."""
    from . import _native

    torch = _native.require_cuda()
    if len(banks) != 3:
        raise ValueError("need the banks of exactly three parties")
    keys = MaterialBank._order(banks[0].sections)
    if any(MaterialBank._order(b.sections) != keys for b in banks):
        raise ValueError("party banks disagree on their material keys")
    layout, chunks, at = [], [], 0
    for key in keys:
        specs = _FIELDS[key[0]]
        for f in range(0, len(specs), 2):
            wb = _word_bytes(key[1]) if specs[f] == "w" else 1
            offs = []
            for b in banks:
                lo, hi = b.sections[key][f], b.sections[key][f + 1]
                for a in (lo, hi):
                    data = _pack(a, key[1]) if specs[f] == "w" else np.ascontiguousarray(a, np.uint8).tobytes()
                    chunks.append(data)
                    offs.append(at)
                    at += len(data)
            layout.append((key, f // 2, wb, int(banks[0].sections[key][f].shape[0]), offs))
    pinned = torch.empty(max(at, 1), dtype=torch.uint8).pin_memory()
    host, pos = pinned.numpy(), 0
    for c in chunks:
        host[pos:pos + len(c)] = np.frombuffer(c, dtype=np.uint8)
        pos += len(c)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    raw = pinned.to(dev, non_blocking=True)
    s = torch.cuda.current_stream(dev)
    out: Dict[MaterialKey, list] = {}
    for key, _, wb, count, offs in layout:
        t = torch.empty((3, count), dtype=torch.int64, device=dev)
        if count:
            bad = _unpack_device(raw, offs[0::2], offs[1::2], wb, wb, count, t, check, s)
            if bad:
                raise ShareError(f"material {key}: replication inconsistency ({bad} words)")
        out.setdefault(key, []).append(t)
    return {k: tuple(v) for k, v in out.items()}


@dataclass
class DealDir:
    """A dealt run's inputs, device-resident (cli.py:260-400 layout)."""

    meta: dict
    seeds: SeedSetup
    X: object = None  # [3, N, nf] features (train)
    Y: object = None  # [3, N] labels (train)
    Q: object = None  # [3, N, nf] queries (infer)
    T: object = None  # [3, 2^H - 1] tree payloads (infer, when dealt)
    material: Optional[List[str]] = None  # the parties' material.bin paths, if present


def _assemble_seeds(base: str) -> SeedSetup:
    """cli.py:316-337: the full seed setup from the three party files."""
    pair, local, filler = {}, {}, b""
    for i in PARTIES:
        with open(os.path.join(base, f"party{i}", "seeds.json")) as fh:
            doc = json.load(fh)
        pair[i], local[i] = bytes.fromhex(doc["pair_next"]), bytes.fromhex(doc["local"])
        filler = bytes.fromhex(doc["filler"])
    with open(os.path.join(base, "enclave.json")) as fh:
        enc = json.load(fh)
    return SeedSetup(master=b"", pair_seeds=pair, local_seeds=local, enclave_seed=bytes.fromhex(enc["seed"]),
                     filler_seed=filler, enclave_channel_keys={i: bytes.fromhex(enc["keys"][str(i)]) for i in PARTIES})


def load_deal_dir(base: str, device=None, check: bool = True) -> DealDir:
    """A reference deal directory straight onto the device."""
    with open(os.path.join(base, "meta.json")) as fh:
        meta = json.load(fh)
    dd = DealDir(meta=meta, seeds=_assemble_seeds(base))
    files = lambda name: [os.path.join(base, f"party{i}", name) for i in PARTIES]  # noqa: E731
    n, ncol = int(meta["n_rows"]), int(meta["n_columns"])
    if meta["kind"] == "train":
        dd.X = load_share_files(files("features.shr"), (n, ncol - 1), device, check)
        dd.Y = load_share_files(files("labels.shr"), (n,), device, check)
    else:
        dd.Q = load_share_files(files("queries.shr"), (n, ncol - 1), device, check)
        if all(os.path.exists(p) for p in files("tree_T.shr")):
            dd.T = load_share_files(files("tree_T.shr"), ((1 << int(meta["depth"])) - 1,), device, check)
    if all(os.path.exists(p) for p in files("material.bin")):
        dd.material = files("material.bin")
    return dd


def train_deal_dir(base: str, cfg=None, device=None):
    """Secure training from a deal directory, inputs loaded straight to the
    device.  The device draws its own correlated randomness (Philox keyed
    from the directory's seeds; the dealt material banks are not consumed),
    so the revealed tree equals the reference's for the same directory.
    Returns (trainer, depth): shares on trainer.T / trainer.F."""
    from .seeds import filler_values, make_keys
    from .shares import to_device
    from .train import DeviceTrainer, TrainConfig

    dd = load_deal_dir(base, device)
    if dd.meta["kind"] != "train":
        raise ValueError("not a training deal directory")
    m = dd.meta
    if cfg is None:
        cfg = TrainConfig(depth=int(m["depth"]), tau=int(m.get("tau", 10)), heuristic=m.get("heuristic", "mpc"),
                          policy=m.get("policy", "fixed"))
    n, nf = dd.X.shape[1], dd.X.shape[2]
    tr = DeviceTrainer(n, nf, cfg, device=dd.X.device)
    fill = filler_values(dd.seeds.filler_seed, (1 << tr.depth) - 1, nf + 1)
    keys = make_keys(dd.seeds, derive_seed(dd.seeds.enclave_seed, "b200/dealer"))
    depth = tr.run(dd.X, dd.Y, to_device(fill, tr.device), keys, enclave_seed=dd.seeds.enclave_seed)
    return tr, depth
