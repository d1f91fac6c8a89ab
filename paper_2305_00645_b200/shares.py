"""Share containers at the drop-in boundary and their device layout.

The reference hands every party an ``AVec(ring, lo, hi)`` (rss.py:53-132) with
party p holding components (s_p, s_{p+1}) of x = s_1 + s_2 + s_3 mod 2^l.
On the device all three parties are co-resident, so a share is one
component-major uint64 tensor ``[3, ...]`` with component i = party (i+1)'s
``lo``; replication consistency then holds by construction.  This module
converts between the two views and checks consistency on the way in exactly
like ``reconstruct_pairs`` (rss.py:222-228).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np


class ShareError(ValueError):
    """rss.py:44-45."""


class RingError(ValueError):
    """ring.py:22-23."""


@dataclass(frozen=True)
class Ring:
    """Z_{2^width}, width in {8, 32, 64} (ring.py:27-94)."""

    width: int

    def __post_init__(self) -> None:
        if self.width not in (8, 32, 64):
            raise RingError(f"unsupported ring width {self.width}; expected one of (8, 32, 64)")

    @property
    def mask(self) -> int:
        return (1 << self.width) - 1

    @property
    def modulus(self) -> int:
        return 1 << self.width

    @property
    def nbytes(self) -> int:
        return self.width // 8

    def reduce(self, x):
        if isinstance(x, np.ndarray):
            return x.astype(np.uint64, copy=False) & np.uint64(self.mask)
        return int(x) & self.mask


RING8, RING32, RING64 = Ring(8), Ring(32), Ring(64)


@dataclass
class AVec:
    """One party's arithmetic share pair (rss.py:53-63)."""

    ring: Ring
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self) -> None:
        if self.lo.shape != self.hi.shape:
            raise ShareError("share components disagree on shape")

    @property
    def shape(self) -> tuple:
        return self.lo.shape

    @property
    def size(self) -> int:
        return self.lo.size

    def reshape(self, *shape) -> "AVec":
        return AVec(self.ring, self.lo.reshape(*shape), self.hi.reshape(*shape))

    def ravel(self) -> "AVec":
        return AVec(self.ring, self.lo.ravel(), self.hi.ravel())

    def take(self, idx) -> "AVec":
        return AVec(self.ring, self.lo[idx], self.hi[idx])


@dataclass
class BitVec:
    """One party's XOR-shared bits, uint8 {0,1} (rss.py:151-160)."""

    lo: np.ndarray
    hi: np.ndarray

    @property
    def shape(self) -> tuple:
        return self.lo.shape


def ring_of(vec) -> Ring:
    r = getattr(vec, "ring", None)
    return Ring(int(r.width)) if r is not None else RING64


def components_from_pairs(pairs: Sequence[Tuple[np.ndarray, np.ndarray]], ring: Ring = RING64,
                          check: bool = True) -> np.ndarray:
    """Three parties' (lo, hi) pairs -> component-major [3, ...] uint64."""
    if len(pairs) != 3:
        raise ShareError("need the share pairs of exactly three parties")
    los = [np.asarray(p[0], dtype=np.uint64) for p in pairs]
    his = [np.asarray(p[1], dtype=np.uint64) for p in pairs]
    shape = los[0].shape
    if any(x.shape != shape for x in los + his):
        raise ShareError("share components disagree on shape")
    if check:
        for i in range(3):
            if not np.array_equal(his[i], los[(i + 1) % 3]):
                raise ShareError("replication inconsistency between party pairs")
    return np.stack([ring.reduce(x) for x in los])


def stage_pairs(pairs: Sequence[Tuple[np.ndarray, np.ndarray]], out: Optional[np.ndarray], check: bool = True,
                shape: Optional[Tuple[int, ...]] = None) -> None:
    """components_from_pairs written straight into `out` [3, ...] uint64 (the
    pinned staging buffer of a host-operand device call): party i's lo is
    component i; the replication check compares party i's hi with party
    i+1's lo without temporaries beyond one reusable bool buffer.  out=None
    runs the check alone (on `shape`)."""
    if len(pairs) != 3:
        raise ShareError("need the share pairs of exactly three parties")
    los = [np.asarray(p[0], dtype=np.uint64) for p in pairs]
    his = [np.asarray(p[1], dtype=np.uint64) for p in pairs]
    shape = out.shape[1:] if out is not None else tuple(shape if shape is not None else los[0].shape)
    if any(x.shape != shape for x in los + his):
        raise ShareError("share components disagree on shape")
    if out is None and not check:
        return
    if all(x.flags.c_contiguous for x in los + his) and (out is None or out.flags.c_contiguous):
        import ctypes

        from . import _native

        lib = _native.load()
        arr = ctypes.c_void_p * 3
        rc = lib.gt_stage_pairs(arr(*[x.ctypes.data for x in los]), arr(*[x.ctypes.data for x in his]),
                                int(np.prod(shape, dtype=np.int64)), None if out is None else out.ctypes.data,
                                1 if check else 0)
        if rc:
            raise ShareError(lib.gt_last_error().decode())
        return
    eq = np.empty(shape, dtype=bool) if check else None
    for i in range(3):
        if check:
            np.equal(his[i], los[(i + 1) % 3], out=eq)
            if not eq.all():
                raise ShareError("replication inconsistency between party pairs")
        if out is not None:
            np.copyto(out[i], los[i])


def components_from_avecs(vecs: Sequence, check: bool = True) -> np.ndarray:
    ring = ring_of(vecs[0])
    return components_from_pairs([(v.lo, v.hi) for v in vecs], ring, check)


def pairs_from_components(comp: np.ndarray) -> List[Tuple[np.ndarray, np.ndarray]]:
    comp = np.asarray(comp, dtype=np.uint64)
    return [(comp[i].copy(), comp[(i + 1) % 3].copy()) for i in range(3)]


def avecs_from_components(comp: np.ndarray, ring: Ring = RING64) -> List[AVec]:
    return [AVec(ring, lo, hi) for lo, hi in pairs_from_components(comp)]


def reconstruct(comp: np.ndarray, ring: Ring = RING64) -> np.ndarray:
    c = np.asarray(comp, dtype=np.uint64)
    return (c[0] + c[1] + c[2]) & np.uint64(ring.mask)


def share_values(values: np.ndarray, ring: Ring, rng: np.random.Generator) -> np.ndarray:
    """Fresh component-major sharing of public values (test/bench plumbing;
    the dealer-side split of make_arith_shares, rss.py:205-211)."""
    v = ring.reduce(np.asarray(values, dtype=np.uint64))
    s1 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) ^ (rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) << np.uint64(1))
    s2 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) ^ (rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) << np.uint64(1))
    s1, s2 = ring.reduce(s1), ring.reduce(s2)
    s3 = ring.reduce(v - s1 - s2)
    return np.stack([s1, s2, s3])


# --------------------------------------------------------------------------
# device tensors (torch is plumbing: allocation, copies, streams)
# --------------------------------------------------------------------------


def to_device(arr: np.ndarray, device="cuda"):
    import torch

    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return torch.from_numpy(a.view(np.int64)).to(device)


def from_device(t) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def ptr(t) -> int:
    if t is None:
        return 0
    if not t.is_contiguous():
        raise ValueError("device share tensors must be contiguous")
    return t.data_ptr()


# --------------------------------------------------------------------------
# on-disk share files (OBS1, reference rss.py:452-481)
# --------------------------------------------------------------------------

import struct as _struct

SHARE_MAGIC = b"OBS1"
_SHARE_HEADER = _struct.Struct("<4sBBBxQ")  # magic, width, kind, party, count


def _pack(arr: np.ndarray, ring: Ring) -> bytes:
    flat = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64).ravel())
    if ring.width == 64:
        return flat.astype("<u8").tobytes()
    if ring.width == 32:
        return flat.astype("<u4").tobytes()
    return flat.astype(np.uint8).tobytes()


def _unpack(raw: bytes, ring: Ring, n: int) -> np.ndarray:
    dt = {64: "<u8", 32: "<u4", 8: np.uint8}[ring.width]
    return np.frombuffer(raw, dtype=dt, count=n).astype(np.uint64)


def write_share_file(path: str, lo: np.ndarray, hi: np.ndarray, ring: Ring, party: int, kind: int = 0) -> None:
    """One party's share pair, interleaved little-endian (rss.py:460-469)."""
    lo = np.asarray(lo, dtype=np.uint64).ravel()
    hi = np.asarray(hi, dtype=np.uint64).ravel()
    inter = np.empty(lo.size * 2, dtype=np.uint64)
    inter[0::2], inter[1::2] = lo, hi
    with open(path, "wb") as f:
        f.write(_SHARE_HEADER.pack(SHARE_MAGIC, ring.width, kind, party, lo.size))
        f.write(_pack(inter, ring))


def read_share_file(path: str):
    """-> (lo, hi, ring, party) (rss.py:472-481)."""
    with open(path, "rb") as f:
        head = f.read(_SHARE_HEADER.size)
        magic, width, kind, party, count = _SHARE_HEADER.unpack(head)
        if magic != SHARE_MAGIC:
            raise ShareError(f"{path}: not a share file")
        ring = Ring(width)
        inter = _unpack(f.read(2 * count * ring.nbytes), ring, 2 * count)
    return inter[0::2], inter[1::2], ring, party
