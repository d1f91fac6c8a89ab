"""Seed derivation, pairwise PRG keys and the public filler stream.

Mirrors the reference's key schedule (pkg/src/obtree/transport.py:58-128):
``derive_seed`` and ``SeedSetup`` are restated byte-for-byte so a run's
pairwise seeds and the public filler seed are the ones the reference derives
from the same master.  The device PRG is Philox4x32-10 keyed with the first 8
bytes of each 16-byte seed (little endian); the reference's AES-CTR streams
only ever shape share values, never revealed outputs.

``filler_values`` is the one stream that reaches revealed outputs (the
placeholder payloads in T, tree.py:160-169), so it is computed exactly as the
reference does: AES-128-CTR over the filler seed, zero IV, little-endian
uint64 words modulo (n_columns - 1).  It is public and host-side.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass
from typing import Dict

import numpy as np

from ._native import gt_keys

PARTIES = (1, 2, 3)
SEED_BYTES = 16


def derive_seed(master: bytes, label: str) -> bytes:
    """transport.py:58-60."""
    return hashlib.sha256(master + b"/" + label.encode()).digest()[:SEED_BYTES]


@dataclass
class SeedSetup:
    """transport.py:97-128."""

    master: bytes
    pair_seeds: Dict[int, bytes]
    local_seeds: Dict[int, bytes]
    enclave_seed: bytes
    filler_seed: bytes
    enclave_channel_keys: Dict[int, bytes]

    @classmethod
    def from_master(cls, master: bytes) -> "SeedSetup":
        if len(master) == 0:
            raise ValueError("empty master seed")
        return cls(
            master=master,
            pair_seeds={i: derive_seed(master, f"pair/{i}") for i in PARTIES},
            local_seeds={i: derive_seed(master, f"local/{i}") for i in PARTIES},
            enclave_seed=derive_seed(master, "enclave"),
            filler_seed=derive_seed(master, "filler"),
            enclave_channel_keys={i: derive_seed(master, f"enclave-chan/{i}") for i in PARTIES},
        )

    @classmethod
    def from_int(cls, seed: int) -> "SeedSetup":
        return cls.from_master(int(seed).to_bytes(16, "little", signed=False))


def philox_key(seed: bytes):
    if len(seed) < 8:
        raise ValueError("PRG seed must be at least 8 bytes")
    return struct.unpack("<II", seed[:8])


def make_keys(setup: SeedSetup, dealer_seed: bytes) -> gt_keys:
    """Device keys: dealer key + pair[i] = SeedSetup.pair_seeds[i+1]."""
    k = gt_keys()
    k.dealer.k0, k.dealer.k1 = philox_key(dealer_seed)
    for i in range(3):
        k.pair[i].k0, k.pair[i].k1 = philox_key(setup.pair_seeds[i + 1])
    return k


def keys_tuple(k: gt_keys):
    return ((k.dealer.k0, k.dealer.k1),) + tuple((k.pair[i].k0, k.pair[i].k1) for i in range(3))


def aes_ctr_words(seed: bytes, count: int) -> np.ndarray:
    """AES-128-CTR keystream (zero IV, zero plaintext) as LE uint64 words
    (AesCtrPrg.next_words(count, 64), transport.py:63-89)."""
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes

    if len(seed) != SEED_BYTES:
        raise ValueError("PRG seed must be 16 bytes")
    enc = Cipher(algorithms.AES(seed), modes.CTR(b"\x00" * 16)).encryptor()
    raw = enc.update(b"\x00" * (8 * count))
    return np.frombuffer(raw, dtype="<u8").astype(np.uint64)


def filler_values(seed: bytes, total: int, n_columns: int) -> np.ndarray:
    """Public placeholder features per heap slot (tree.py:160-169)."""
    if n_columns < 2:
        raise ValueError("need at least one feature column")
    return aes_ctr_words(seed, total) % np.uint64(n_columns - 1)


def share_values(values: np.ndarray, width: int, seed: bytes):
    """The reference dealer's input split (dealer.py:259-263): AES-CTR stream
    of derive_seed(seed, "input"); s1, s2 = next n words each, s3 = v - s1 - s2.
    Returns the three parties' (lo, hi) pairs."""
    mask = np.uint64((1 << width) - 1) if width < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    flat = np.asarray(values, dtype=np.uint64).ravel() & mask
    n = flat.size
    if width != 64:
        raise ValueError("input sharing here is for the Z_2^64 count ring")
    words = aes_ctr_words(derive_seed(seed, "input"), 2 * n)
    s1, s2 = words[:n], words[n:]
    s3 = flat - s1 - s2
    return [(s1, s2), (s2, s3), (s3, s1)]
