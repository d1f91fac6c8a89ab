"""Test configuration: the `gpu` marker, repo import path, shared helpers.

`-m "not gpu"` runs here (no GPU): oracle vs reference golden fixtures, ledger
vs reference transcripts, host logic, C-ABI exports, gloo multi-process.
`-m gpu` runs on a B200: device kernels vs the oracle (share-exact) and vs the
reference's revealed outputs.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and the library if missing) once per session."""
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)
    lib = os.path.join(ROOT, "paper_2305_00645_b200", "libgtree_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", ROOT, "-s", "-j4", "paper_2305_00645_b200/libgtree_b200.so"], check=True)


def golden_npz(name):
    z = np.load(os.path.join(GOLDEN, name))
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def share(values, rng, width=64):
    """Fresh component-major sharing [3, ...] of public values."""
    v = np.asarray(values, dtype=np.uint64)
    m = np.uint64((1 << width) - 1) if width < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    s1 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, v.shape, dtype=np.uint64)
    s2 = rng.integers(0, 1 << 63, v.shape, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, v.shape, dtype=np.uint64)
    s1, s2 = s1 & m, s2 & m
    return np.stack([s1, s2, (v - s1 - s2) & m])


def share_bits(bits, rng):
    b = np.asarray(bits, dtype=np.uint8) & 1
    s1 = rng.integers(0, 2, b.shape, dtype=np.uint8)
    s2 = rng.integers(0, 2, b.shape, dtype=np.uint8)
    return np.stack([s1, s2, b ^ s1 ^ s2])


def opened(comp, width=64):
    c = np.asarray(comp, dtype=np.uint64)
    v = c[0] + c[1] + c[2]
    return v & np.uint64((1 << width) - 1) if width < 64 else v


def opened_bits(b):
    b = np.asarray(b, dtype=np.uint8)
    return (b[0] ^ b[1] ^ b[2]) & 1


KEYS = ((0x1234, 0x5678), (0xA1, 0xB2), (0xC3, 0xD4), (0xE5, 0xF6))


def run_keys(seed: bytes):
    """Device/oracle keys of a run the reference helpers would set up
    (tests/helpers.py:79-99): master = derive_seed(seed, "run"), dealer seed
    derive_seed(seed, "deal")."""
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, keys_tuple, make_keys

    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    k = make_keys(setup, derive_seed(seed, "deal"))
    return setup, k, keys_tuple(k)


def ref_cases():
    z, meta = golden_npz("trees_mpc.npz")
    for k, m in enumerate(meta):
        yield m, z[f"data{k}"], z[f"T{k}"], z[f"F{k}"]
