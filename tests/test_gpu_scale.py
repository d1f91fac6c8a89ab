"""The 10^6-scale configurations and the depth policies as first-class parity
tests (B200):

* C4 at its exact config (10^6 x 32 + label, depth 8, default_rng(10**6)):
  revealed tree == the fixed-point shadow oracle (oracle/shadow.py, pinned to
  reference runs by tests/test_oracle.py);
* a C4-shaped 2*10^5-sample run share-for-share equal to the C oracle port;
* C5 at its exact config (random_tree(default_rng(10), 10, 33), 10^7
  queries): every prediction == the plaintext walk;
* depth policies (train.py:81-86): feature_cap and grow to the default cap
  (= column count, AND-reducing the stop bit over > 64 nodes) against trees
  the reference itself trained (tests/golden/trees_policy.npz), plus shares
  vs the oracle.
"""

import numpy as np
import pytest
import torch

import oracle
from oracle import shadow
from conftest import golden_npz, opened, run_keys, share

pytestmark = pytest.mark.gpu


def _dev_share(values, gen):
    """Component-major shares [3, ...] of public values drawn on the device."""
    v = torch.as_tensor(values, device="cuda").to(torch.int64)
    s1 = torch.randint(-(2 ** 63), 2 ** 63 - 1, v.shape, dtype=torch.int64, device="cuda", generator=gen)
    s2 = torch.randint(-(2 ** 63), 2 ** 63 - 1, v.shape, dtype=torch.int64, device="cuda", generator=gen)
    return torch.stack([s1, s2, v - s1 - s2]).contiguous()


def _open_dev(t):
    return t.sum(dim=0).cpu().numpy().view(np.uint64)


def test_c4_full_config_tree_equals_shadow_oracle():
    from paper_2305_00645_b200 import TrainConfig
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, filler_values, make_keys
    from paper_2305_00645_b200.train import DeviceTrainer

    n, nf, depth = 10 ** 6, 32, 8
    data = np.random.default_rng(10 ** 6).integers(0, 2, (n, nf + 1), dtype=np.uint8)
    seed = (40_000).to_bytes(16, "little")
    setup = SeedSetup.from_master(derive_seed(seed, "run"))
    keys = make_keys(setup, derive_seed(seed, "deal"))
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    X, Y = _dev_share(data[:, :-1], gen), _dev_share(data[:, -1], gen)
    tr = DeviceTrainer(n, nf, TrainConfig(depth=depth))
    assert tr.run(X, Y, torch.from_numpy(fill.view(np.int64)).cuda(), keys) == depth
    want_T, want_F = shadow.mpc_train(data, depth, fill)
    assert np.array_equal(_open_dev(tr.T), want_T) and np.array_equal(_open_dev(tr.F), want_F)


def test_c4_shaped_2e5_share_exact_vs_oracle():
    from paper_2305_00645_b200 import TrainConfig
    from paper_2305_00645_b200.seeds import derive_seed, filler_values
    from paper_2305_00645_b200.train import train_components

    n, nf, depth = 200_000, 32, 8
    rng = np.random.default_rng(10 ** 6)
    data = rng.integers(0, 2, (n, nf + 1), dtype=np.uint8)
    seed = (40_001).to_bytes(16, "little")
    setup, k, keys = run_keys(seed)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    T, F, d = train_components(X, Y, TrainConfig(depth=depth), setup, derive_seed(seed, "deal"))
    fill = filler_values(setup.filler_seed, (1 << depth) - 1, nf + 1)
    To, Fo, _ = oracle.train(X, Y, fill, depth, keys)
    assert np.array_equal(T, To) and np.array_equal(F, Fo)
    want_T, want_F = shadow.mpc_train(data, depth, fill)
    assert np.array_equal(opened(T), want_T) and np.array_equal(opened(F), want_F)


def test_c5_full_config_every_prediction_equals_plaintext():
    from paper_2305_00645_b200.infer import infer_device
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed, make_keys

    n, nf, depth = 10 ** 7, 32, 10
    Tv, _ = shadow.random_tree(np.random.default_rng(10), depth, nf + 1)
    q = np.random.default_rng(10).integers(0, 2, (n, nf), dtype=np.uint8)
    setup = SeedSetup.from_master(derive_seed(b"\x05" * 16, "run"))
    keys = make_keys(setup, derive_seed(b"\x05" * 16, "deal"))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    Q = _dev_share(torch.from_numpy(q).cuda(), gen)
    T = _dev_share(torch.from_numpy(Tv.view(np.int64)).cuda(), gen)
    out = torch.empty((3, n), dtype=torch.int64, device="cuda")
    infer_device(T, depth, Q, keys, out=out)
    del Q
    got = _open_dev(out)
    assert np.array_equal(got, shadow.plaintext_infer(Tv, depth, q))


@pytest.mark.parametrize("case", ["feature_cap_80x4", "grow_default_cap_3000x10"])
def test_depth_policies_match_reference_trees_and_oracle(case):
    from paper_2305_00645_b200 import TrainConfig
    from paper_2305_00645_b200.seeds import derive_seed, filler_values
    from paper_2305_00645_b200.train import resolved_depth, train_components

    z, meta = golden_npz("trees_policy.npz")
    k = next(i for i, m in enumerate(meta) if m["name"] == case)
    m, data = meta[k], z[f"data{k}"]
    cfg = TrainConfig(depth=m["depth_arg"], policy=m["policy"])
    seed = bytes.fromhex(m["seed"])
    setup, _, keys = run_keys(seed)
    rng = np.random.default_rng(k)
    X, Y = share(data[:, :-1], rng), share(data[:, -1], rng)
    T, F, d = train_components(X, Y, cfg, setup, derive_seed(seed, "deal"))
    assert d == m["trained_depth"]
    assert np.array_equal(opened(T), z[f"T{k}"]) and np.array_equal(opened(F), z[f"F{k}"])
    cap = resolved_depth(cfg, data.shape[1])
    fill = filler_values(setup.filler_seed, (1 << cap) - 1, data.shape[1])
    To, Fo, do = oracle.train(X, Y, fill, cap, keys, policy=1 if m["policy"] == "grow" else 0)
    slots = (1 << d) - 1
    assert do == d and np.array_equal(T, To[:, :slots]) and np.array_equal(F, Fo[:, :slots])
