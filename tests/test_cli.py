"""CLI parity against the reference CLI's own outputs (tests/golden/cli/cli.json,
written by make_golden.py running obtree.cli.main on the same argv).

CPU: dealing (byte-identical share / seed / meta files), the communication
tables of ``bench`` (analytic, no device run), config files and usage errors.
GPU: train / infer / compare end to end -- stdout, tree.json, tree_meta.json,
metrics.json, predictions.csv and compare reports must equal the reference's
text exactly (reference test_cli.py style)."""

import contextlib
import hashlib
import io
import json
from pathlib import Path

import pytest

from paper_2305_00645_b200 import cli

G = Path(__file__).parent / "golden" / "cli"
GOLD = json.loads((G / "cli.json").read_text())


def _run(name, tmp_path):
    rec = GOLD[name]
    argv = [a.format(g=G, t=tmp_path) for a in rec["argv"]]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    return rec, argv, code, buf.getvalue().replace(str(tmp_path), "{t}")


def _check_files(rec, argv):
    target = Path(argv[argv.index("--out") + 1])
    for fname, want in rec["files"].items():
        if fname == "report":
            assert json.loads(target.read_text()) == json.loads(want)
        else:
            assert (target / fname).read_text() == want, fname


def test_deal_writes_reference_identical_files(tmp_path):
    rec, argv, code, out = _run("deal_train", tmp_path)
    assert code == rec["exit"] == 0 and out == rec["stdout"]
    target = Path(argv[argv.index("--out") + 1])
    for fname, digest in rec["files"].items():
        assert hashlib.sha256((target / fname).read_bytes()).hexdigest() == digest, fname
    assert not list(target.rglob("material.bin"))


@pytest.mark.parametrize("name", ["bench_oaa", "bench_train", "bench_infer"])
def test_bench_tables_match_reference(name):
    rec = GOLD[name]
    argv = [a.format(g=G, t="/nonexistent") for a in rec["argv"]]
    args = cli.build_parser().parse_args(argv)
    rows = cli.bench_rows(args.suite, args, cli.build_run_config(args), run=False)
    assert rows == json.loads(rec["files"]["report"])


@pytest.mark.parametrize("name", ["err_reveal_prod", "err_width"])
def test_usage_errors_exit_like_reference(name, tmp_path):
    rec, argv, code, out = _run(name, tmp_path)
    assert code == rec["exit"] == cli.EXIT_USAGE


def test_config_file_and_seed_parsing(tmp_path):
    assert cli.parse_seed("7") == (7).to_bytes(16, "little")
    assert cli.parse_seed("0x0badcafe") == bytes.fromhex("0badcafe")
    with pytest.raises(cli.UsageError):
        cli.parse_seed("zz")
    conf = cli.load_config_file(str(G / "run.conf"))
    assert conf == {"depth": "3", "seed": "99", "profile": "test"}
    args = cli.build_parser().parse_args(["train", "--data", "x", "--depth", "5", "--out", "o"])
    cli.apply_config(args, conf)
    assert args.depth == 5 and args.seed == "99" and args.profile == "test"
    bad = tmp_path / "bad.conf"
    bad.write_text("nonsense_key = 1\n")
    assert cli.main(["train", "--config", str(bad), "--data", "x", "--out", str(tmp_path / "o")]) == cli.EXIT_USAGE
    bad.write_text("depth 3\n")
    assert cli.main(["train", "--config", str(bad), "--data", "x", "--out", str(tmp_path / "o")]) == cli.EXIT_USAGE


def test_missing_data_file_is_usage_error(tmp_path):
    assert cli.main(["train", "--data", str(tmp_path / "nope.csv"), "--out", str(tmp_path / "o")]) == cli.EXIT_USAGE
    (tmp_path / "bad.csv").write_text("0,1\n1,2\n")
    assert cli.main(["train", "--data", str(tmp_path / "bad.csv"), "--out", str(tmp_path / "o")]) == cli.EXIT_USAGE


GPU_CASES = ["train_mpc", "train_tee", "train_grow", "train_conf", "infer_dir", "infer_plain", "compare_mpc",
             "compare_tee", "train_deal", "err_tolerance", "bench_oaa", "bench_train", "bench_infer"]


@pytest.mark.gpu
def test_cli_end_to_end_matches_reference(tmp_path):
    # order matters: infer_dir reads train_mpc's shares, infer_plain train_tee's tree.json,
    # train_deal reads deal_train's directory
    for name in ["deal_train"] + GPU_CASES:
        rec, argv, code, out = _run(name, tmp_path)
        assert code == rec["exit"], name
        if name.startswith("bench"):  # the seconds column is this machine's device time
            assert out.splitlines()[0] == rec["stdout"].splitlines()[0]
        else:
            assert out == rec["stdout"], name
        if code == 0 and name != "deal_train":
            _check_files(rec, argv)
