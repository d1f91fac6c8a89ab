"""``--backend b200`` on the reference's own CLI (paper_2305_00645_b200.backend).

The golden records (tests/golden/cli/cli.json) are what the UNMODIFIED
reference CLI printed and wrote for each argv (make_golden.py, obtree.cli.main
on its own backend).  Here the same obtree.cli.main runs with its protocol
entry points switched to the B200 drop-ins: stdout (byte and round totals),
tree.json, tree_meta.json, metrics.json, predictions.csv and the compare /
bench reports must equal the reference's text exactly.  The reference package
is needed (obtree importable, $OBTREE_SRC, or the repo's baseline/_ref
install); without it these tests skip."""

import contextlib
import hashlib
import io
import json
from pathlib import Path

import pytest

from paper_2305_00645_b200 import backend, engine

G = Path(__file__).parent / "golden" / "cli"
GOLD = json.loads((G / "cli.json").read_text())

try:
    REF = backend.reference_cli()
except ImportError:  # pragma: no cover - depends on the box
    REF = None
needs_ref = pytest.mark.skipif(REF is None, reason="reference CLI (obtree) not importable")


def _run(name, tmp_path, *extra):
    rec = GOLD[name]
    argv = [a.format(g=G, t=tmp_path) for a in rec["argv"]]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = backend.main([*extra, *argv])
    return rec, argv, code, buf.getvalue().replace(str(tmp_path), "{t}")


def _check_files(rec, argv):
    target = Path(argv[argv.index("--out") + 1])
    for fname, want in rec["files"].items():
        if fname == "report":
            assert json.loads(target.read_text()) == json.loads(want)
        else:
            assert (target / fname).read_text() == want, fname


@needs_ref
def test_switch_rebinds_the_reference_entry_points_and_restores_them():
    before = {k: getattr(REF, k) for k in backend.SWITCHED}
    with backend.switched(REF) as mod:
        assert mod.train_tree is engine.train_tree and mod.run_local is engine.run_local
        assert mod.infer_batch is engine.infer_batch and mod.oaa is engine.oaa
    assert {k: getattr(REF, k) for k in backend.SWITCHED} == before


@needs_ref
def test_deal_through_the_switched_cli_writes_reference_identical_files(tmp_path):
    rec, argv, code, out = _run("deal_train", tmp_path)
    assert code == rec["exit"] == 0 and out == rec["stdout"]
    target = Path(argv[argv.index("--out") + 1])
    for fname, digest in rec["files"].items():
        assert hashlib.sha256((target / fname).read_bytes()).hexdigest() == digest, fname


@needs_ref
@pytest.mark.parametrize("name", ["err_reveal_prod", "err_width"])
def test_usage_errors_keep_the_reference_exit_codes(name, tmp_path):
    rec, argv, code, out = _run(name, tmp_path)
    assert code == rec["exit"] == 1


def test_unknown_backend_is_a_usage_error():
    assert backend.main(["--backend", "cpu", "train"]) == 1


def test_drop_ins_refuse_foreign_engines():
    with pytest.raises(engine.TransportError):
        engine.train_tree(object(), None, None, None)
    with pytest.raises(engine.TransportError):
        engine.oaa(object(), None, None)


GPU_CASES = ["train_mpc", "train_tee", "train_grow", "train_conf", "infer_dir", "infer_plain", "compare_mpc",
             "compare_tee", "train_deal", "err_tolerance", "bench_oaa", "bench_train", "bench_infer"]


@pytest.mark.gpu
@needs_ref
def test_reference_cli_on_the_b200_backend_matches_reference_outputs(tmp_path):
    # order matters: infer_dir reads train_mpc's shares, infer_plain train_tee's tree.json,
    # train_deal reads deal_train's directory
    for name in ["deal_train"] + GPU_CASES:
        rec, argv, code, out = _run(name, tmp_path, "--backend", "b200")
        assert code == rec["exit"], name
        if name.startswith("bench"):  # the seconds column is this machine's time
            assert out.splitlines()[0] == rec["stdout"].splitlines()[0]
        else:
            assert out == rec["stdout"], name
        if code == 0 and name != "deal_train":
            _check_files(rec, argv)
