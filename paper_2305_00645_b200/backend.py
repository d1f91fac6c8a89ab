"""``--backend b200`` for the reference's own command line.

The reference CLI (``obtree.cli``, pkg/src/obtree/cli.py) builds every
secure run the same way: ``run_local(body, seeds=..., materials=...,
enclave_handler=..., lane_limit=..., timeout=...)`` (rss.py:489-542) with a
``body`` that calls ``train_tree`` (cmd_train cli.py:419-483, cmd_compare
:617-688, _bench_train :738-775), ``infer_batch`` (cmd_infer :531-577,
_bench_infer :777-808) or ``oaa`` (_bench_oaa :696-735).  Those four names
are module globals of ``obtree.cli`` (its ``from .rss import run_local``
etc., cli.py:26-49), so switching the backend is rebinding them to this
package's drop-ins (engine.py): the reference's argument parsing, config
files, dealing, share files, tree validation, compare/bench reports and exit
codes run unchanged, and every secure computation runs on the B200 through
the C ABI.  ``metrics.json`` / the printed byte and round totals come from
the drop-in's transcript (ledger.py), which reproduces the reference's
record for record.

    python -m paper_2305_00645_b200.backend [--backend b200|reference] <obtree argv>

A maintainer adds the same switch inside obtree.cli with the four-line patch
in INTEGRATION.md.  The reference package itself is found on ``sys.path``,
else under ``$OBTREE_SRC``, else in this repo's ``baseline/_ref`` install.
"""

from __future__ import annotations

import contextlib
import importlib
import os
import sys
from typing import Dict, Iterator, Optional, Sequence

from . import engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

#: obtree.cli global -> the B200 drop-in that replaces it
SWITCHED = {
    "run_local": engine.run_local,
    "train_tree": engine.train_tree,
    "infer_batch": engine.infer_batch,
    "oaa": engine.oaa,
}


def reference_cli():
    """Import the reference's ``obtree.cli`` module (ImportError if absent)."""
    try:
        return importlib.import_module("obtree.cli")
    except ImportError:
        pass
    for extra in (os.environ.get("OBTREE_SRC"), os.path.join(ROOT, "baseline", "_ref")):
        if extra and os.path.isdir(os.path.join(extra, "obtree")) and extra not in sys.path:
            sys.path.append(extra)
    return importlib.import_module("obtree.cli")


@contextlib.contextmanager
def switched(cli_module=None) -> Iterator[object]:
    """Rebind the reference CLI's protocol entry points to the B200 drop-ins
    for the duration of the block; restores them afterwards."""
    mod = cli_module if cli_module is not None else reference_cli()
    saved: Dict[str, object] = {}
    for name, repl in SWITCHED.items():
        if not hasattr(mod, name):
            raise ImportError(f"{mod.__name__} has no {name!r} to switch (incompatible reference CLI)")
        saved[name] = getattr(mod, name)
        setattr(mod, name, repl)
    try:
        yield mod
    finally:
        for name, orig in saved.items():
            setattr(mod, name, orig)


def main(argv: Optional[Sequence[str]] = None) -> int:
    args = list(sys.argv[1:] if argv is None else argv)
    backend = "b200"
    if args and args[0].startswith("--backend"):
        flag = args.pop(0)
        backend = flag.split("=", 1)[1] if "=" in flag else (args.pop(0) if args else "")
    if backend not in ("b200", "reference"):
        print(f"error: unknown backend {backend!r} (b200 | reference)", file=sys.stderr)
        return 1
    try:
        mod = reference_cli()
    except ImportError as e:
        print(f"error: the reference CLI (obtree) is not importable: {e}", file=sys.stderr)
        return 1
    if backend == "reference":
        return mod.main(args)
    with switched(mod):
        return mod.main(args)


if __name__ == "__main__":
    sys.exit(main())
