"""pytest plugin: run the REFERENCE's own test suite against this package.

    python -m pytest -p scripts.reftests.inthist_alias baseline/ref_tests

Maps the module name ``inthist`` and its submodules (the reference package,
pkg/src/inthist/__init__.py:1-75) onto ``paper_1711_01919_b200`` before the
reference's conftest.py imports it, so every ``from inthist... import`` in the
unmodified reference tests binds to the B200 drop-in.  Test infrastructure
only: the reference test files are copied at run time into the git-ignored
``baseline/ref_tests`` by scripts/reftests/run.sh (never committed).
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# reference submodule -> module of this package that provides its names
SUBMODULES = {
    "core": "domain", "strategies": "strategies", "likelihood": "likelihood",
    "streaming": "streaming", "imgio": "imgio", "bench": "bench", "scan": "scan",
    "cli": "cli", "errors": "errors",
}


def install() -> None:
    pkg = importlib.import_module("paper_1711_01919_b200")
    if "inthist" in sys.modules and sys.modules["inthist"] is not pkg:
        raise RuntimeError("a different 'inthist' is already imported")
    sys.modules["inthist"] = pkg
    for ref_name, ours in SUBMODULES.items():
        mod = importlib.import_module(f"paper_1711_01919_b200.{ours}")
        sys.modules[f"inthist.{ref_name}"] = mod
        setattr(pkg, ref_name, mod)


install()
