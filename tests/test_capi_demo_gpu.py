"""The C ABI from plain C (examples/capi_demo.c): gcc + libcudart + the
in-tree libinthist_b200.so, no Python or torch on the call path."""

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_plain_c_client():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    r = subprocess.run([os.path.join(ROOT, "examples", "capi_demo")], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("capi_demo ok:"), r.stdout
