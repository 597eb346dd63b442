"""Run the reference's own unit tests against this package (build container only).

``/root/reference`` exists only in the build container; the GPU box skips
this file.  Every reference test module (model, dag, pebble, bounds, dataflow,
autotune, cli, acceptance) imports ``convio``; they are executed with ``convio`` aliased to
``paper_2012_15667_b200`` -- the drop-in claim, tested literally.
"""

import importlib
import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not mounted")

CONFTEST = f'''
import importlib, sys
sys.path.insert(0, {ROOT!r})
pkg = importlib.import_module("paper_2012_15667_b200")
sys.modules["convio"] = pkg
for sub in ("model", "dag", "bounds", "dataflow", "autotune", "pebble", "fixtures", "cli"):
    sys.modules["convio." + sub] = importlib.import_module("paper_2012_15667_b200." + sub)
'''


MODULES = ["test_model.py", "test_dataflow.py", "test_autotune.py", "test_dag.py", "test_pebble.py",
           "test_bounds.py", "test_cli.py", "test_acceptance.py"]


@pytest.mark.parametrize("module", MODULES)
def test_reference_module_passes_against_this_package(module, tmp_path):
    (tmp_path / "conftest.py").write_text(CONFTEST)
    (tmp_path / module).write_text(open(os.path.join(REF_TESTS, module)).read())
    golden = tmp_path / "golden"          # test_cli.py reads golden/tune_best.json beside itself
    golden.mkdir()
    for fn in os.listdir(os.path.join(REF_TESTS, "golden")):
        (golden / fn).write_text(open(os.path.join(REF_TESTS, "golden", fn)).read())
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        str(tmp_path / module)], cwd=tmp_path, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
