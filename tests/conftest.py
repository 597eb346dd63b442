"""Shared pytest setup.

``-m gpu`` tests need a B200 and the in-tree ``libconvio_b200.so``; every
other test runs on a CPU-only machine.  Nothing here reads ``/root/reference``
(the GPU box does not have it); the few tests that cross-check against the
live reference skip themselves when it is absent.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    """Skip ``gpu``-marked tests on machines without a CUDA device (a plain
    ``pytest`` here then passes instead of failing on the driver probe)."""
    if not any("gpu" in item.keywords for item in items):
        return
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


# ---- measured parity errors (CONVIO_PARITY_LOG=path): every oracle.rel_err call of a
# test is recorded with its test id, so the stated tolerances can be set against the
# measured errors (tests/golden/parity_errors_*.json keeps the GPU runs' logs)
_ERRORS: list = []


@pytest.fixture(autouse=True)
def _record_rel_err(request):
    path = os.environ.get("CONVIO_PARITY_LOG")
    if not path:
        yield
        return
    from oracle import conv_oracle
    orig = conv_oracle.rel_err

    def rel_err(y, ref):
        v = orig(y, ref)
        _ERRORS.append({"test": request.node.nodeid, "rel_err": v})
        return v

    conv_oracle.rel_err = rel_err
    try:
        yield
    finally:
        conv_oracle.rel_err = orig


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("CONVIO_PARITY_LOG")
    if path and _ERRORS:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as fh:
            json.dump(_ERRORS, fh, indent=0)
