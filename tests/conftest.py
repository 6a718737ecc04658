import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")
    config.addinivalue_line("markers", "reference: needs the reference package at /root/reference (build container only)")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "zsort"))


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(REPO, "tests", "golden", "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def ref():
    """The reference package itself (only in the build container)."""
    if not reference_available():
        pytest.skip("reference package not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import zsort
    return zsort
