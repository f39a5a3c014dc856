import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference package (CPU tests in the build container only)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import moesim

    return moesim


@pytest.fixture(scope="session")
def golden():
    return ROOT / "tests" / "golden"


@pytest.fixture
def parity_log(request):
    """parity_log(name, measured, bar): append the measured error of a parity
    check and its bar to gpurun_out/parity_log.jsonl (REALB_PARITY_LOG overrides),
    so the margins the tolerances leave are on record."""
    import json

    path = Path(os.environ.get("REALB_PARITY_LOG", ROOT / "gpurun_out" / "parity_log.jsonl"))

    def log(name, measured, bar):
        try:
            path.parent.mkdir(parents=True, exist_ok=True)
            with open(path, "a") as f:
                f.write(json.dumps({"test": request.node.nodeid, "check": name, "measured": float(measured),
                                    "bar": float(bar)}) + "\n")
        except OSError:
            pass

    return log
