import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def programs():
    from paper_2509_16248_b200.harness import programs as load

    return load()


def pytest_sessionfinish(session, exitstatus):
    """Decision margins |stat - threshold| logged by parity.check_scalars go
    to $GM_MARGINS_OUT (JSON lines) when set (tools/gpu_round.sh sets it)."""
    out = os.environ.get("GM_MARGINS_OUT")
    if out:
        from parity import dump_margins

        dump_margins(out)
