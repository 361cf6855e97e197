import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# Near-tie counts (north_star: "bit-exact except where a threshold lies within 1e-9
# of a cumulative-sum boundary, with that count reported"):
# parity tests record them here and the terminal summary prints them.
_NEAR_TIES = []


@pytest.fixture
def near_tie_report(request):
    def rec(**kw):
        _NEAR_TIES.append(dict(test=request.node.name, **kw))
    return rec


def pytest_terminal_summary(terminalreporter):
    if not _NEAR_TIES:
        return
    terminalreporter.section("near-tie counts (resampling thresholds within 1e-9; label sets within 1e-5)")
    for r in _NEAR_TIES:
        terminalreporter.write_line(" ".join("%s=%s" % (k, v) for k, v in r.items()))
    out = os.environ.get("PHD_NEAR_TIE_LOG")
    if out:
        import json
        with open(out, "w") as fh:
            json.dump(_NEAR_TIES, fh, indent=1)
