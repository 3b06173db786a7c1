import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built C-ABI library")
    config.addinivalue_line("markers", "slow: oracle-heavy test (minutes of CPU)")


# ---- parity margins: every GPU parity assertion records (measured error, bound); the session writes
# them to $RTE_MARGINS_OUT (default gpurun_out/parity_margins.json) so the margins are visible
# (profiles/r02/parity_margins.md is generated from it by scripts/margins_table.py)
_MARGINS = []


@pytest.fixture
def margin(request):
    def rec(value, bound, what=""):
        value, bound = float(value), float(bound)
        _MARGINS.append({"test": request.node.nodeid, "what": what, "value": value, "bound": bound,
                         "ratio": value / bound if bound else None})
        return value
    return rec


def pytest_sessionfinish(session, exitstatus):
    if not _MARGINS:
        return
    import json
    out = os.environ.get("RTE_MARGINS_OUT", os.path.join(ROOT, "gpurun_out", "parity_margins.json"))
    try:
        os.makedirs(os.path.dirname(out), exist_ok=True)
        old = []
        if os.path.exists(out):
            with open(out) as f:
                old = json.load(f)
        seen = {(m["test"], m["what"]) for m in _MARGINS}
        keep = [m for m in old if (m["test"], m["what"]) not in seen]
        with open(out, "w") as f:
            json.dump(keep + _MARGINS, f, indent=1)
    except OSError:
        pass
