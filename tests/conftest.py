import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) -- run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


# ------------------------------------------------------------------------------------------------
# parity counts ("all flagged and masked counts are reported with every parity result"):
# tests call parity_log(name, **counts); the table is printed in the terminal summary and written to
# gpurun_out/parity_counts.jsonl when that directory exists (GPU runs)
@pytest.fixture
def parity_log():
    from tests import parity
    return parity.log


def pytest_terminal_summary(terminalreporter):
    import sys
    mod = sys.modules.get("tests.parity")
    _PARITY = getattr(mod, "LOG", None) if mod else None
    if not _PARITY:
        return
    import json
    tr = terminalreporter
    tr.section("parity counts (masked stop-margin pixels / flagged face-switch primitives / worst tolerance ratio)")
    for r in _PARITY:
        w = r.get("worst", {})
        ws = " ".join(f"{k}={v:.3g}" for k, v in w.items()) if isinstance(w, dict) else str(w)
        extra = " ".join(f"{k}={v}" for k, v in r.items() if k not in ("test", "worst"))
        tr.write_line(f"{r['test']}: {extra} worst[{ws}]")
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "parity_counts.jsonl"), "a") as f:
            for r in _PARITY:
                f.write(json.dumps(r) + "\n")
