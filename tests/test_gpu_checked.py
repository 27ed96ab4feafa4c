"""Device-side bounds checks (the compute-sanitizer stand-in: compute-sanitizer is closed on the GPU
pool).  liblinprim_checked.so (-DLP_CHECKED) traps on any violated index invariant (record gathers,
tile-list entries, hit-bit words, transmittance checkpoints, deterministic partials, emission
positions, K5 items).  A fresh process loads it through LP_LIB and runs C1 forward + backward in the
ray-space, deterministic and no-ray-space modes plus one small C5 TrainStep, then a parity subset."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_clean():
    from paper_2501_16312_b200 import _build
    lib = _build.build(variant="checked")
    env = dict(os.environ, LP_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_c1.py")], capture_output=True, text=True,
                       env=env, cwd=ROOT, timeout=600)
    assert p.returncode == 0 and "LP_CHECK failed" not in p.stdout + p.stderr, (p.stdout[-2000:], p.stderr[-2000:])
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py::test_edge_scenes", "tests/test_gpu_parity.py::test_random_small_scenes",
                        "tests/test_gpu_deterministic.py::test_deterministic_parity", "tests/test_gpu_exact.py"],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert p.returncode == 0 and "LP_CHECK failed" not in p.stdout + p.stderr, (p.stdout[-3000:], p.stderr[-2000:])


def test_checked_build_traps_on_a_corrupted_entry():
    """The checks are live: an out-of-range primitive id in the tile list stops the forward."""
    from paper_2501_16312_b200 import _build
    lib = _build.build(variant="checked")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_negative.py")], capture_output=True,
                       text=True, env=dict(os.environ, LP_LIB=lib), cwd=ROOT, timeout=300)
    assert p.returncode != 0 and "NOT TRAPPED" not in p.stdout
    assert "LP_CHECK failed" in p.stdout + p.stderr
