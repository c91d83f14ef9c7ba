"""The checked build (-DPRS_CHECKS, paper_2502_08370_b200/_build.py): bounds of every async-copy
destination and scratch index on the TMA / bulk-copy paths (c3 x pass, split DD stage,
partitioned full tensor) and bounded mbarrier waits, asserted on the device (a violation traps;
compute-sanitizer is not available on the GPU pool).  A subset of the GPU parity tests that
covers those paths runs against libprs_chk.so in a child process and must pass unchanged."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SUBSET = ("test_benchmarked_long_line_parareal_matches_oracle_every_iteration and FIE-DR and n4096"
          " or test_batched_step_parity or test_dd_single_step_parity or test_full_tensor_batched_steps"
          " or (test_twin_iterates_match_stored_oracle_digests and c4r_FIE-FIE)"
          " or test_parareal_iterates_match_oracle_every_iteration")


def test_parity_subset_passes_on_the_checked_build():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    from paper_2502_08370_b200 import _build
    so = _build.build(checks=True)
    env = dict(os.environ, PRS_SO=so)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-q", "-x", "-p", "no:cacheprovider", "-k", SUBSET], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=3000)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-15:])
    assert r.returncode == 0, tail
    assert "passed" in tail and "PRS_CHECK failed" not in r.stdout + r.stderr, tail
