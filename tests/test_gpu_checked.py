"""The device-checked build (-DMCS_DEVICE_CHECKS: bounds, probe termination, ladder and donor
invariants asserted on device; compute-sanitizer is not available on this pool) runs every
kernel family without a failed check, and its results equal the plain build's."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(lib):
    env = dict(os.environ, MCS_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_workload.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_checked_build_passes_and_matches_plain():
    from paper_2504_18056_b200 import build as b
    checked = b.CHECKED_LIB if os.path.exists(b.CHECKED_LIB) else b.build_checked()
    got = _run(checked)
    ref = _run(b.LIB)
    assert got == ref
