"""The boundary from plain C: examples/c_api_demo.c compiles as strict C99 against
include/mcs.h alone and links to libmcs.so; without a CUDA device the first call fails loudly
(MCS_E_CUDA with the driver's message) instead of falling back to anything."""
import json
import subprocess

import pytest

from c_api_build import build_demo


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def test_c_demo_builds_as_strict_c99(tmp_path):
    assert build_demo(str(tmp_path))


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_c_demo_fails_loudly_without_a_device(tmp_path):
    exe = build_demo(str(tmp_path))
    r = subprocess.run([exe, "64", "32"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3, (r.returncode, r.stdout, r.stderr)  # MCS_E_CUDA
    assert json.loads(r.stdout.strip().splitlines()[-1]) == {"status": 3,
                                                             "call": "mcs_create(&cfg, &ctx)"}
    assert "CUDA" in r.stderr
