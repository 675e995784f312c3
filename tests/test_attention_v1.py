"""The single-warpgroup attention kernel (fo_attention.cu, FO_ATTN_IMPL=v1)
passes the same attention parity tests as the default column-split kernel.
The implementation is chosen once per process, so the tests run in a child."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_v1_kernel_attention_parity():
    env = dict(os.environ, FO_ATTN_IMPL="v1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu",
                        "tests/test_gpu_parity.py", "-k", "attention or materialize or update"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
