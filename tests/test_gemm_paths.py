"""Both dense GEMM-Q kernels (CTA-pair cta_group::2 and the 1-CTA multicast one)
agree with the oracle. The kernel is chosen once per process (FO_GEMM_2SM), so
the 1-CTA run happens in a child process."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_dense_gemm_q_one_cta_path():
    env = dict(os.environ, FO_GEMM_2SM="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu",
                        "tests/test_gpu_parity.py", "tests/test_gpu_kernels.py",
                        "tests/test_engine.py", "-k", "gemm_q or engine or run"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
