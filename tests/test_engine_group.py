"""The process-group code paths on the GPU (head sharding with one NCCL
all-reduce per layer) at world size 1, in a child process: the sharded engine
run and the layer steps must give the same bytes as the ungrouped ones. The
decomposition itself (world size 2) is covered on CPU by test_multigpu_gloo."""

import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

SCRIPT = r'''
import numpy as np, torch, torch.distributed as dist
import paper_2509_25401_b200 as fo
from paper_2509_25401_b200.engine import EngineConfig, run
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
cfg = EngineConfig(n_text=128, n_vision=896, d_model=256, heads=4, tau_q=0.3, tau_kv=0.4,
                   interval_n=3, order_d=1, steps=5, layers=2, seed=3)
a = run(cfg, group=dist.group.WORLD)
b = run(cfg)
for t, (x, y) in enumerate(zip(a.outputs, b.outputs)):
    assert np.array_equal(x, y), f"step {t}"
assert a.report.to_dict() == b.report.to_dict()
dist.destroy_process_group()
print("group ok")
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_engine_with_process_group_matches():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()),
               PYTHONPATH=str(ROOT))
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "group ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
