"""The head-sharded engine at world size 2 on ONE GPU: two
processes, each owning half of the heads (pipeline.shard_heads), run the
repo's own engine and layer steps over a gloo process group on cuda:0 and are
compared with the unsharded run.

Per-head work does not depend on the sharding, so it must be bit-exact:
symbol bytes from the GPU mask policy, decoded skip sets, per-head pair counts,
and the bias orders of each rank's head subset. The layer output is a sum of
per-rank partial GEMM-O projections (gemm.py:155-158, 216-217: linear in the
heads), so it differs from one kernel's fp32 accumulation only by bf16
rounding: the stated bf16 tolerance (conftest.py). The dispatch step also runs
its row-chunked GEMM-O / all-reduce overlap (pipeline._dispatch_out_allreduce)
and must equal the unchunked all-reduce bit for bit (the reduction is per row).
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, assert_bf16_close

pytestmark = pytest.mark.gpu

WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
import paper_2509_25401_b200 as fo
from paper_2509_25401_b200.engine import EngineConfig, run
from paper_2509_25401_b200.pipeline import (LayerParams, dispatch_step, new_layer_state,
                                             shard_heads, update_step)
torch.cuda.set_device(0)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
out_dir = sys.argv[1]
res = {}
# 1) the whole engine: GPU policy -> symbols -> cache -> update / dispatch steps
cfg = EngineConfig(n_text=128, n_vision=896, d_model=256, heads=4, tau_q=0.3, tau_kv=0.4,
                   interval_n=3, order_d=1, steps=5, layers=1, seed=3)
r = run(cfg, group=dist.group.WORLD)
lay = r.states[0]
res["heads"] = np.array(shard_heads(cfg.heads, world, rank))
res["s_c"], res["s_s"] = lay.sym.s_c.cpu().numpy(), lay.sym.s_s.cpu().numpy()
act, pair = lay.sym.decoded()
res["active"], res["pair_bits"] = act.cpu().numpy(), pair.cpu().numpy()
res["orders"] = lay.bias.orders.cpu().numpy()
res["outputs"] = np.stack(r.outputs)
res["report"] = np.array([str(r.report.to_dict())])
# 2) the layer steps with the chunked GEMM-O / all-reduce overlap
rng = np.random.default_rng(11)
S, dm, H, order, T = 1024, 256, 4, 1, 128
t = S // T
w = lambda *s: rng.standard_normal(s).astype(np.float32) * s[-2] ** -0.5
wq, wk, wv = w(H, dm, T), w(H, dm, T), w(H, dm, T)
wo = rng.standard_normal((H, T, dm)).astype(np.float32) * T ** -0.5
qn = (1 + 0.05 * rng.standard_normal((H, T))).astype(np.float32)
kn = (1 + 0.05 * rng.standard_normal((H, T))).astype(np.float32)
xs = [torch.from_numpy(rng.standard_normal((S, dm)).astype(np.float32)).cuda() for _ in range(3)]
cb = rng.random((H, t)) < 0.6
cb[:, 0] = True
sb = rng.random((H, t, t)) < 0.5
sb[:, np.arange(t), np.arange(t)] = True
heads = shard_heads(H, world, rank)
params = LayerParams.from_reference(wq, wk, wv, qn, kn, wo, heads=heads)
st = new_layer_state(params, S, order)
sym = fo.encode_symbols(cb[heads], sb[heads], 1)
update_step(st, xs[0], sym, order, group=dist.group.WORLD)
res["step_update"] = update_step(st, xs[1], sym, order, group=dist.group.WORLD).float().cpu().numpy()
res["step_orders"] = st.bias.orders.cpu().numpy()
whole = dispatch_step(st, xs[2], 1, 4, order, group=dist.group.WORLD).float().cpu().numpy()
chunked = dispatch_step(st, xs[2], 1, 4, order, group=dist.group.WORLD, chunks=3,
                        comm_sms=8).float().cpu().numpy()
res["step_dispatch"], res["step_dispatch_chunked"] = whole, chunked
torch.cuda.synchronize()
np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
dist.destroy_process_group()
print("rank", rank, "ok")
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_on_one_gpu_match_unsharded(tmp_path):
    import torch

    import paper_2509_25401_b200 as fo
    from paper_2509_25401_b200.engine import EngineConfig, run
    from paper_2509_25401_b200.pipeline import (LayerParams, dispatch_step, new_layer_state,
                                                 update_step)

    world, port = 2, _free_port()
    procs = []
    for rank in range(world):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE=str(world), LOCAL_RANK="0", PYTHONPATH=str(ROOT))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER, str(tmp_path)], cwd=ROOT,
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, o[-2000:] + e[-4000:]
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]

    # unsharded reference runs in this process
    cfg = EngineConfig(n_text=128, n_vision=896, d_model=256, heads=4, tau_q=0.3, tau_kv=0.4,
                       interval_n=3, order_d=1, steps=5, layers=1, seed=3)
    full = run(cfg)
    lay = full.states[0]
    s_c, s_s = lay.sym.s_c.cpu().numpy(), lay.sym.s_s.cpu().numpy()
    act, pair = (a.cpu().numpy() for a in lay.sym.decoded())
    for g in ranks:
        h = g["heads"]
        # per-head policy decisions, symbol bytes and skip sets: bit-exact
        np.testing.assert_array_equal(g["s_c"], s_c[h])
        np.testing.assert_array_equal(g["s_s"], s_s[h])
        np.testing.assert_array_equal(g["active"], act[h])
        np.testing.assert_array_equal(g["pair_bits"], pair[h])
        # the aggregated report (pair / MAC counts all-reduced) is identical
        want = str(full.report.to_dict())
        if g["report"][0] != want:
            import ast

            a, b = ast.literal_eval(str(g["report"][0])), full.report.to_dict()
            diff = {k: (a[k], b[k]) for k in b if k != "steps" and a[k] != b[k]}
            steps = [(x, y) for x, y in zip(a["steps"], b["steps"]) if x != y]
            raise AssertionError(f"report differs: {diff} first step diff {steps[:1]}")
        for t_, (a, b) in enumerate(zip(g["outputs"], full.outputs)):
            assert_bf16_close(a, b, f"engine step {t_}")
    np.testing.assert_array_equal(ranks[0]["outputs"], ranks[1]["outputs"])

    # layer steps: the same weights and symbols, unsharded and per rank subset
    rng = np.random.default_rng(11)
    S, dm, H, order, T = 1024, 256, 4, 1, 128
    t = S // T
    w = lambda *s: rng.standard_normal(s).astype(np.float32) * s[-2] ** -0.5  # noqa: E731
    wq, wk, wv = w(H, dm, T), w(H, dm, T), w(H, dm, T)
    wo = rng.standard_normal((H, T, dm)).astype(np.float32) * T ** -0.5
    qn = (1 + 0.05 * rng.standard_normal((H, T))).astype(np.float32)
    kn = (1 + 0.05 * rng.standard_normal((H, T))).astype(np.float32)
    xs = [torch.from_numpy(rng.standard_normal((S, dm)).astype(np.float32)).cuda() for _ in range(3)]
    cb = rng.random((H, t)) < 0.6
    cb[:, 0] = True
    sb = rng.random((H, t, t)) < 0.5
    sb[:, np.arange(t), np.arange(t)] = True

    def steps(heads):
        st = new_layer_state(LayerParams.from_reference(wq, wk, wv, qn, kn, wo, heads=heads), S,
                             order)
        sym = fo.encode_symbols(cb[heads], sb[heads], 1)
        update_step(st, xs[0], sym, order)
        u = update_step(st, xs[1], sym, order).float().cpu().numpy()
        d = dispatch_step(st, xs[2], 1, 4, order).float().cpu().numpy()
        return u, d, st.bias.orders.cpu().numpy()

    u_all, d_all, _ = steps(list(range(H)))
    parts = [steps(list(g["heads"])) for g in ranks]
    for g, (u_p, d_p, ord_p) in zip(ranks, parts):
        np.testing.assert_array_equal(g["step_orders"], ord_p)  # bias orders of the rank's heads
        # the chunked overlap equals the whole-tensor all-reduce, bit for bit
        np.testing.assert_array_equal(g["step_dispatch_chunked"], g["step_dispatch"])
        assert_bf16_close(g["step_update"], u_all, "update step (sharded + all-reduce)")
        assert_bf16_close(g["step_dispatch"], d_all, "dispatch step (sharded + all-reduce)")
        # the all-reduce is the sum of the two ranks' partial projections
        assert_bf16_close(g["step_dispatch"], parts[0][1] + parts[1][1], "sum of partials")
