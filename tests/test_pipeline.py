"""Layer composition (reference pipeline.py:223-326) on the GPU against the
oracle restatement, plus the bench contract of the reference arm (CPU)."""

import json
import subprocess
import sys

import numpy as np
import pytest

import oracle
from conftest import ROOT, assert_bf16_close

T = 128


def _oracle_layer(x, P, cb, order, steps):
    """Oracle Update(t=0) then Dispatch(t=1..) with the same symbols."""
    n = x[0].shape[0]
    H = P["w_q"].shape[0]
    t = n // T
    pos = np.arange(n)
    stacks = [[None] * t for _ in range(H)]
    valid = [[0] * t for _ in range(H)]
    outs = []
    bias = orders = None
    for step, xs in enumerate(x):
        if step == 0:
            q = oracle.project_q(xs, P["w_q"], P["q_norm"], None, T)
        else:
            q = oracle.project_q(xs, P["w_q"], P["q_norm"], cb, T, fill=0.0)
        k = np.stack([oracle.rope(oracle.rms_norm(xs @ P["w_k"][h], P["k_norm"][h]), pos) for h in range(H)])
        v = np.stack([xs @ P["w_v"][h] for h in range(H)])
        if step == 0:
            o = np.stack([oracle.masked_attention(q[h], k[h], v[h], np.ones(t, bool), np.ones((t, t), bool), T, T)
                          for h in range(H)])
            for h in range(H):
                for i in range(t):
                    stacks[h][i], valid[h][i] = oracle.update_entry(stacks[h][i], valid[h][i],
                                                                    o[h, i * T:(i + 1) * T], order)
            out, bias, orders = oracle.project_out_update(o, P["w_out"], cb.T, stacks, valid, order, T)
        else:
            o = np.stack([oracle.masked_attention(q[h], k[h], v[h], cb[h], P["skip"][h], T, T)
                          for h in range(H)])
            o = np.nan_to_num(o)  # cached rows are never read by GEMM-O dispatch
            out = oracle.project_out_dispatch(o, P["w_out"], cb.T, bias, orders, step, 4, order, T)
        outs.append(out)
    return outs


@pytest.mark.gpu
def test_update_then_dispatch_matches_oracle():
    import torch

    import paper_2509_25401_b200 as fo

    rng = np.random.default_rng(5)
    n, dm, H, order = 384, 256, 2, 1
    t = n // T

    def bfr(a):
        return torch.from_numpy(a.astype(np.float32)).bfloat16().float().numpy()

    P = dict(w_q=bfr(rng.standard_normal((H, dm, T)) * dm ** -0.5),
             w_k=bfr(rng.standard_normal((H, dm, T)) * dm ** -0.5),
             w_v=bfr(rng.standard_normal((H, dm, T)) * dm ** -0.5),
             q_norm=(1 + 0.05 * rng.standard_normal((H, T))).astype(np.float32),
             k_norm=(1 + 0.05 * rng.standard_normal((H, T))).astype(np.float32),
             w_out=bfr(rng.standard_normal((H, T, dm)) * T ** -0.5))
    cb = np.zeros((H, t), bool)
    sb = np.zeros((H, t, t), bool)
    for h in range(H):
        cb[h], sb[h] = oracle.random_masks(rng, t, t, 1, density=0.6, cache_density=0.6)
    P["skip"] = sb
    xs = [bfr(rng.standard_normal((n, dm))) for _ in range(3)]
    want = _oracle_layer(xs, P, cb, order, 3)

    params = fo.LayerParams.from_reference(P["w_q"], P["w_k"], P["w_v"], P["q_norm"], P["k_norm"],
                                           P["w_out"])
    state = fo.new_layer_state(params, n, order)
    sym = fo.encode_symbols(cb, sb, 1)
    got = [fo.update_step(state, torch.from_numpy(xs[0]).cuda(), sym, order)]
    for step in (1, 2):
        got.append(fo.dispatch_step(state, torch.from_numpy(xs[step]).cuda(), step, 4, order))
    for step, (g, w) in enumerate(zip(got, want)):
        assert_bf16_close(g.float().cpu().numpy(), w, f"step {step}")


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` prints one JSON line with the base keys."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--config", "c1"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] in ("reference", "port")
    # one step = the whole layer (the K slices partition it)
    assert "the whole layer step" in line["cpu_baseline"]["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
