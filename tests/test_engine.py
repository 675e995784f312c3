"""The GPU Update–Dispatch scheduler (engine.run) against the reference run().

tests/golden/run.npz was produced by the reference pipeline.run
(pkg/src/omniattn/pipeline.py:337-371) on bf16-rounded weights and inputs
(oracle/gen_golden.py::pipeline_run). Symbols, step costs and the cost report
must match exactly; per-step outputs within the stated bf16 tolerance.
"""

import numpy as np
import pytest

from conftest import TESTS, assert_bf16_close

from paper_2509_25401_b200 import costs
from paper_2509_25401_b200.engine import (EngineConfig, SyntheticWorkload, config_from_dict,
                                          max_rel_error)
from paper_2509_25401_b200.errors import ConsistencyError, ParameterError

GOLD = np.load(TESTS / "golden" / "run.npz")
STEP_KEYS = ("attn_pairs_total", "attn_pairs_computed", "attn_pairs_mask_skipped",
             "gemm_q_macs_dense", "gemm_q_macs_actual", "gemm_o_macs_dense", "gemm_o_macs_actual",
             "gemm_o_bias_macs")
# the configurations oracle/gen_golden.py::RUN_CASES ran through the reference
RUN_CASES = [
    dict(n_text=128, n_vision=896, d_model=128, heads=2, tau_q=0.3, tau_kv=0.4, interval_n=3,
         order_d=1, steps=6, layers=2, workload="drift", smoothness=0.05, seed=7),
    dict(n_text=200, n_vision=1848, d_model=128, heads=2, pool_n=2, tau_q=0.8, tau_kv=0.7,
         interval_n=3, order_d=0, steps=6, layers=1, warmup=4, workload="poly2", smoothness=0.1,
         seed=8),
]


def bf16_round(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16
    return r.astype(np.uint32).view(np.float32)


# ----------------------------------------------------------------- host side
def test_config_validation_mirrors_reference():
    with pytest.raises(ParameterError):
        EngineConfig(n_text=0, n_vision=128)
    with pytest.raises(ParameterError):
        EngineConfig(n_text=1, n_vision=128, tau_q=1.5)
    with pytest.raises(ParameterError):
        EngineConfig(n_text=1, n_vision=128, workload="nope")
    with pytest.raises(ParameterError):
        EngineConfig(n_text=1, n_vision=128, order_d=-1)
    with pytest.raises(ParameterError):  # sm_100a tile geometry
        EngineConfig(n_text=1, n_vision=128, b_q=16, b_k=16, d=16)
    with pytest.raises(ParameterError):
        EngineConfig(n_text=1, n_vision=128, d_model=200)
    with pytest.raises(ParameterError):
        config_from_dict({"n_text": 1, "n_vision": 1, "bogus": 3})
    with pytest.raises(ParameterError):
        config_from_dict({"n_text": 1})
    cfg = config_from_dict({"n_text": 100, "n_vision": 300})
    assert (cfg.n_tokens, cfg.t_q, cfg.t_kv) == (400, 4, 4)


@pytest.mark.parametrize("ci", range(len(RUN_CASES)))
def test_workload_draws_match_reference(ci):
    """Same seed -> the reference's weights and trajectory, bit for bit."""
    cfg = EngineConfig(**RUN_CASES[ci])
    wl = SyntheticWorkload(cfg)
    lp = wl.layer_params[-1]
    probe = np.concatenate([lp.w_q[-1, -3:, :5].ravel(), lp.q_norm[0, :5], lp.k_norm[-1, -5:],
                            lp.w_out[0, :3, -5:].ravel()])
    np.testing.assert_array_equal(probe, GOLD[f"r{ci}_w_probe"])
    xs = np.stack([wl.x(t)[-4:, :6] for t in range(cfg.steps)])
    np.testing.assert_array_equal(xs, GOLD[f"r{ci}_x_probe"])


def test_costs_invariants_and_models():
    sc = costs.StepCost(step=0, phase="dispatch", attn_pairs_total=10, attn_pairs_computed=4,
                        attn_pairs_mask_skipped=6, gemm_q_macs_dense=8, gemm_q_macs_actual=4,
                        gemm_o_macs_dense=8, gemm_o_macs_actual=4)
    rep = costs.account_run([sc], 4)
    assert rep.sparsity == 0.6 and rep.attn_pairs_skipped == 6
    assert rep.speedup_attention == pytest.approx(2.5)
    assert rep.speedup_gemm_o == pytest.approx(4 / (1 + 3 * 0.4))
    assert rep.to_dict()["steps"][0]["sparsity"] == 0.6
    bad = costs.StepCost(step=1, phase="dispatch", attn_pairs_total=10, attn_pairs_computed=4,
                         attn_pairs_mask_skipped=5)
    with pytest.raises(ConsistencyError):
        costs.account_run([bad], 4)
    over = costs.StepCost(step=2, phase="update", attn_pairs_total=1, attn_pairs_computed=1,
                          gemm_q_macs_dense=1, gemm_q_macs_actual=2)
    with pytest.raises(ConsistencyError):
        costs.account_run([over], 1)
    with pytest.raises(ParameterError):
        costs.theoretical_speedup_attention(1.0)
    with pytest.raises(ParameterError):
        costs.sparsity(3, 2)
    assert max_rel_error([1.0, 2.0], [1.0, 4.0]) == 0.5


# ----------------------------------------------------------------- GPU side
@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["drift", "poly1", "poly2"])
def test_x_device_is_bitexact(kind):
    import torch

    cfg = EngineConfig(n_text=64, n_vision=448, d_model=256, steps=5, workload=kind,
                       smoothness=0.07)
    wl = SyntheticWorkload(cfg)
    for t in range(cfg.steps):
        got = wl.x_device(t)
        want = torch.from_numpy(wl.x(t)).to(torch.bfloat16)
        assert torch.equal(got.cpu(), want), f"{kind} t={t}"


def _gold_symbols(ci, li):
    return GOLD[f"r{ci}_l{li}_sc"], GOLD[f"r{ci}_l{li}_ss"]


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(len(RUN_CASES)))
def test_run_matches_reference_run(ci):
    from paper_2509_25401_b200 import engine

    cfg = EngineConfig(**RUN_CASES[ci])
    res = engine.run(cfg)
    # the symbols the last window ran under, per layer
    for li, layer in enumerate(res.states):
        sc, ss = _gold_symbols(ci, li)
        np.testing.assert_array_equal(layer.sym.s_c.cpu().numpy(), sc)
        np.testing.assert_array_equal(layer.sym.s_s.cpu().numpy().reshape(ss.shape), ss)
    # exact work accounting, step by step
    got = np.array([[getattr(sc, k) for k in STEP_KEYS] for sc in res.step_costs], np.int64)
    np.testing.assert_array_equal(got, GOLD[f"r{ci}_costs"])
    r = res.report
    np.testing.assert_array_equal(
        [r.attn_pairs_total, r.attn_pairs_skipped, r.gemm_q_macs_dense, r.gemm_q_macs_actual,
         r.gemm_o_macs_dense, r.gemm_o_macs_actual, r.gemm_o_bias_macs], GOLD[f"r{ci}_report"])
    np.testing.assert_allclose([r.sparsity, r.speedup_attention or 0.0, r.speedup_gemm_o],
                               GOLD[f"r{ci}_speedups"], rtol=1e-12)
    want = GOLD[f"r{ci}_out"].astype(np.float32)
    for t, (g, w) in enumerate(zip(res.outputs, want)):
        assert_bf16_close(g, w, f"case {ci} step {t}")


@pytest.mark.gpu
def test_graphs_equal_eager_and_dense_reference():
    """CUDA-graph replay is bit-identical to eager launches; with no sparsity
    the run equals the dense trajectory."""
    from paper_2509_25401_b200 import engine

    cfg = EngineConfig(**RUN_CASES[0])
    a = engine.run(cfg, graphs=True)
    b = engine.run(cfg, graphs=False)
    for t, (x, y) in enumerate(zip(a.outputs, b.outputs)):
        np.testing.assert_array_equal(x, y, err_msg=f"step {t}")
    dense_cfg = EngineConfig(**dict(RUN_CASES[0], tau_q=0.0, tau_kv=0.0))
    c = engine.run(dense_cfg)
    d = engine.dense_reference(dense_cfg)
    assert c.report.sparsity == 0.0
    for t, (x, y) in enumerate(zip(c.outputs, d)):
        if t % cfg.interval_n == 0:
            np.testing.assert_array_equal(x, y, err_msg=f"update step {t}")
        else:  # dispatch: all heads active, bias empty -> same math, other kernel
            assert_bf16_close(x, y, f"dispatch step {t}")
