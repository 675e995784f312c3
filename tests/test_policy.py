"""Update-step mask policy (reference policy.py:44-234).

CPU: the oracle restatement against fixtures produced by running the
reference's generate_masks (oracle/gen_golden.py -> tests/golden/policy.npz)
and the reference test suite's anchors (pkg/tests/test_policy.py); host-side
threshold logic. GPU: fo_generate_masks through the C ABI, bit-exact against
the fixtures and the oracle, plus the reference suite's invariants at the
sm_100a block size (b = d = 128)."""

import numpy as np
import pytest

import oracle
from conftest import ROOT

GOLD = ROOT / "tests" / "golden" / "policy.npz"
T = 128


def bf16(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def _cases():
    g = np.load(GOLD)
    for ci in range(int(g["n_cases"])):
        p = f"p{ci}_"
        n, n_text, pool, tq, tkv, sq, guard = g[p + "args"]
        yield (ci, bf16(g[p + "q"]), bf16(g[p + "k"]), g[p + "cache"], g[p + "skip"],
               dict(pool_n=int(pool), n_text=int(n_text), tau_q=float(tq), tau_kv=float(tkv),
                    s_q=float(sq), guard=bool(guard)))


def _structured_qk(rng, n, heads):
    """Blocks sharing a random direction plus noise (as gen_golden.policy)."""
    t = -(-n // T)
    q = np.empty((n, heads, T), np.float32)
    k = np.empty((n, heads, T), np.float32)
    for h in range(heads):
        bq = rng.standard_normal((t, T)) * 1.5
        bk = rng.standard_normal((t, T)) * 1.5
        q[:, h] = np.repeat(bq, T, 0)[:n] + rng.standard_normal((n, T))
        k[:, h] = np.repeat(bk, T, 0)[:n] + rng.standard_normal((n, T))
    import torch

    rnd = lambda a: torch.from_numpy(a).bfloat16().float().numpy()  # noqa: E731
    return rnd(q), rnd(k)


# --------------------------------------------------------------------------
# CPU: oracle pinned to the reference
# --------------------------------------------------------------------------
@pytest.mark.parametrize("case", list(range(5)))
def test_oracle_matches_reference_fixture(case):
    ci, q, k, cache, skip, kw = list(_cases())[case]
    cb, sb = oracle.generate_masks(q, k, T, T, **kw)
    assert np.array_equal(cb, cache)
    assert np.array_equal(sb, skip)


def test_fixtures_are_nontrivial():
    dens = [c.mean() for _, _, _, c, _, _ in _cases()]
    assert min(dens) < 0.5 and max(dens) == 1.0  # degrade case keeps only text
    skips = [s[c].mean() for _, _, _, c, s, _ in _cases()]
    assert all(0.0 < s < 1.0 for s in skips)


def test_oracle_anchor_worked_example():
    # reference pkg/tests/test_policy.py:126-130
    c = np.array([0.1, 0.4, 0.2, 0.3])
    g = np.array([0.05, 0.5, 0.15, 0.3])
    sel = oracle.ascending_budget_prefix(c, 0.35) & oracle.ascending_budget_prefix(g, 0.35)
    assert set(np.flatnonzero(sel)) == {0, 2}


def test_oracle_anchor_uniform_row_budget():
    # reference pkg/tests/test_policy.py:167-178: 2 * 0.1 <= 0.25 < 3 * 0.1
    scores = np.full(10, 0.1, np.float32).astype(np.float64)
    assert list(np.flatnonzero(oracle.ascending_budget_prefix(scores, 0.25, absolute=True))) == [0, 1]


def test_ramp_threshold_host():
    # reference pkg/tests/test_policy.py:251-263
    from paper_2509_25401_b200.policy import ramp_threshold

    assert ramp_threshold(0.5, 0, 10) == 0.0
    assert ramp_threshold(0.5, 10, 10) == 0.5 and ramp_threshold(0.5, 25, 10) == 0.5
    assert ramp_threshold(0.5, 5, 10) == pytest.approx(0.25)
    assert ramp_threshold(0.7, 0, 0) == 0.7
    assert oracle.ramp_threshold(0.5, 5, 10) == ramp_threshold(0.5, 5, 10)


def test_mask_policy_validation_host():
    from paper_2509_25401_b200 import MaskPolicy, ParameterError

    with pytest.raises(ParameterError):
        MaskPolicy(n_text=0, tau_q=1.5, tau_kv=0.1)
    with pytest.raises(ParameterError):
        MaskPolicy(n_text=0, tau_q=0.5, tau_kv=0.1, s_q=-0.1)
    with pytest.raises(ParameterError):
        MaskPolicy(n_text=0, tau_q=0.5, tau_kv=0.1, pool_n=0)


# --------------------------------------------------------------------------
# GPU: fo_generate_masks, bit-exact
# --------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("case", list(range(5)))
def test_gpu_policy_matches_reference_fixture(case):
    import paper_2509_25401_b200 as fo

    ci, q, k, cache, skip, kw = list(_cases())[case]
    cb, sb = fo.generate_masks(q, k, b_q=T, b_k=T, **kw)
    assert cb.dtype == bool and cb.shape == cache.shape and sb.shape == skip.shape
    assert np.array_equal(cb, cache), f"case {ci}: cache bits differ"
    assert np.array_equal(sb, skip), f"case {ci}: skip bits differ at {np.argwhere(sb != skip)[:5]}"


@pytest.mark.gpu
@pytest.mark.parametrize("pool_n,n,n_text,heads", [(1, 2304, 256, 4), (2, 2944, 384, 3),
                                                   (3, 2000, 0, 2), (1, 33024, 512, 2),
                                                   (1, 131072, 512, 1)])
def test_gpu_policy_batched_heads_match_oracle(pool_n, n, n_text, heads):
    """All heads in one call equal the oracle run head by head; (1, 33024) is
    the bench workload's sequence (258 x 258 compressed map) and (1, 131072)
    the largest map the kernels take (1024 x 1024: 16 score chunks, 176 KB of
    shared memory per CTA)."""
    import torch

    import paper_2509_25401_b200 as fo

    rng = np.random.default_rng(100 + pool_n + heads)
    q, k = _structured_qk(rng, n, heads)
    kw = dict(pool_n=pool_n, n_text=n_text, tau_q=0.4, tau_kv=0.3, s_q=0.0, guard=True)
    cb, sb = fo.generate_masks_heads(torch.from_numpy(q), torch.from_numpy(k), **kw)
    cb, sb = cb.bool().cpu().numpy(), sb.bool().cpu().numpy()
    for h in range(heads):
        wc, ws = oracle.generate_masks(q[:, h], k[:, h], T, T, **kw)
        assert np.array_equal(cb[h], wc), f"head {h} cache"
        assert np.array_equal(sb[h], ws), f"head {h} skip"


@pytest.mark.gpu
def test_gpu_policy_guard_off_and_degrade():
    import torch

    import paper_2509_25401_b200 as fo

    rng = np.random.default_rng(7)
    q, k = _structured_qk(rng, 1536, 2)
    for kw in (dict(pool_n=1, n_text=0, tau_q=0.3, tau_kv=0.9, s_q=0.0, guard=False),
               dict(pool_n=2, n_text=256, tau_q=0.7, tau_kv=0.2, s_q=0.8, guard=True),
               dict(pool_n=1, n_text=128, tau_q=1.0, tau_kv=1.0, s_q=0.0, guard=False)):
        cb, sb = fo.generate_masks_heads(torch.from_numpy(q), torch.from_numpy(k), **kw)
        cb, sb = cb.bool().cpu().numpy(), sb.bool().cpu().numpy()
        for h in range(2):
            wc, ws = oracle.generate_masks(q[:, h], k[:, h], T, T, **kw)
            assert np.array_equal(cb[h], wc) and np.array_equal(sb[h], ws), (kw, h)


@pytest.mark.gpu
def test_gpu_policy_invariants():
    """reference pkg/tests/test_policy.py:266-295 at b = d = 128."""
    import torch

    import paper_2509_25401_b200 as fo

    rng = np.random.default_rng(16)
    n, n_text = 2048, 256
    q = torch.from_numpy(rng.standard_normal((n, 3, T)).astype(np.float32))
    k = torch.from_numpy(rng.standard_normal((n, 3, T)).astype(np.float32))
    cb, sb = fo.generate_masks_heads(q, k, pool_n=2, n_text=n_text, tau_q=0.6, tau_kv=0.3)
    cb, sb = cb.bool().cpu().numpy(), sb.bool().cpu().numpy()
    t_text = -(-n_text // T)
    for h in range(3):
        assert cb[h, :t_text].all()
        assert np.array_equal(cb[h, 0::2], cb[h, 1::2])
        for i in range(cb.shape[1]):
            if cb[h, i]:
                assert sb[h, i].any() and sb[h, i, :t_text].all()
            else:
                assert not sb[h, i].any()
    cb, sb = fo.generate_masks_heads(q, k, pool_n=1, n_text=128, tau_q=0.0, tau_kv=0.0)
    assert cb.bool().all() and sb.bool().all()


@pytest.mark.gpu
def test_gpu_policy_errors():
    import torch

    import paper_2509_25401_b200 as fo

    q = torch.zeros(512, 1, T)
    with pytest.raises(fo.ParameterError):
        fo.generate_masks_heads(q, q, pool_n=1, n_text=0, tau_q=1.2, tau_kv=0.1)
    with pytest.raises(fo.ParameterError):
        fo.generate_masks_heads(q, q, pool_n=1, n_text=0, tau_q=0.2, tau_kv=float("nan"))
    with pytest.raises(fo.ParameterError):  # text fills every compressed row
        fo.generate_masks_heads(q, q, pool_n=1, n_text=512, tau_q=0.2, tau_kv=0.1)
    # the per-head reference signature runs the policy stages at any block
    # size (policy.py:196-234); with no text both scores are 0, every prefix sum
    # 0 <= tau * 0 holds and the reference caches every block
    cb, sb = fo.generate_masks(np.zeros((512, 64), np.float32), np.zeros((512, 64), np.float32),
                               b_q=64, b_k=64, pool_n=1, n_text=0, tau_q=0.1, tau_kv=0.1)
    assert cb.shape == (8,) and sb.shape == (8, 8) and not cb.any() and not sb.any()
    with pytest.raises(fo.ParameterError):
        fo.generate_masks(np.zeros((512, 64), np.float32), np.zeros((512, 64), np.float32), b_q=64,
                          b_k=32, pool_n=1, n_text=0, tau_q=0.1, tau_kv=0.1)


@pytest.mark.gpu
def test_gpu_update_step_with_policy():
    """update_step(policy=...) derives the next symbols from its own q/k
    exactly as the oracle policy does on those tensors (pipeline.py:254-266)."""
    import torch

    import paper_2509_25401_b200 as fo

    rng = np.random.default_rng(21)
    n, dm, H, order = 1024, 256, 2, 1
    w = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32) * s[-2] ** -0.5)  # noqa: E731
    params = fo.LayerParams.from_reference(w(H, dm, T), w(H, dm, T), w(H, dm, T),
                                           torch.ones(H, T), torch.ones(H, T), w(H, T, dm))
    state = fo.new_layer_state(params, n, order)
    pol = fo.MaskPolicy(n_text=128, tau_q=0.5, tau_kv=0.4, warmup=4)
    x = torch.from_numpy(rng.standard_normal((n, dm)).astype(np.float32)).cuda().bfloat16()
    fo.update_step(state, x, None, order, policy=pol, t=2)
    q = fo.project_q(x, params.w_q, params.q_norm, None, "update", fill=None)
    k, _ = fo.project_kv(x, params)
    qn, kn = q.float().cpu().numpy(), k.float().cpu().numpy()
    got_c, got_s = state.symbols.decoded()
    got_c, got_s = got_c.bool().cpu().numpy(), got_s.bool().cpu().numpy()
    for h in range(H):
        wc, ws = oracle.generate_masks(qn[:, h], kn[:, h], T, T, pool_n=1, n_text=128,
                                       tau_q=0.25, tau_kv=0.2)
        assert np.array_equal(got_c[h], wc)
        assert np.array_equal(got_s[h][wc], ws[wc])  # skip rows of cached blocks are don't-care
