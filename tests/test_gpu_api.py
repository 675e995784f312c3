"""GPU parity of the reference's tile-level and policy building blocks
(attention.py:21-113, policy.py:21-178, tensor.py:33-126) against outputs of
the reference itself (tests/golden/api.npz, oracle/gen_golden.py api).

Where the reference's arithmetic order is fixed by numpy (sequential and
pairwise sums, single-rounded float32 ops) the device result must be
bit-exact: update_entry, forecast, mean_pool_blocks, rms_norm, rope, the
policy stages fed the reference's own intermediate values, and every mask
decision. Where it is BLAS- or libm-defined (p @ v, exp, float64 GEMMs) the
bar is the reference tests' own 1e-5 relative tolerance
(tests/test_attention.py:181-189) or a few float32 ulps."""

import numpy as np
import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu
G = np.load(ROOT / "tests" / "golden" / "api.npz")


def fo():
    import paper_2509_25401_b200 as m

    return m


def ulps(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    return int(np.abs(a - b).max()) if a.size else 0


def test_online_softmax_update_and_finalize():
    m = fo()
    st = m.OnlineSoftmaxState.fresh(24, 16)
    for b in range(3):
        st = m.online_softmax_update(st, G[f"os{b}_scores"], G[f"os{b}_v"])
        assert isinstance(st.m, np.ndarray)
        np.testing.assert_array_equal(st.m, G[f"os{b}_m"])  # max: exact
        np.testing.assert_allclose(st.l, G[f"os{b}_l"], rtol=1e-5)
        np.testing.assert_allclose(st.acc, G[f"os{b}_acc"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(m.online_softmax_finalize(st), G["os_final"], rtol=1e-5, atol=1e-6)
    # device-resident state stays on the device
    dev = m.OnlineSoftmaxState(*(torch.as_tensor(a).cuda() for a in
                                 (G["os0_m"], G["os0_l"], G["os0_acc"])))
    nxt = m.online_softmax_update(dev, torch.as_tensor(G["os1_scores"]).cuda(),
                                  torch.as_tensor(G["os1_v"]).cuda())
    assert nxt.acc.is_cuda
    np.testing.assert_allclose(nxt.acc.cpu().numpy(), G["os1_acc"], rtol=1e-5, atol=1e-5)


def test_online_softmax_finalize_empty_row_raises():
    m = fo()
    st = m.OnlineSoftmaxState.fresh(4, 8)
    with pytest.raises(m.ConsistencyError):
        m.online_softmax_finalize(st)
    # the status word is clean afterwards
    st.l[:] = 1.0
    np.testing.assert_array_equal(m.online_softmax_finalize(st), np.zeros((4, 8), np.float32))


def test_update_entry_and_forecast_bit_exact():
    m = fo()
    e = None
    for t in range(4):
        e = m.update_entry(e, G[f"ue{t}_o"], 2)
        np.testing.assert_array_equal(e.diff_stack, G[f"ue{t}_stack"])
        assert e.valid_orders == int(G[f"ue{t}_valid"])
        for k, n in ((1, 4), (3, 6)):
            for od in (0, 1, 2):
                np.testing.assert_array_equal(m.forecast(e, k, n, od), G[f"ue{t}_fc_{k}_{n}_{od}"])


def test_forecast_error_order():
    m = fo()
    with pytest.raises(m.StateError):
        m.forecast(None, 0, 4, 1)  # cold entry first, even with a bad elapsed_k
    e = m.update_entry(None, np.ones((4, 4), np.float32), 1)
    with pytest.raises(m.ParameterError):
        m.forecast(e, 0, 4, 1)
    with pytest.raises(m.ParameterError):
        m.forecast(e, 4, 4, 1)
    with pytest.raises(m.ShapeError):
        m.update_entry(e, np.ones((4, 5), np.float32), 1)
    with pytest.raises(m.ParameterError):
        m.update_entry(None, np.full((2, 2), np.nan, np.float32), 1)


def test_tensor_numerics():
    m = fo()
    x, w = G["t_x"], G["t_w"]
    np.testing.assert_array_equal(m.rms_norm(x, w), G["t_rms"])
    np.testing.assert_array_equal(m.rope(x, G["t_pos"]), G["t_rope"])
    np.testing.assert_array_equal(m.rope(x[3], 7.0), G["t_rope_vec"])
    for pool in (1, 4, 7, 64):
        np.testing.assert_array_equal(m.mean_pool_blocks(x, pool), G[f"t_pool{pool}"])
    assert ulps(m.row_softmax(x), G["t_softmax"]) <= 1
    assert ulps(m.matmul(G["t_a"], G["t_b"]), G["t_matmul"]) <= 1
    np.testing.assert_allclose(m.dense_attention(G["t_q"], G["t_k"], G["t_v"]), G["t_dense_attn"],
                               rtol=1e-5, atol=1e-6)
    # torch in -> torch out, on the device
    xt = torch.as_tensor(x).cuda()
    r = m.rms_norm(xt, torch.as_tensor(w).cuda())
    assert r.is_cuda and np.array_equal(r.cpu().numpy(), G["t_rms"])
    with pytest.raises(m.ParameterError):
        m.mean_pool_blocks(x, 0)
    with pytest.raises(m.ShapeError):
        m.rope(x[:, :5], G["t_pos"])
    with pytest.raises(m.ShapeError):
        m.matmul(G["t_a"], G["t_a"])


def _case(ci):
    n, dd, pq, pk, n_text = (int(v) for v in G[f"p{ci}_cfg"])
    return n, dd, pq, pk, n_text


@pytest.mark.parametrize("ci", range(5))
def test_policy_stages_match_reference(ci):
    m = fo()
    n, dd, pq, pk, n_text = _case(ci)
    q, k = G[f"p{ci}_q"], G[f"p{ci}_k"]
    cm = m.compressed_attention(q, k, pq, pk, n_text)
    assert cm.n_t == int(G[f"p{ci}_nt"])
    assert cm.p_tilde.shape == G[f"p{ci}_map"].shape
    assert ulps(cm.p_tilde, G[f"p{ci}_map"]) <= 2
    # each stage fed the reference's own map: bit-exact
    ref_map = m.CompressedAttnMap(p_tilde=G[f"p{ci}_map"], n_t=int(G[f"p{ci}_nt"]))
    c = m.vision_to_text_contribution(ref_map)
    g = m.text_to_vision_guidance(ref_map)
    np.testing.assert_array_equal(c, G[f"p{ci}_contrib"])
    np.testing.assert_array_equal(g, G[f"p{ci}_guid"])
    rows, cols = ref_map.p_tilde.shape
    for ti, tau in enumerate((0.0, 0.3, 0.7, 1.0)):
        if rows == cols:
            got = m.select_cached_blocks(G[f"p{ci}_contrib"], G[f"p{ci}_guid"], tau)
            np.testing.assert_array_equal(got, G[f"p{ci}_cached{ti}"])
        cbits = G[f"p{ci}_cbits{ti}"]
        for guard in (True, False):
            keep = m.select_skip_blocks(ref_map, cbits, tau * 0.6, guard=guard)
            np.testing.assert_array_equal(keep, G[f"p{ci}_keep{ti}_{int(guard)}"])
        np.testing.assert_array_equal(m.degrade_to_full_cache(cbits, ref_map.n_t, 0.25 * ti),
                                      G[f"p{ci}_degrade{ti}"])


@pytest.mark.parametrize("ci", [0, 1, 3, 4])
def test_generate_masks_float32_bit_exact(ci):
    """The per-head reference signature on float32 q/k (not bf16-rounded),
    small d and blocks: every decision equals the reference's."""
    m = fo()
    n, dd, pq, pk, n_text = _case(ci)
    for gi in range(3):
        tq, tkv, sq, guard = G[f"p{ci}_gm{gi}_cfg"]
        cb, sb = m.generate_masks(G[f"p{ci}_q"], G[f"p{ci}_k"], b_q=pq, b_k=pk, pool_n=1,
                                  n_text=n_text, tau_q=float(tq), tau_kv=float(tkv), s_q=float(sq),
                                  guard=bool(guard))
        np.testing.assert_array_equal(cb, G[f"p{ci}_gm{gi}_cache"])
        np.testing.assert_array_equal(sb, G[f"p{ci}_gm{gi}_skip"])


def test_policy_stage_errors():
    m = fo()
    p = np.full((4, 4), 0.25, np.float32)
    with pytest.raises(m.ParameterError):
        m.CompressedAttnMap(p_tilde=p, n_t=4)
    with pytest.raises(m.ParameterError):
        m.CompressedAttnMap(p_tilde=p * 2, n_t=0)
    with pytest.raises(m.ShapeError):
        m.select_cached_blocks(np.ones(3), np.ones(4), 0.5)
    with pytest.raises(m.ParameterError):
        m.select_cached_blocks(np.ones(3), np.ones(3), 1.5)
    cm = m.CompressedAttnMap(p_tilde=p, n_t=1)
    with pytest.raises(m.ShapeError):
        m.select_skip_blocks(cm, np.ones(3, bool), 0.5)
    with pytest.raises(m.ParameterError):
        m.select_skip_blocks(cm, np.ones(4, bool), -0.1)
    with pytest.raises(m.ParameterError):
        m.degrade_to_full_cache(np.ones(4, bool), 1, 2.0)
    q = np.random.default_rng(0).standard_normal((64, 8)).astype(np.float32)
    with pytest.raises(m.ParameterError):  # non-square map
        m.generate_masks(q, q, b_q=8, b_k=4, pool_n=1, n_text=0, tau_q=0.5, tau_kv=0.5)


def test_feature_cache_update_tile_sized():
    """FeatureCache.update pushes one tile with one tile-sized launch and
    leaves every other entry alone; the entry matches update_entry (bf16
    storage: the reference stack of the bf16-rounded tiles, within bf16)."""
    m = fo()
    S, H, order = 300, 3, 2
    t = -(-S // 128)
    fc = m.FeatureCache(H, t, order, seq=S)
    base = torch.randn(S, H, 128, device="cuda").bfloat16()
    fc.push(base)
    before = fc.stacks.clone()
    rng = np.random.default_rng(5)
    e = m.update_entry(None, base[256:300, 1].float().cpu().numpy(), order)
    for _ in range(3):
        tile = rng.standard_normal((44, 128)).astype(np.float32)
        tile = torch.as_tensor(tile).bfloat16().float().numpy()
        fc.update(1, 2, tile)
        e = m.update_entry(e, tile, order)
    got = fc.entry(1, 2)
    assert got.valid_orders == e.valid_orders == 3
    np.testing.assert_allclose(got.diff_stack, e.diff_stack, rtol=2e-2, atol=3e-2)
    diff = (fc.stacks != before)
    diff[:, 256:300, 128:256] = False
    assert not bool(diff.any())
    assert fc.valid_orders(0, 2) == 1 and fc.valid_orders(1, 1) == 1
    with pytest.raises(IndexError):
        fc.update(3, 0, np.zeros((128, 128), np.float32))
    with pytest.raises(m.ShapeError):
        fc.update(0, 0, np.zeros((44, 128), np.float32))


# ---------------------------------------------------------------------------
# The reference's known-answer properties of the cache and the forecast
# (test_attention.py:85-160, test_acceptance.py:235-253), on the
# device update_entry / forecast / FeatureCache.
# ---------------------------------------------------------------------------
def test_forecast_affine_trajectories_exact():
    m = fo()
    rng = np.random.default_rng(7)
    for _ in range(20):
        a = rng.standard_normal((8, 16)).astype(np.float32)
        b = (0.2 * rng.standard_normal((8, 16))).astype(np.float32)
        n = int(rng.integers(2, 8))
        f = lambda t: (a + t * b).astype(np.float32)  # noqa: E731
        e = m.update_entry(m.update_entry(None, f(0), 1), f(n), 1)
        for k in range(1, n):
            got = m.forecast(e, k, n, 1)
            assert np.abs(got - f(n + k)).max() / np.abs(f(n + k)).max() < 1e-5
        const = m.update_entry(None, a, 0)  # order 0: exact reuse after one update
        np.testing.assert_array_equal(m.forecast(const, 1, n, 0), a)


def test_quadratic_second_difference_and_repeats():
    m = fo()
    rng = np.random.default_rng(5)
    a, b, c = (rng.standard_normal((4, 8)).astype(np.float32) for _ in range(3))
    f = lambda t: (a + t * b + t * t * c).astype(np.float32)  # noqa: E731
    e = None
    for t in (0, 1, 2):
        e = m.update_entry(e, f(t), 2)
    assert e.valid_orders == 3
    np.testing.assert_allclose(e.diff_stack[2], 2 * c, atol=1e-5)
    o = rng.standard_normal((4, 8)).astype(np.float32)
    e2 = m.update_entry(m.update_entry(None, o, 1), o, 1)  # a repeated tile: zero difference
    assert e2.valid_orders == 2 and not e2.diff_stack[1].any()


def test_forecast_hand_coefficients_and_exact_linearity():
    m = fo()
    assert m.forecast_coefficients(2, 4, 2).tolist() == [1.0, 0.5]
    s0 = np.full((2, 2), 4.0, np.float32)
    s1 = np.full((2, 2), 2.0, np.float32)
    e = m.update_entry(m.update_entry(None, s0 - s1, 1), s0, 1)
    np.testing.assert_array_equal(e.diff_stack[0], s0)
    np.testing.assert_array_equal(e.diff_stack[1], s1)
    np.testing.assert_array_equal(m.forecast(e, 2, 4, 1), s0 + 0.5 * s1)
    # coefficients 1, 1/2, 1/8 and small-integer stacks: every operation exact
    rng = np.random.default_rng(9)
    ints = lambda: rng.integers(-8, 9, (3, 4)).astype(np.float32)  # noqa: E731
    s_a, s_b = [ints() for _ in range(3)], [ints() for _ in range(3)]
    entry = lambda st: m.CacheEntry(diff_stack=np.stack(st), valid_orders=3)  # noqa: E731
    lhs = m.forecast(entry([3.0 * x + 5.0 * y for x, y in zip(s_a, s_b)]), 2, 4, 2)
    rhs = 3.0 * m.forecast(entry(s_a), 2, 4, 2) + 5.0 * m.forecast(entry(s_b), 2, 4, 2)
    np.testing.assert_array_equal(lhs, rhs)


def test_feature_cache_valid_order_counting():
    """FeatureCache.update on the device counts valid orders as the reference
    (test_attention.py:101-106): min(updates, order + 1)."""
    m = fo()
    cache = m.FeatureCache(1, 1, 2, seq=128)
    rng = np.random.default_rng(6)
    for u in range(1, 6):
        cache.update(0, 0, rng.standard_normal((128, 128)).astype(np.float32))
        assert cache.valid_orders(0, 0) == min(u, 3)
