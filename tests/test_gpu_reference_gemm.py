"""The reference's own GEMM tests (reference tests/test_gemm.py) restated
against this engine's reference-signature GEMMs: numpy in / out, head-major o,
one SymbolBuffer per head, d_model 24, head dim 8, blocks of 4-8 tokens. These
run gemm_ref (fo_matmul_f32 plus the device RMS norm / RoPE kernels) and are
held to the reference's float32 tolerances; the oracle restatement of
gemm.py:44-229 is the checker. Bit-exactness against numpy's BLAS is not
claimed (its float32 summation order is not fixed).
"""

import numpy as np
import pytest

import oracle
from conftest import rel_err

pytestmark = pytest.mark.gpu


def fo():
    import paper_2509_25401_b200 as m

    return m


def head_symbols(m, active_per_head, t_kv, pool_n=1):
    """active_per_head: bool [t_q, heads]."""
    t_q, heads = active_per_head.shape
    return [m.build_symbols(active_per_head[:, h], np.ones((t_q, t_kv), bool), pool_n)
            for h in range(heads)]


def make_model(rng, heads, d_model, d):
    w_q = (rng.standard_normal((heads, d_model, d)) * d_model ** -0.5).astype(np.float32)
    norm = (1.0 + 0.05 * rng.standard_normal((heads, d))).astype(np.float32)
    w_out = (rng.standard_normal((heads, d, d_model)) * d ** -0.5).astype(np.float32)
    return w_q, norm, w_out


def warm_cache(m, rng, heads, t_q, b_q, n, d, order, updates):
    cache = m.FeatureCache(heads, t_q, order)  # per-entry stacks (no seq)
    host = [[None] * t_q for _ in range(heads)]  # the oracle's copy
    valid = np.zeros((heads, t_q), int)
    tiles = []
    for _ in range(updates):
        o = rng.standard_normal((heads, n, d)).astype(np.float32)
        tiles.append(o)
        for h in range(heads):
            for i in range(t_q):
                tile = o[h, i * b_q:min((i + 1) * b_q, n)]
                cache.update(h, i, tile)
                host[h][i], valid[h, i] = oracle.update_entry(host[h][i], valid[h, i], tile, order)
    return cache, tiles, host, valid


def test_project_q_update_matches_oracle():
    m = fo()
    rng = np.random.default_rng(0)
    n, dm, d, heads, b_q = 32, 24, 8, 2, 8
    x = rng.standard_normal((n, dm)).astype(np.float32)
    w_q, norm, _ = make_model(rng, heads, dm, d)
    got = m.project_q(x, w_q, norm, None, "update", b_q=b_q, positions=np.arange(n))
    want = oracle.project_q(x, w_q, norm, None, b_q)
    assert got.shape == (heads, n, d)
    assert rel_err(got, want) < 1e-5


def test_project_q_all_cached_dispatch_zero_macs():
    m = fo()
    rng = np.random.default_rng(1)
    n, dm, d, heads, b_q = 32, 24, 8, 2, 8
    x = rng.standard_normal((n, dm)).astype(np.float32)
    w_q, norm, _ = make_model(rng, heads, dm, d)
    syms = head_symbols(m, np.zeros((4, heads), bool), 4)
    gc = m.GemmCounters()
    got = m.project_q(x, w_q, norm, syms, "dispatch", b_q=b_q, counters=gc, fill=np.nan)
    assert gc.q_macs_actual == 0
    assert np.isnan(got).all()


def test_project_q_active_rows_match_update_rows():
    m = fo()
    rng = np.random.default_rng(2)
    n, dm, d, heads, b_q = 40, 24, 8, 3, 8
    t_q = n // b_q
    x = rng.standard_normal((n, dm)).astype(np.float32)
    w_q, norm, _ = make_model(rng, heads, dm, d)
    active = rng.random((t_q, heads)) < 0.6
    pos = np.arange(n) + 7
    gc = m.GemmCounters()
    got = m.project_q(x, w_q, norm, head_symbols(m, active, t_q), "dispatch", b_q=b_q,
                      positions=pos, counters=gc, fill=np.nan)
    ref = m.project_q(x, w_q, norm, None, "update", b_q=b_q, positions=pos)
    want = oracle.project_q(x, w_q, norm, active.T, b_q, positions=pos, fill=np.nan)
    rows_active = 0
    for h in range(heads):
        rows = np.repeat(active[:, h], b_q)
        rows_active += int(rows.sum())
        assert np.array_equal(got[h, rows], ref[h, rows])  # the same rows, bit for bit
        assert rel_err(got[h, rows], want[h, rows]) < 1e-5
        assert np.isnan(got[h, ~rows]).all()
    assert gc.q_macs_actual == rows_active * dm * d
    assert gc.q_macs_dense == heads * n * dm * d


def test_project_out_update_all_active_is_dense():
    m = fo()
    rng = np.random.default_rng(3)
    n, d, dm, heads, b_q = 32, 8, 24, 4, 8
    t_q = n // b_q
    _, _, w_out = make_model(rng, heads, dm, d)
    cache, _, _, _ = warm_cache(m, rng, heads, t_q, b_q, n, d, 1, 1)
    o = rng.standard_normal((heads, n, d)).astype(np.float32)
    out, bias = m.project_out_update(o, w_out, head_symbols(m, np.ones((t_q, heads), bool), t_q),
                                     cache, 1, b_q=b_q)
    ref = sum(o[h].astype(np.float64) @ w_out[h].astype(np.float64) for h in range(heads))
    assert rel_err(out, ref) < 1e-5
    assert all(s.shape[0] == 0 for s in bias.stacks)


@pytest.mark.parametrize("order", [0, 1, 2])
def test_project_out_update_and_dispatch_match_oracle(order):
    """Bias stacks, orders and both outputs against the oracle, then the
    dispatch against the materialized-forecast oracle (test_gemm.py:146-249)."""
    m = fo()
    rng = np.random.default_rng(10 + order)
    n, d, dm, heads, b_q, interval = 36, 8, 24, 4, 8, 5  # ragged last block
    t_q = -(-n // b_q)
    _, _, w_out = make_model(rng, heads, dm, d)
    cache, _, host, valid = warm_cache(m, rng, heads, t_q, b_q, n, d, order, order + 2)
    o = rng.standard_normal((heads, n, d)).astype(np.float32)
    for _ in range(3):
        active = rng.random((t_q, heads)) < 0.5
        syms = head_symbols(m, active, t_q)
        gc = m.GemmCounters()
        out, bias = m.project_out_update(o, w_out, syms, cache, order, b_q=b_q, counters=gc)
        assert gc.o_macs_actual == gc.o_macs_dense == heads * n * d * dm
        w_out_ref, b_ref, ord_ref = oracle.project_out_update(o, w_out, active, host, valid, order,
                                                              b_q)
        np.testing.assert_array_equal(bias.orders, ord_ref)
        np.testing.assert_array_equal(bias.active_heads, active)
        assert rel_err(out, w_out_ref) < 1e-5
        for i in range(t_q):
            assert bias.stacks[i].shape == b_ref[i].shape
            if b_ref[i].size:
                assert rel_err(bias.stacks[i], b_ref[i]) < 1e-5
        elapsed = 1 + int(rng.integers(interval - 1))
        gc = m.GemmCounters()
        got = m.project_out_dispatch(o, w_out, syms, bias, elapsed, interval, order, b_q=b_q,
                                     counters=gc)
        rows = sum(min(b_q, n - i * b_q) * int(active[i].sum()) for i in range(t_q))
        assert gc.o_macs_actual == rows * d * dm
        want = oracle.project_out_dispatch(o, w_out, active, b_ref, ord_ref, elapsed, interval,
                                           order, b_q)
        assert rel_err(got, want) < 1e-5
        # against the materialized forecast (every cached tile forecast, then dense)
        full = o.astype(np.float64).copy()
        for h in range(heads):
            for i in range(t_q):
                if not active[i, h]:
                    r = slice(i * b_q, min((i + 1) * b_q, n))
                    full[h, r] = oracle.forecast(host[h][i], valid[h, i], elapsed, interval, order)
        ref = sum(full[h] @ w_out[h].astype(np.float64) for h in range(heads))
        assert rel_err(got, ref) < 1e-4


def test_all_cached_order_zero_pure_reuse():
    m = fo()
    rng = np.random.default_rng(9)
    n, d, dm, heads, b_q = 32, 8, 24, 2, 8
    t_q = n // b_q
    _, _, w_out = make_model(rng, heads, dm, d)
    cache, _, _, _ = warm_cache(m, rng, heads, t_q, b_q, n, d, 0, 1)
    o = rng.standard_normal((heads, n, d)).astype(np.float32)
    syms = head_symbols(m, np.zeros((t_q, heads), bool), t_q)
    _, bias = m.project_out_update(o, w_out, syms, cache, 0, b_q=b_q)
    gc = m.GemmCounters()
    got = m.project_out_dispatch(o, w_out, syms, bias, 1, 4, 0, b_q=b_q, counters=gc)
    assert gc.o_macs_actual == 0
    for i in range(t_q):
        assert np.array_equal(got[i * b_q:(i + 1) * b_q], bias.stacks[i][0])


def test_errors_in_reference_order():
    m = fo()
    rng = np.random.default_rng(13)
    n, d, dm, heads, b_q = 16, 4, 8, 2, 4
    t_q = n // b_q
    _, _, w_out = make_model(rng, heads, dm, d)
    o = rng.standard_normal((heads, n, d)).astype(np.float32)
    syms = head_symbols(m, np.zeros((t_q, heads), bool), t_q)
    with pytest.raises(m.StateError):  # cold cache
        m.project_out_update(o, w_out, syms, m.FeatureCache(heads, t_q, 1), 1, b_q=b_q)
    cache, _, _, _ = warm_cache(m, rng, heads, t_q, b_q, n, d, 1, 2)
    active = rng.random((t_q, heads)) < 0.5
    _, bias = m.project_out_update(o, w_out, head_symbols(m, active, t_q), cache, 1, b_q=b_q)
    with pytest.raises(m.StateError):  # stale symbols
        m.project_out_dispatch(o, w_out, head_symbols(m, ~active, t_q), bias, 1, 4, 1, b_q=b_q)
    with pytest.raises(m.StateError):  # missing bias
        m.project_out_dispatch(o, w_out, head_symbols(m, active, t_q), None, 1, 4, 1, b_q=b_q)
    with pytest.raises(m.ParameterError):  # elapsed_k outside [1, N-1]
        m.project_out_dispatch(o, w_out, head_symbols(m, active, t_q), bias, 4, 4, 1, b_q=b_q)
    x = rng.standard_normal((n, dm)).astype(np.float32)
    w_q, norm, _ = make_model(rng, heads, dm, d)
    with pytest.raises(m.ParameterError):
        m.project_q(x, w_q, norm, None, "sideways", b_q=b_q)
    x[3, 1] = np.inf
    with pytest.raises(m.ParameterError):
        m.project_q(x, w_q, norm, None, "update", b_q=b_q)


def test_matmul_f32_against_float64():
    """fo_matmul_f32 at ragged sizes, with and without accumulation."""
    import torch

    from paper_2509_25401_b200 import _lib
    from paper_2509_25401_b200._runtime import stream_ptr

    rng = np.random.default_rng(31)
    for mm, nn, kk in [(1, 1, 1), (7, 130, 33), (129, 65, 200), (64, 64, 16)]:
        a = rng.standard_normal((mm, kk)).astype(np.float32)
        b = rng.standard_normal((kk, nn)).astype(np.float32)
        c0 = rng.standard_normal((mm, nn)).astype(np.float32)
        ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        for acc in (0, 1):
            c = torch.from_numpy(c0.copy()).cuda()
            _lib.call("fo_matmul_f32", ad.data_ptr(), bd.data_ptr(), c.data_ptr(), mm, nn, kk,
                      acc, stream_ptr(None))
            want = a.astype(np.float64) @ b.astype(np.float64) + (c0 if acc else 0)
            assert rel_err(c.cpu().numpy(), want) < 1e-5
