"""The reference's own sparse-attention tests (reference tests/test_attention.py
:180-300, `TestSparseAttention` / `TestBackendAgreement`) restated against this
engine's reference-signature API, at the reference's shapes: head dims 4-16,
blocks of 4-16 tokens, b_q != b_k, per-entry feature caches. These shapes run
the fp32 tile kernel (fo_masked_block_attention_f32), so the reference's
float32 tolerance (rel err < 1e-5) holds; 128-token blocks take the tcgen05
kernel and are covered elsewhere at the bf16 tolerance.

The oracle (fp64 brute-force masked softmax, verify.py:47-65, and the fp32
pyref kernel restated) is the checker.
"""

import numpy as np
import pytest

import oracle
from conftest import rel_err

pytestmark = pytest.mark.gpu


def fo():
    import paper_2509_25401_b200 as m

    return m


def rand_qkv(rng, n, d):
    return tuple(rng.standard_normal((n, d)).astype(np.float32) for _ in range(3))


def all_active(m, t_q, t_kv, pool_n=1):
    return m.build_symbols(np.ones(t_q, bool), np.ones((t_q, t_kv), bool), pool_n)


def dense(q, k, v):
    s = q.astype(np.float64) @ k.astype(np.float64).T / np.sqrt(q.shape[1])
    s -= s.max(axis=1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=1, keepdims=True)
    return (p @ v.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("n,d,b", [(32, 8, 8), (64, 16, 16), (48, 8, 16)])
def test_dense_equivalence(n, d, b):
    m = fo()
    q, k, v = rand_qkv(np.random.default_rng(10), n, d)
    sym = all_active(m, -(-n // b), -(-n // b))
    got = m.sparse_attention(q, k, v, sym, None, 0, 0, 1, 0, b_q=b, b_k=b)
    assert rel_err(got, dense(q, k, v)) < 1e-5


def test_full_cache_forecast_only():
    m = fo()
    rng = np.random.default_rng(11)
    n, d, b = 32, 8, 8
    q, k, v = rand_qkv(rng, n, d)
    t_q = n // b
    cache = m.FeatureCache(1, t_q, order=1)  # no seq: per-entry stacks
    stored = rng.standard_normal((n, d)).astype(np.float32)
    for i in range(t_q):
        cache.update(0, i, stored[i * b:(i + 1) * b])
    sym = m.build_symbols(np.zeros(t_q, bool), np.zeros((t_q, t_q), bool), 1)
    ac = m.AttnCounters()
    out = m.sparse_attention(q, k, v, sym, cache, 0, 1, 4, 1, b_q=b, b_k=b, counters=ac)
    assert ac.pairs_computed == 0
    for i in range(t_q):  # cached tiles are bit-identical to the forecast
        want = m.forecast(cache.entry(0, i), 1, 4, 1)
        assert np.array_equal(out[i * b:(i + 1) * b], want)
        # and to the oracle's restatement of the stack arithmetic
        st, val = oracle.update_entry(None, 0, stored[i * b:(i + 1) * b], 1)
        np.testing.assert_allclose(want, oracle.forecast(st, val, 1, 4, 1), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("pool_n", [1, 2])
def test_masked_oracle_and_skip_accounting(pool_n):
    m = fo()
    rng = np.random.default_rng(12 + pool_n)
    n, d, b_q, b_k = 128, 8, 16, 16
    t_q, t_kv = n // b_q, n // b_k
    for _ in range(10):
        q, k, v = rand_qkv(rng, n, d)
        cache_bits, skip_bits = oracle.random_masks(rng, t_q, t_kv, pool_n)
        sym = m.build_symbols(cache_bits, skip_bits, pool_n)
        cache = m.FeatureCache(1, t_q, order=0)
        for i in range(t_q):
            cache.update(0, i, v[i * b_q:(i + 1) * b_q])
        ac = m.AttnCounters()
        got = m.sparse_attention(q, k, v, sym, cache, 0, 1, 2, 0, b_q=b_q, b_k=b_k, mode="bias",
                                 fill=np.nan, counters=ac)
        want = oracle.masked_attention(q, k, v, cache_bits, skip_bits, b_q, b_k)
        rows = np.repeat(cache_bits, b_q)
        assert rel_err(got[rows], want[rows]) < 1e-5
        assert np.isnan(got[~rows]).all()  # cached tiles stay untouched in bias mode
        assert ac.pairs_computed == int(skip_bits[cache_bits].sum())
        assert ac.pairs_total == t_q * t_kv


def test_unequal_blocks_and_materialize():
    """b_q != b_k (the reference allows it; the tcgen05 path does not) with
    materialized forecasts for the cached blocks."""
    m = fo()
    rng = np.random.default_rng(21)
    n, d, b_q, b_k = 96, 16, 16, 8
    t_q, t_kv = n // b_q, n // b_k
    q, k, v = rand_qkv(rng, n, d)
    cache_bits, skip_bits = oracle.random_masks(rng, t_q, t_kv, 1)
    cache = m.FeatureCache(1, t_q, order=2)
    for rep in range(3):
        for i in range(t_q):
            cache.update(0, i, v[i * b_q:(i + 1) * b_q] * (1 + rep))
    sym = m.build_symbols(cache_bits, skip_bits, 1)
    got = m.sparse_attention(q, k, v, sym, cache, 0, 2, 6, 2, b_q=b_q, b_k=b_k)
    want = oracle.masked_attention(q, k, v, cache_bits, skip_bits, b_q, b_k)
    rows = np.repeat(cache_bits, b_q)
    assert rel_err(got[rows], want[rows]) < 1e-5
    for i in np.flatnonzero(~cache_bits):
        assert np.array_equal(got[i * b_q:(i + 1) * b_q], m.forecast(cache.entry(0, i), 2, 6, 2))


def test_partial_trailing_blocks():
    m = fo()
    n, d, b = 52, 8, 16  # 4 blocks, the last has 4 rows
    q, k, v = rand_qkv(np.random.default_rng(14), n, d)
    t = -(-n // b)
    got = m.sparse_attention(q, k, v, all_active(m, t, t), None, 0, 0, 1, 0, b_q=b, b_k=b)
    assert rel_err(got, dense(q, k, v)) < 1e-5


def test_all_skipped_active_row_rejected():
    m = fo()
    q, k, v = rand_qkv(np.random.default_rng(15), 16, 4)
    skip_bits = np.ones((4, 4), bool)
    skip_bits[2] = False
    sym = m.build_symbols(np.ones(4, bool), skip_bits, 1)
    with pytest.raises(m.ConsistencyError):
        m.sparse_attention(q, k, v, sym, None, 0, 0, 1, 0, b_q=4, b_k=4)


def test_cold_cache_rejected():
    m = fo()
    q, k, v = rand_qkv(np.random.default_rng(16), 16, 4)
    cache_bits = np.array([True, False, True, True])
    skip_bits = np.ones((4, 4), bool)
    skip_bits[1] = False
    sym = m.build_symbols(cache_bits, skip_bits, 1)
    with pytest.raises(m.StateError):
        m.sparse_attention(q, k, v, sym, m.FeatureCache(1, 4, order=0), 0, 1, 2, 0, b_q=4, b_k=4)


def test_nonfinite_inputs_rejected_in_reference_order():
    m = fo()
    q, k, v = rand_qkv(np.random.default_rng(18), 16, 4)
    sym = all_active(m, 4, 4)
    bad = k.copy()
    bad[3, 1] = np.nan
    with pytest.raises(m.ParameterError):
        m.sparse_attention(q, bad, v, sym, None, 0, 0, 1, 0, b_q=4, b_k=4)
    # q rows of cached blocks may hold placeholders; only active rows are read
    cache = m.FeatureCache(1, 4, order=0)
    for i in range(4):
        cache.update(0, i, v[i * 4:(i + 1) * 4])
    cache_bits = np.array([True, False, True, True])
    skip_bits = np.ones((4, 4), bool)
    skip_bits[1] = False
    qn = q.copy()
    qn[4:8] = np.nan
    out = m.sparse_attention(qn, k, v, m.build_symbols(cache_bits, skip_bits, 1), cache, 0, 1, 2, 0,
                             b_q=4, b_k=4)
    assert np.isfinite(out).all()
    qn[0, 0] = np.inf
    with pytest.raises(m.ParameterError):
        m.sparse_attention(qn, k, v, m.build_symbols(cache_bits, skip_bits, 1), cache, 0, 1, 2, 0,
                           b_q=4, b_k=4)


def test_backend_matches_oracle_kernel():
    """TestBackendAgreement: the b200 backend's masked_block_attention against
    the reference CPU kernel (restated in the oracle) at b = 16, d = 16."""
    from paper_2509_25401_b200._kernels import b200

    rng = np.random.default_rng(17)
    n, d, b = 96, 16, 16
    t = n // b
    q, k, v = rand_qkv(rng, n, d)
    cache_bits, skip_bits = oracle.random_masks(rng, t, t, 1)
    got, want = np.zeros((n, d), np.float32), np.zeros((n, d), np.float32)
    pg = b200.masked_block_attention(q, k, v, cache_bits.astype(np.uint8),
                                     skip_bits.astype(np.uint8), b, b, 1.0 / np.sqrt(d), got)
    pw = oracle.masked_block_attention(q, k, v, cache_bits.astype(np.uint8),
                                       skip_bits.astype(np.uint8), b, b, 1.0 / np.sqrt(d), want)
    assert pg == pw
    rows = np.repeat(cache_bits, b)
    assert rel_err(got[rows], want[rows]) < 1e-5
    assert not got[~rows].any()  # rows of cached blocks are not written


@pytest.mark.parametrize("d", [3, 40, 100, 200])
def test_general_head_dims(d):
    """Head dims off the power-of-two grid and past 128 (the kernel pads to
    16/32/64/128/256 columns in registers)."""
    m = fo()
    n, b = 80, 16
    q, k, v = rand_qkv(np.random.default_rng(d), n, d)
    t = n // b
    got = m.sparse_attention(q, k, v, all_active(m, t, t), None, 0, 0, 1, 0, b_q=b, b_k=b)
    assert rel_err(got, dense(q, k, v)) < 1e-5
