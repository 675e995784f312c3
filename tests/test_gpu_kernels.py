"""GPU parity of every sm_100a kernel against fp32/fp64 references of the same op.

The references here are plain torch float64 restatements (for the floating
point kernels) and numpy packbits (for the codec); the oracle/ package and the
reference-generated golden fixtures are checked in test_gpu_parity.py.
"""

import math

import numpy as np
import pytest
import torch

from conftest import assert_bf16_close

pytestmark = pytest.mark.gpu

T = 128


def fo():
    import paper_2509_25401_b200 as m

    return m


def rand_masks(rng, heads, t, cached_ratio=0.25, skip_ratio=0.5):
    """Random valid masks in the reference's random_masks rule (verify.py:29-44)."""
    cache = rng.random((heads, t)) >= cached_ratio
    skip = rng.random((heads, t, t)) >= skip_ratio
    for h in range(heads):
        if not cache[h].any():
            cache[h, rng.integers(t)] = True
        for r in range(t):
            if cache[h, r] and not skip[h, r].any():
                skip[h, r, rng.integers(t)] = True
            if not cache[h, r]:
                skip[h, r] = False
    return cache, skip


def torch_masked_attention(q, k, v, cache, skip):
    """float64 softmax over exactly the allowed key blocks; cached rows NaN."""
    S, H, D = q.shape
    out = torch.full((S, H, D), float("nan"), dtype=torch.float64, device=q.device)
    for h in range(H):
        qh, kh, vh = (a[:, h].double() for a in (q, k, v))
        s = (qh @ kh.T) / math.sqrt(D)
        mask = torch.from_numpy(np.repeat(np.repeat(skip[h], T, 0), T, 1)[:S, :S]).to(q.device)
        s = s.masked_fill(~mask, float("-inf"))
        rows = torch.from_numpy(np.repeat(cache[h], T)[:S]).to(q.device)
        p = torch.softmax(s[rows], dim=1)
        out[rows, h] = p @ vh
    return out


@pytest.mark.parametrize("pool_n", [1, 2, 3])
def test_codec_roundtrip_device(pool_n):
    m = fo()
    rng = np.random.default_rng(pool_n)
    heads, rows, cols = 3, 37, 29
    comp_r, comp_c = -(-rows // pool_n), -(-cols // pool_n)
    cc = rng.random((heads, comp_r)) < 0.7
    ss = rng.random((heads, comp_r, comp_c)) < 0.5
    cache = np.repeat(cc, pool_n, 1)[:, :rows]
    skip = np.repeat(np.repeat(ss, pool_n, 1), pool_n, 2)[:, :rows, :cols]
    sym = m.encode_symbols(cache, skip, pool_n)
    # bytes: MSB-first packbits of the compressed rows (symbols.py:56-62)
    want_c = np.stack([np.packbits(cc[h]) for h in range(heads)])
    want_s = np.stack([np.stack([np.packbits(ss[h, r]) for r in range(comp_r)]) for h in range(heads)])
    assert np.array_equal(sym.s_c.cpu().numpy(), want_c)
    assert np.array_equal(sym.s_s.cpu().numpy(), want_s)
    active, pairs = sym.decoded()
    assert np.array_equal(active.cpu().numpy().astype(bool), cache)
    assert np.array_equal(pairs.cpu().numpy().astype(bool), skip)


def test_codec_nonuniform_group_rejected():
    m = fo()
    with pytest.raises(m.ConsistencyError):
        m.encode_symbols(np.array([[1, 0, 1, 1]], bool), np.ones((1, 4, 4), bool), 2)
    with pytest.raises(m.ConsistencyError):
        m.encode_symbols(np.ones((1, 2), bool), np.array([[[1, 0], [1, 1]]], bool), 2)


@pytest.mark.parametrize("seq,heads", [(512, 2), (300, 3), (1024, 4)])
def test_sparse_attention_bias_mode(seq, heads):
    m = fo()
    torch.manual_seed(0)
    rng = np.random.default_rng(seq)
    t = -(-seq // T)
    q, k, v = (torch.randn(seq, heads, T, device="cuda").bfloat16() for _ in range(3))
    cache_bits, skip_bits = rand_masks(rng, heads, t)
    sym = m.encode_symbols(cache_bits, skip_bits, 1)
    fc = m.FeatureCache(heads, t, 0, seq=seq)
    fc.push(v)  # warm cache so cached tiles are legal
    ac = m.AttnCounters()
    out = m.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias", fill=float("nan"),
                             counters=ac)
    want = torch_masked_attention(q, k, v, cache_bits, skip_bits)
    got = out.float().cpu().numpy()
    w = want.cpu().numpy()
    for h in range(heads):
        rows = np.repeat(cache_bits[h], T)[:seq]
        assert_bf16_close(got[rows, h], w[rows, h], f"head {h}")
        assert np.isnan(got[~rows, h]).all(), "cached rows must stay untouched"
    assert ac.pairs_computed == int(sum(skip_bits[h][cache_bits[h]].sum() for h in range(heads)))
    assert ac.pairs_total == heads * t * t


def test_dense_attention_update_and_cache():
    m = fo()
    torch.manual_seed(1)
    seq, heads, order = 384, 2, 2
    t = seq // T
    fc = m.FeatureCache(heads, t, order, seq=seq)
    outs = []
    for step in range(3):
        q, k, v = (torch.randn(seq, heads, T, device="cuda").bfloat16() for _ in range(3))
        o = m.dense_attention_update(q, k, v, fc)
        dense = torch_masked_attention(q, k, v, np.ones((heads, t), bool), np.ones((heads, t, t), bool))
        assert_bf16_close(o.float().cpu().numpy(), dense.cpu().numpy(), f"step {step}")
        outs.append(o.float())
    assert (fc.valid.cpu().numpy() == 3).all()
    st = fc.stacks.float().view(order + 1, seq, heads, T)
    assert torch.allclose(st[0], outs[2], atol=0, rtol=0)
    d1 = outs[2] - outs[1]
    d2 = d1 - (outs[1] - outs[0])
    assert_bf16_close(st[1].cpu().numpy(), d1.cpu().numpy(), "diff 1")
    # second difference: larger relative error (difference of differences of bf16 values)
    err = (st[2] - d2).abs().max().item()
    assert err < 0.03, err


def _rms_rope_ref(y, w, pos):
    D = y.shape[-1]
    ms = (y.double() ** 2).mean(-1, keepdim=True)
    y = y * w / torch.sqrt(ms + 1e-6)
    j = torch.arange(D // 2, dtype=torch.float64, device=y.device)
    ang = pos.double()[:, None] * (10000.0 ** (-2.0 * j / D))
    c, s = torch.cos(ang), torch.sin(ang)
    e, o = y[:, 0::2], y[:, 1::2]
    out = torch.empty_like(y)
    out[:, 0::2] = e * c - o * s
    out[:, 1::2] = e * s + o * c
    return out


@pytest.mark.parametrize("phase", ["update", "dispatch"])
@pytest.mark.parametrize("seq,dm,heads", [(384, 256, 3), (700, 192, 4), (1280, 384, 8)])
def test_gemm_q(phase, seq, dm, heads):
    """Odd heads (1-CTA dense path), even heads (CTA-pair dense path), a ragged
    last block and d_model not a multiple of 128."""
    m = fo()
    torch.manual_seed(2)
    t = -(-seq // T)
    rng = np.random.default_rng(3)
    x = torch.randn(seq, dm, device="cuda").bfloat16()
    w_q = torch.randn(heads, dm, T, device="cuda") * dm ** -0.5
    norm = 1 + 0.05 * torch.randn(heads, T, device="cuda")
    cache_bits, skip_bits = rand_masks(rng, heads, t, cached_ratio=0.4)
    sym = m.encode_symbols(cache_bits, skip_bits, 1) if phase == "dispatch" else None
    gc = m.GemmCounters()
    q = m.project_q(x, w_q, norm, sym, phase, fill=float("nan"), counters=gc)
    wq_b = w_q.bfloat16().double()
    pos = torch.arange(seq, device="cuda")
    for h in range(heads):
        ref = _rms_rope_ref(x.double() @ wq_b[h], norm[h].double(), pos)
        rows = np.repeat(cache_bits[h], T)[:seq] if phase == "dispatch" else np.ones(seq, bool)
        got = q[:, h].float().cpu().numpy()
        assert_bf16_close(got[rows], ref.cpu().numpy()[rows], f"head {h}")
        assert np.isnan(got[~rows]).all()
    n_rows = sum(int(np.repeat(cache_bits[h], T)[:seq].sum()) for h in range(heads)) \
        if phase == "dispatch" else heads * seq
    assert gc.q_macs_actual == n_rows * dm * T
    assert gc.q_macs_dense == heads * seq * dm * T


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("seq,dm", [(384, 256), (640, 384), (300, 640)])
def test_gemm_o_update_dispatch(order, seq, dm):
    """d_model 384 / 640 end on a 128-wide dispatch tile; 300 is a ragged block."""
    m = fo()
    torch.manual_seed(4)
    heads, interval = 4, 4
    t = -(-seq // T)
    rng = np.random.default_rng(5)
    w_out = torch.randn(heads, T, dm, device="cuda") * T ** -0.5
    fc = m.FeatureCache(heads, t, order, seq=seq)
    hist = []
    for _ in range(order + 1):
        o = torch.randn(seq, heads, T, device="cuda").bfloat16()
        fc.push(o)
        hist.append(o)
    o = hist[-1]
    active, skip = rand_masks(rng, heads, t, cached_ratio=0.5)
    sym = m.encode_symbols(active, skip, 1)
    out_u, bias = m.project_out_update(o, w_out, sym, fc, order)
    wb = w_out.bfloat16().double()
    dense = sum(o[:, h].double() @ wb[h] for h in range(heads))
    assert_bf16_close(out_u.float().cpu().numpy(), dense.cpu().numpy(), "update out")
    stacks = fc.stacks.double().view(order + 1, seq, heads, T)
    elapsed = 2
    coef = m.forecast_coefficients(elapsed, interval, order + 1)
    o2 = torch.randn(seq, heads, T, device="cuda").bfloat16()
    got = m.project_out_dispatch(o2, w_out, sym, bias, elapsed, interval, order)
    # oracle: materialize forecast tiles, then one dense projection
    full = o2.double().clone()
    for h in range(heads):
        for i in range(t):
            if not active[h, i]:
                r = slice(i * T, (i + 1) * T)
                full[r, h] = sum(float(coef[d]) * stacks[d, r, h] for d in range(order + 1))
    ref = sum(full[:, h] @ wb[h] for h in range(heads))
    assert_bf16_close(got.float().cpu().numpy(), ref.cpu().numpy(), "dispatch out")


def test_gemm_o_stale_symbols_rejected():
    m = fo()
    seq, dm, heads = 256, 128, 2
    t = seq // T
    rng = np.random.default_rng(6)
    w_out = torch.randn(heads, T, dm, device="cuda")
    fc = m.FeatureCache(heads, t, 0, seq=seq)
    o = torch.randn(seq, heads, T, device="cuda").bfloat16()
    fc.push(o)
    active, skip = rand_masks(rng, heads, t, cached_ratio=0.5)
    sym = m.encode_symbols(active, skip, 1)
    _, bias = m.project_out_update(o, w_out, sym, fc, 0)
    other = m.encode_symbols(~active, np.ones((heads, t, t), bool), 1)
    with pytest.raises(m.StateError):
        m.project_out_dispatch(o, w_out, other, bias, 1, 4, 0)
    with pytest.raises(m.StateError):
        m.project_out_dispatch(o, w_out, sym, None, 1, 4, 0)


def test_empty_active_row_and_cold_cache():
    m = fo()
    seq, heads = 512, 1
    t = seq // T
    q, k, v = (torch.randn(seq, heads, T, device="cuda").bfloat16() for _ in range(3))
    cache_bits = np.ones((1, t), bool)
    skip_bits = np.ones((1, t, t), bool)
    skip_bits[0, 2] = False
    sym = m.encode_symbols(cache_bits, skip_bits, 1)
    with pytest.raises(m.ConsistencyError):
        m.sparse_attention(q, k, v, sym, None, None, 0, 1, 0, mode="bias")
    cache_bits[0, 1] = False
    skip_bits[0, 2] = True
    skip_bits[0, 1] = False
    sym = m.encode_symbols(cache_bits, skip_bits, 1)
    cold = m.FeatureCache(heads, t, 0, seq=seq)
    with pytest.raises(m.StateError):
        m.sparse_attention(q, k, v, sym, cold, None, 1, 2, 0, mode="bias")
