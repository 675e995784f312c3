"""Parity at the bench's own shapes (BASELINE configs C1, C2, C3/C4).

C4 / C3: S = 33,024 tokens (258 blocks), d_model 3072, 24 heads x 128 — the
exact GEMM-Q and GEMM-O shapes bench.py times. Full-size outputs are compared
against the CPU oracle (oracle/, a restatement of gemm.py / attention.py) on
sampled row blocks: every (block, head) computation is block-local, so a
subset of blocks, fed to the oracle as a short sequence, is an exact
restatement of those rows. Tolerance: the stated bf16 bound (conftest.py).

GEMM-Q is checked from mostly-N=256 (heads 2p, 2p+1 active together) to
almost-only-N=128 job mixes, and the plan's job list is checked for exact
coverage of the active tiles.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bf16_close

pytestmark = pytest.mark.gpu

T = 128
S_C4, DM, H = 33024, 3072, 24
T_C4 = S_C4 // T


def fo():
    import paper_2509_25401_b200 as m

    return m


def bf16_np(t):
    return t.float().cpu().numpy()


def sample_blocks(rng, t, n=6):
    """First, last (ragged-free at C4) and a few random blocks."""
    pick = {0, t - 1}
    while len(pick) < n:
        pick.add(int(rng.integers(t)))
    return np.array(sorted(pick))


def rows_of(blocks, seq):
    return np.concatenate([np.arange(b * T, min(b * T + T, seq)) for b in blocks])


def cache_masks(rng, heads, t, cached_ratio):
    active = rng.random((heads, t)) >= cached_ratio
    for h in range(heads):
        if not active[h].any():
            active[h, rng.integers(t)] = True
    return active


# ---------------------------------------------------------------------------
# GEMM-Q at C4, CTA-pair path on / off
# ---------------------------------------------------------------------------
def check_gq_jobs(plan, active):
    """Every active (block, head) tile is in exactly one GEMM-Q job, no cached
    tile is in any, N=256 jobs pair two distinct heads active together in both
    blocks, and the list is ordered by cost class, then by first block."""
    jobs = plan.gq_jobs()
    H, t = active.shape
    seen = np.zeros((H, t), int)
    for i0, i1, h, n256, h2 in jobs:
        heads = (h, h2) if n256 else (h,)
        if n256:
            assert h < h2 < H
        for i in (i0, i1):
            if i < 0:
                continue
            for hh in heads:
                seen[hh, i] += 1
    assert np.array_equal(seen, active.astype(int))
    # ordered by cost class (N=256 pairs of blocks, N=128 pairs, single-block
    # jobs), then by first block
    cls = np.where(jobs[:, 1] < 0, 2, np.where(jobs[:, 3] > 0, 0, 1))
    assert np.all(np.diff(cls) >= 0)
    for c in range(3):
        assert np.all(np.diff(jobs[cls == c, 0]) >= 0)
    return jobs


@pytest.mark.parametrize("cached_ratio", [0.1, 0.5, 0.9])
def test_gemm_q_c4_dispatch(cached_ratio):
    """One CTA-pair launch mixes N=256 (both heads of a pair active) and N=128
    jobs; 10% cached is mostly N=256, 90% almost only N=128."""
    m = fo()
    torch.manual_seed(21)
    rng = np.random.default_rng(int(cached_ratio * 100))
    x = torch.randn(S_C4, DM, device="cuda").bfloat16()
    w_q = (torch.randn(H, DM, T, device="cuda") * DM ** -0.5).bfloat16().float()
    norm = 1 + 0.05 * torch.randn(H, T, device="cuda")
    active = cache_masks(rng, H, T_C4, cached_ratio)
    sym = m.encode_symbols(active, np.ones((H, T_C4, T_C4), bool) & active[:, :, None], 1)
    plan = sym.plan()
    jobs = check_gq_jobs(plan, active)
    # share of the active tiles in N=256 jobs (heads paired per block): fixed
    # pairs alone would give ~0.9 / 0.5 / 0.1 here
    tiles256 = 4 * int((jobs[:, 3] * (jobs[:, 1] >= 0)).sum())
    share = tiles256 / int(active.sum())
    assert share > {0.1: 0.9, 0.5: 0.8, 0.9: 0.3}[cached_ratio], share
    gc = m.GemmCounters()
    q = m.project_q(x, w_q, norm, sym, "dispatch", fill=float("nan"), counters=gc)
    torch.cuda.synchronize()
    assert gc.q_macs_actual == int(active.sum()) * T * DM * T
    blocks = sample_blocks(rng, T_C4)
    rows = rows_of(blocks, S_C4)
    want = oracle.project_q(bf16_np(x)[rows], w_q.cpu().numpy(), norm.cpu().numpy(),
                            active[:, blocks], T, positions=rows, fill=np.nan)
    got = bf16_np(q[torch.from_numpy(rows).cuda()])
    for h in range(H):
        sel = np.repeat(active[h, blocks], T)
        if sel.any():
            assert_bf16_close(got[sel, h], want[h][sel], f"head {h}")
        assert np.isnan(got[~sel, h]).all(), "skipped tiles keep the fill"


def test_gemm_q_c4_update_phase():
    m = fo()
    torch.manual_seed(22)
    rng = np.random.default_rng(22)
    x = torch.randn(S_C4, DM, device="cuda").bfloat16()
    w_q = (torch.randn(H, DM, T, device="cuda") * DM ** -0.5).bfloat16().float()
    norm = 1 + 0.05 * torch.randn(H, T, device="cuda")
    q = m.project_q(x, w_q, norm, None, "update")
    blocks = sample_blocks(rng, T_C4)
    rows = rows_of(blocks, S_C4)
    want = oracle.project_q(bf16_np(x)[rows], w_q.cpu().numpy(), norm.cpu().numpy(), None, T,
                            positions=rows)
    got = bf16_np(q[torch.from_numpy(rows).cuda()])
    for h in range(H):
        assert_bf16_close(got[:, h], want[h], f"head {h}")


# ---------------------------------------------------------------------------
# GEMM-O update + dispatch at C3/C4, orders 0..3
# ---------------------------------------------------------------------------
def _filled_cache(m, rng, order, seq=S_C4, heads=H):
    """order+1 pushes: every entry's valid order is order+1, except a random
    subset pushed one time fewer (mixed valid orders per block)."""
    t = seq // T
    fc = m.FeatureCache(heads, t, order, seq=seq)
    hist = []
    for r in range(order + 1):
        o = torch.randn(seq, heads, T, device="cuda").bfloat16()
        sel = None if r == 0 or r < order else (rng.random((heads, t)) < 0.7).astype(np.uint8)
        fc.push(o, select=sel)
        hist.append(o)
    return fc, hist


def _oracle_stacks(fc, blocks, heads):
    """Per-head, per-sampled-block diff stacks and valid orders from the
    device cache (the oracle consumes the cache state, not its history)."""
    st = fc.stacks.float().view(fc.order + 1, fc.seq, heads, T)
    valid = fc.valid.cpu().numpy()
    stacks = [[None] * len(blocks) for _ in range(heads)]
    vsub = np.zeros((heads, len(blocks)), int)
    for bi, b in enumerate(blocks):
        tile = st[:, b * T:(b + 1) * T].cpu().numpy()  # [order+1, 128, heads, 128]
        for h in range(heads):
            stacks[h][bi] = tile[:, :, h]
            vsub[h, bi] = valid[h, b]
    return stacks, vsub


@pytest.mark.parametrize("order,cached_ratio", [(0, 0.25), (1, 0.25), (1, 0.9), (2, 0.5),
                                                (3, 0.75)])
def test_gemm_o_c4_update_and_dispatch(order, cached_ratio):
    m = fo()
    torch.manual_seed(30 + order)
    rng = np.random.default_rng(30 + order)
    w_out = (torch.randn(H, T, DM, device="cuda") * T ** -0.5).bfloat16().float()
    fc, hist = _filled_cache(m, rng, order)
    # o != the cache's stack 0: the update must take cached heads' order-0
    # term from the cache (gemm.py:155-161), active heads from o
    o = torch.randn(S_C4, H, T, device="cuda").bfloat16()
    active = cache_masks(rng, H, T_C4, cached_ratio)
    sym = m.encode_symbols(active, np.ones((H, T_C4, T_C4), bool) & active[:, :, None], 1)
    gc = m.GemmCounters()
    out_u, bias = m.project_out_update(o, w_out, sym, fc, order, counters=gc)
    torch.cuda.synchronize()
    blocks = sample_blocks(rng, T_C4)
    rows = rows_of(blocks, S_C4)
    stacks, vsub = _oracle_stacks(fc, blocks, H)
    o_sub = bf16_np(o[torch.from_numpy(rows).cuda()]).transpose(1, 0, 2)  # [H, n, 128]
    wn = w_out.cpu().numpy()
    want_out, want_bias, want_orders = oracle.project_out_update(
        o_sub, wn, active[:, blocks].T, stacks, vsub, order, T)
    got_out = bf16_np(out_u[torch.from_numpy(rows).cuda()])
    assert_bf16_close(got_out, want_out, f"update out, order {order}")
    orders = bias.orders.cpu().numpy()
    assert np.array_equal(orders[blocks], want_orders), "bias orders"
    bs = bias.stacks.float()
    for bi, b in enumerate(blocks):
        for d in range(int(want_orders[bi])):
            assert_bf16_close(bs[d, b * T:(b + 1) * T].cpu().numpy(), want_bias[bi][d],
                              f"B_c[{d}] block {b}")
    # every active head once, every cached head once per populated order
    full_orders = orders
    n_cached = (~active).sum(0)
    assert gc.o_bias_macs == int((n_cached * np.maximum(full_orders - 1, 0)).sum()) * T * T * DM

    # dispatch: active heads of a fresh o plus the forecast of the bias
    o2 = torch.randn(S_C4, H, T, device="cuda").bfloat16()
    for elapsed, interval in ((1, 6), (5, 6)):
        got = m.project_out_dispatch(o2, w_out, sym, bias, elapsed, interval, order)
        bias_sub = [bs[:int(orders[b]), b * T:(b + 1) * T].cpu().numpy() for b in blocks]
        o2_sub = bf16_np(o2[torch.from_numpy(rows).cuda()]).transpose(1, 0, 2)
        want = oracle.project_out_dispatch(o2_sub, wn, active[:, blocks].T, bias_sub,
                                           orders[blocks], elapsed, interval, order, T)
        assert_bf16_close(bf16_np(got[torch.from_numpy(rows).cuda()]), want,
                          f"dispatch out, order {order}, k={elapsed}")


def test_gemm_o_update_takes_cached_order0_from_cache():
    """Small shape, exact structure: with o != cache stack 0, a block whose
    heads are all cached must equal sum_h stack0_h W_h, and an all-active block
    sum_h o_h W_h."""
    m = fo()
    torch.manual_seed(40)
    seq, heads, dm = 512, 4, 256
    t = seq // T
    w_out = (torch.randn(heads, T, dm, device="cuda") * T ** -0.5).bfloat16().float()
    fc = m.FeatureCache(heads, t, 0, seq=seq)
    c0 = torch.randn(seq, heads, T, device="cuda").bfloat16()
    fc.push(c0)
    o = torch.randn(seq, heads, T, device="cuda").bfloat16()
    active = np.ones((heads, t), bool)
    active[:, 1] = False  # block 1: every head cached
    active[0, 2] = False  # block 2: one head cached
    sym = m.encode_symbols(active, np.ones((heads, t, t), bool) & active[:, :, None], 1)
    out, bias = m.project_out_update(o, w_out, sym, fc, 0)
    wb = w_out.double()
    src = torch.where(torch.from_numpy(np.repeat(active.T, T, 0)).cuda()[:, :, None], o, c0)
    want = sum(src[:, h].double() @ wb[h] for h in range(heads))
    assert_bf16_close(out.float().cpu().numpy(), want.cpu().numpy(), "update out")
    b1 = sum(c0[T:2 * T, h].double() @ wb[h] for h in range(heads))
    assert_bf16_close(bias.stacks[0, T:2 * T].float().cpu().numpy(), b1.cpu().numpy(), "B_c[0]")


# ---------------------------------------------------------------------------
# OP_reuse (forecast) at orders 2 and 3 against oracle.forecast
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("order", [2, 3])
def test_forecast_orders_2_3_against_oracle(order):
    m = fo()
    torch.manual_seed(50 + order)
    rng = np.random.default_rng(50 + order)
    n, heads = 1536, 3
    t = n // T
    fc = m.FeatureCache(heads, t, order, seq=n)
    hist = []
    sels = []
    for r in range(order + 2):  # one push past the order: the stack saturates
        o = torch.randn(n, heads, T, device="cuda").bfloat16()
        sel = np.ones((heads, t), np.uint8) if r == 0 else (rng.random((heads, t)) < 0.8).astype(np.uint8)
        fc.push(o, select=sel)
        hist.append(bf16_np(o))
        sels.append(sel)
    q, k, v = (torch.randn(n, heads, T, device="cuda").bfloat16() for _ in range(3))
    cb = np.zeros((heads, t), bool)
    sb = np.zeros((heads, t, t), bool)
    for h in range(heads):
        cb[h], sb[h] = oracle.random_masks(rng, t, t, 1, density=0.5, cache_density=0.4)
    sym = m.encode_symbols(cb, sb, 1)
    for elapsed, interval in ((1, 4), (3, 4), (2, 8)):
        out = m.sparse_attention(q, k, v, sym, fc, None, elapsed, interval, order,
                                 mode="materialize")
        of = bf16_np(out)
        for h in range(heads):
            for i in range(t):
                if cb[h, i]:
                    continue
                r = slice(i * T, (i + 1) * T)
                st, vv = None, 0
                for step, tile in enumerate(hist):
                    if sels[step][h, i]:
                        # the device stores each difference in bf16: restate the
                        # recurrence on the rounded values the cache holds
                        st, vv = oracle.update_entry(st, vv, tile[r, h], order)
                want = oracle.forecast(st, vv, elapsed, interval, order)
                assert int(fc.valid[h, i]) == vv
                assert_bf16_close(of[r, h], want, f"forecast ({h},{i}) k={elapsed}")


# ---------------------------------------------------------------------------
# attention at C1 (S=4096) and C2 (FLUX, S=4608) shapes
# ---------------------------------------------------------------------------
def _attention_check(m, seq, heads, cb, sb, check_heads, seed):
    torch.manual_seed(seed)
    t = -(-seq // T)
    q, k, v = (torch.randn(seq, heads, T, device="cuda").bfloat16() for _ in range(3))
    sym = m.encode_symbols(cb, sb, 1)
    fc = m.FeatureCache(heads, t, 0, seq=seq)
    fc.push(v)
    ac = m.AttnCounters()
    out = m.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias", fill=float("nan"),
                             counters=ac)
    assert ac.pairs_computed == int(sum(sb[h][cb[h]].sum() for h in range(heads)))
    assert ac.pairs_total == heads * t * t
    qf, kf, vf, of = (bf16_np(a) for a in (q, k, v, out))
    for h in check_heads:
        want = oracle.masked_attention(qf[:, h], kf[:, h], vf[:, h], cb[h], sb[h], T, T)
        rows = np.repeat(cb[h], T)[:seq]
        assert_bf16_close(of[rows, h], want[rows], f"head {h}")
        assert np.isnan(of[~rows, h]).all()


def test_attention_c1():
    """C1: H=24, S=4096, 25% cached q-blocks, 50% KV skip (verify.py:29-44 rule)."""
    m = fo()
    rng = np.random.default_rng(60)
    t = 32
    cb = np.zeros((H, t), bool)
    sb = np.zeros((H, t, t), bool)
    for h in range(H):
        cb[h], sb[h] = oracle.random_masks(rng, t, t, 1, density=0.5, cache_density=0.75)
    _attention_check(m, 4096, H, cb, sb, [0, 7, 23], 60)


@pytest.mark.parametrize("sparsity", [0.0, 0.7, 0.9])
def test_attention_c2_flux(sparsity):
    """C2: FLUX joint attention, 4,608 tokens (4 text + 32 image blocks), block
    sparsity sweep; text rows/columns stay dense (the policy's guard)."""
    m = fo()
    rng = np.random.default_rng(61 + int(sparsity * 10))
    t, n_text = 36, 4
    cb = np.ones((H, t), bool)
    sb = rng.random((H, t, t)) >= sparsity
    sb[:, :, :n_text] = True
    sb[:, :n_text, :] = True
    for h in range(H):
        np.fill_diagonal(sb[h], True)
    _attention_check(m, 4608, H, cb, sb, [0, 11, 23], 61)


def test_fused_qkv_projection_matches_separate_launches():
    """fo_gemm_qkv (one launch: the plan's active Q tiles + dense K and V)
    equals the three separate projections bit for bit (same tiles, same K
    order), in the dispatch and the update phase, at the bench's shape."""
    import torch

    m = fo()
    rng = np.random.default_rng(17)
    S, H, dm, T = 4096 + 128 * 3, 24, 3072, 128
    t = -(-S // T)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(S, dm, device="cuda", generator=g).bfloat16()
    w = [torch.randn(H, dm, T, device="cuda", generator=g) * dm ** -0.5 for _ in range(3)]
    qn = 1 + 0.05 * torch.randn(H, T, device="cuda", generator=g)
    kn = 1 + 0.05 * torch.randn(H, T, device="cuda", generator=g)
    params = m.LayerParams.from_reference(w[0], w[1], w[2], qn, kn,
                                          torch.randn(H, T, dm, device="cuda") * T ** -0.5)
    active = rng.random((H, t)) >= 0.6
    sym = m.encode_symbols(active, np.ones((H, t, t), bool), 1)
    for phase, sy in (("dispatch", sym), ("update", None)):
        q, k, v = m.project_qkv(x, params.w_qkv, qn, kn, sy, phase, fill=float("nan"))
        q0 = m.project_q(x, params.w_q, qn, sy, phase, fill=float("nan"))
        k0, v0 = m.project_kv(x, params)
        torch.cuda.synchronize()
        assert torch.equal(k, k0) and torch.equal(v, v0)
        rows = torch.ones(S, H, dtype=torch.bool, device="cuda")
        if phase == "dispatch":
            rows = torch.from_numpy(np.repeat(active.T, T, axis=0)[:S]).cuda()
            assert torch.isnan(q[~rows]).all()  # skipped tiles keep the fill
        assert torch.equal(q[rows], q0[rows])


@pytest.mark.parametrize("S,H,dm", [(1000, 3, 256), (777, 5, 384), (128, 1, 128)])
def test_fused_qkv_ragged_and_odd_heads(S, H, dm):
    """The fused projection at a ragged last block (rows past S clipped), odd
    head counts (the last head alone: N = 128 jobs in every segment) and one
    block: still equal to the separate launches bit for bit."""
    import torch

    m = fo()
    rng = np.random.default_rng(S + H)
    T = 128
    t = -(-S // T)
    g = torch.Generator(device="cuda").manual_seed(S)
    x = torch.randn(S, dm, device="cuda", generator=g).bfloat16()
    w = [torch.randn(H, dm, T, device="cuda", generator=g) * dm ** -0.5 for _ in range(3)]
    qn = 1 + 0.05 * torch.randn(H, T, device="cuda", generator=g)
    kn = 1 + 0.05 * torch.randn(H, T, device="cuda", generator=g)
    params = m.LayerParams.from_reference(w[0], w[1], w[2], qn, kn,
                                          torch.randn(H, T, dm, device="cuda") * T ** -0.5)
    active = rng.random((H, t)) >= 0.5
    active[:, 0] = True
    sym = m.encode_symbols(active, np.ones((H, t, t), bool), 1)
    for phase, sy in (("dispatch", sym), ("update", None)):
        q, k, v = m.project_qkv(x, params.w_qkv, qn, kn, sy, phase, fill=float("nan"))
        q0 = m.project_q(x, params.w_q, qn, sy, phase, fill=float("nan"))
        k0, v0 = m.project_kv(x, params)
        torch.cuda.synchronize()
        assert torch.equal(k, k0) and torch.equal(v, v0)
        rows = torch.ones(S, H, dtype=torch.bool, device="cuda")
        if phase == "dispatch":
            rows = torch.from_numpy(np.repeat(active.T, T, axis=0)[:S]).cuda()
        assert torch.equal(q[rows], q0[rows])
        assert torch.isfinite(k).all() and torch.isfinite(v).all()


@pytest.mark.parametrize("H,t", [(1, 9), (2, 5), (5, 33), (17, 40), (24, 258), (64, 12)])
@pytest.mark.parametrize("ratio", [0.0, 0.3, 0.7, 0.95])
def test_gq_job_list_invariants(H, t, ratio):
    """The per-block head pairing covers every active tile exactly once at odd
    head counts, a single head, 64 heads and every density (including none
    and all active), and the kernel's output equals the per-head oracle rows."""
    m = fo()
    rng = np.random.default_rng(H * 100 + t + int(ratio * 10))
    active = rng.random((H, t)) >= ratio
    sym = m.encode_symbols(active, np.ones((H, t, t), bool), 1)
    if not active.any():
        return
    check_gq_jobs(sym.plan(), active)
    if H * t > 2000:
        return
    S, dm = t * T - 37, 256
    g = torch.Generator(device="cuda").manual_seed(H + t)
    x = torch.randn(S, dm, device="cuda", generator=g).bfloat16()
    w_q = (torch.randn(H, dm, T, device="cuda", generator=g) * dm ** -0.5).bfloat16().float()
    norm = 1 + 0.05 * torch.randn(H, T, device="cuda", generator=g)
    q = m.project_q(x, w_q, norm, sym, "dispatch", fill=float("nan"))
    want = oracle.project_q(bf16_np(x), w_q.cpu().numpy(), norm.cpu().numpy(), active, T,
                            fill=np.nan)
    got = bf16_np(q)
    for h in range(H):
        sel = np.repeat(active[h], T)[:S]
        if sel.any():
            assert_bf16_close(got[sel, h], want[h][sel], f"head {h}")
        assert np.isnan(got[~sel, h]).all()
