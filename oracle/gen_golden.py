"""Generate tests/golden/*.npz by running the REFERENCE implementation.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Imports `omniattn` from the read-only reference tree (numpy backend) in this
container only; the fixtures are committed so nothing at test time needs
/root/reference. Float inputs are rounded to bf16-representable values first,
so the GPU engine (bf16 operands) and the reference (fp32) see identical
numbers and the only difference left is arithmetic precision.
"""

import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from omniattn import attention as ref_attn  # noqa: E402
from omniattn import gemm as ref_gemm  # noqa: E402
from omniattn import symbols as ref_sym  # noqa: E402
from omniattn import policy as ref_policy  # noqa: E402
from omniattn import verify as ref_verify  # noqa: E402
from omniattn import pipeline as ref_pipeline  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parents[1] / "tests" / "golden"
T = 128


def bf16_bits(a):
    """fp32 -> bf16 bit pattern (round to nearest even)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def from_bf16_bits(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def bf16_round(a):
    return from_bf16_bits(bf16_bits(a))


def codec():
    d = {}
    idx = 0
    for pool_n in (1, 2, 4):
        rng = np.random.default_rng(100 + pool_n)
        for _ in range(12):
            t_q = int(rng.integers(1, 70))
            t_kv = int(rng.integers(1, 70))
            cb, sb = ref_verify.random_masks(rng, t_q, t_kv, pool_n)
            sym = ref_sym.build_symbols(cb, sb, pool_n)
            d[f"c{idx}_cache"] = cb
            d[f"c{idx}_skip"] = sb
            d[f"c{idx}_pool"] = np.array(pool_n)
            d[f"c{idx}_sc"] = np.frombuffer(sym.s_c, np.uint8)
            d[f"c{idx}_ss"] = np.frombuffer(sym.s_s, np.uint8)
            d[f"c{idx}_blob"] = np.frombuffer(sym.to_bytes(), np.uint8)
            idx += 1
    d["n_cases"] = np.array(idx)
    np.savez_compressed(OUT / "codec.npz", **d)


def attention():
    d = {}
    cases = [(256, 1, 11), (300, 1, 12), (640, 2, 13)]
    for ci, (n, pool_n, seed) in enumerate(cases):
        rng = np.random.default_rng(seed)
        t = -(-n // T)
        q, k, v = (bf16_round(rng.standard_normal((n, T)).astype(np.float32)) for _ in range(3))
        cb, sb = ref_verify.random_masks(rng, t, t, pool_n, density=0.5, cache_density=0.75)
        sym = ref_sym.build_symbols(cb, sb, pool_n)
        cache = ref_attn.FeatureCache(1, t, 0)
        for i in range(t):
            cache.update(0, i, v[i * T:min((i + 1) * T, n)])
        ac = ref_attn.AttnCounters()
        out = ref_attn.sparse_attention(q, k, v, sym, cache, 0, 1, 2, 0, b_q=T, b_k=T, mode="bias",
                                        fill=np.nan, counters=ac)
        p = f"a{ci}_"
        d.update({p + "q": bf16_bits(q), p + "k": bf16_bits(k), p + "v": bf16_bits(v),
                  p + "cache": cb, p + "skip": sb, p + "pool": np.array(pool_n),
                  p + "out": out, p + "pairs": np.array(ac.pairs_computed),
                  p + "total": np.array(ac.pairs_total)})
    d["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "attention.npz", **d)


def gemm_q():
    rng = np.random.default_rng(21)
    n, dm, heads = 256, 256, 3
    t = n // T
    x = bf16_round(rng.standard_normal((n, dm)).astype(np.float32))
    w_q = bf16_round((rng.standard_normal((heads, dm, T)) * dm ** -0.5).astype(np.float32))
    norm = (1.0 + 0.05 * rng.standard_normal((heads, T))).astype(np.float32)
    active = rng.random((t, heads)) < 0.6
    active[0] = True
    syms = [ref_sym.build_symbols(active[:, h], np.ones((t, t), bool), 1) for h in range(heads)]
    gc = ref_gemm.GemmCounters()
    disp = ref_gemm.project_q(x, w_q, norm, syms, "dispatch", b_q=T, counters=gc, fill=np.nan)
    upd = ref_gemm.project_q(x, w_q, norm, None, "update", b_q=T)
    np.savez_compressed(OUT / "gemm_q.npz", x=bf16_bits(x), w_q=bf16_bits(w_q), norm=norm,
                        active=active, dispatch=disp, update=upd,
                        q_macs_actual=np.array(gc.q_macs_actual),
                        q_macs_dense=np.array(gc.q_macs_dense))


def gemm_o():
    rng = np.random.default_rng(31)
    n, dm, heads, order, interval, elapsed = 256, 256, 3, 1, 5, 2
    t = n // T
    w_out = bf16_round((rng.standard_normal((heads, T, dm)) * T ** -0.5).astype(np.float32))
    cache = ref_attn.FeatureCache(heads, t, order)
    hist = []
    for _ in range(order + 1):
        o = bf16_round(rng.standard_normal((heads, n, T)).astype(np.float32))
        hist.append(o)
        for h in range(heads):
            for i in range(t):
                cache.update(h, i, o[h, i * T:(i + 1) * T])
    o_cur = hist[-1]
    active = rng.random((t, heads)) < 0.5
    syms = [ref_sym.build_symbols(active[:, h], np.ones((t, t), bool), 1) for h in range(heads)]
    out_u, bias = ref_gemm.project_out_update(o_cur, w_out, syms, cache, order, b_q=T)
    o_disp = bf16_round(rng.standard_normal((heads, n, T)).astype(np.float32))
    gc = ref_gemm.GemmCounters()
    out_d = ref_gemm.project_out_dispatch(o_disp, w_out, syms, bias, elapsed, interval, order, b_q=T,
                                          counters=gc)
    bias_full = np.zeros((order + 1, n, dm), np.float32)
    for i in range(t):
        st = bias.stacks[i]
        bias_full[:st.shape[0], i * T:(i + 1) * T] = st
    np.savez_compressed(OUT / "gemm_o.npz", hist=np.stack([bf16_bits(a) for a in hist]),
                        w_out=bf16_bits(w_out), active=active, out_update=out_u,
                        bias=bias_full, orders=bias.orders, o_disp=bf16_bits(o_disp),
                        out_dispatch=out_d, order=np.array(order),
                        interval=np.array(interval), elapsed=np.array(elapsed),
                        o_macs_actual=np.array(gc.o_macs_actual))


def cache_push():
    rng = np.random.default_rng(41)
    rows, order = 128, 2
    a, b, c = (bf16_round(rng.standard_normal((rows, T)).astype(np.float32)) for _ in range(3))
    tiles, stacks, valids = [], [], []
    e = None
    for t_ in range(4):
        tile = bf16_round((a + t_ * b + 0.25 * t_ * t_ * c).astype(np.float32))
        e = ref_attn.update_entry(e, tile, order)
        tiles.append(tile)
        stacks.append(e.diff_stack.copy())
        valids.append(e.valid_orders)
    coef = ref_attn.forecast_coefficients(2, 4, order + 1)
    fc = ref_attn.forecast(e, 2, 4, order)
    np.savez_compressed(OUT / "cache.npz", tiles=np.stack([bf16_bits(x) for x in tiles]),
                        stacks=np.stack(stacks), valids=np.array(valids), coef=coef, forecast=fc)


def policy():
    """generate_masks (policy.py:196-234) on structured bf16-representable q/k:
    a text prefix plus vision tokens whose blocks share a random direction, so
    the pooled map has real structure and the selections are non-trivial."""
    d = {}
    cases = [  # (n, n_text, pool_n, tau_q, tau_kv, s_q, guard, seed)
        (1536, 256, 1, 0.3, 0.2, 0.0, True, 51),
        (2048, 128, 1, 0.5, 0.4, 0.0, True, 52),
        (1664, 300, 2, 0.4, 0.3, 0.0, True, 53),
        (1024, 128, 1, 0.6, 0.5, 0.9, True, 54),
        (1280, 200, 1, 0.2, 0.6, 0.0, False, 55),
    ]
    for ci, (n, n_text, pool, tq, tkv, sq, guard, seed) in enumerate(cases):
        rng = np.random.default_rng(seed)
        t = -(-n // T)
        base_q = rng.standard_normal((t, T)) * 1.5
        base_k = rng.standard_normal((t, T)) * 1.5
        q = np.repeat(base_q, T, 0)[:n] + rng.standard_normal((n, T))
        k = np.repeat(base_k, T, 0)[:n] + rng.standard_normal((n, T))
        q, k = bf16_round(q.astype(np.float32)), bf16_round(k.astype(np.float32))
        cb, sb = ref_policy.generate_masks(q, k, b_q=T, b_k=T, pool_n=pool, n_text=n_text,
                                           tau_q=tq, tau_kv=tkv, s_q=sq, guard=guard)
        p = f"p{ci}_"
        d.update({p + "q": bf16_bits(q), p + "k": bf16_bits(k), p + "cache": cb, p + "skip": sb,
                  p + "args": np.array([n, n_text, pool, tq, tkv, sq, float(guard)], np.float64)})
    d["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "policy.npz", **d)


# run() configurations (pipeline.py:337-371) at the sm_100a tile geometry
RUN_CASES = [
    dict(n_text=128, n_vision=896, d_model=128, heads=2, tau_q=0.3, tau_kv=0.4, interval_n=3,
         order_d=1, steps=6, layers=2, workload="drift", smoothness=0.05, seed=7),
    dict(n_text=200, n_vision=1848, d_model=128, heads=2, pool_n=2, tau_q=0.8, tau_kv=0.7,
         interval_n=3, order_d=0, steps=6, layers=1, warmup=4, workload="poly2", smoothness=0.1,
         seed=8),
]
STEP_KEYS = ("attn_pairs_total", "attn_pairs_computed", "attn_pairs_mask_skipped",
             "gemm_q_macs_dense", "gemm_q_macs_actual", "gemm_o_macs_dense", "gemm_o_macs_actual",
             "gemm_o_bias_macs")


class _Bf16Workload:
    """The reference SyntheticWorkload with its projection weights and every
    x(t) rounded to bf16 (norm weights stay fp32, as on the GPU), so the GPU
    engine and the reference consume identical numbers."""

    def __init__(self, cfg):
        self.inner = ref_pipeline.synthetic_workload(cfg)
        for lp in self.inner.layer_params:
            for name in ("w_q", "w_k", "w_v", "w_out"):
                setattr(lp, name, bf16_round(getattr(lp, name)))
        self.layer_params = self.inner.layer_params

    def x(self, t):
        return bf16_round(self.inner.x(t))


def pipeline_run():
    """Reference run(): per-step last-layer outputs, step costs, final symbols."""
    d = {}
    for ci, kw in enumerate(RUN_CASES):
        cfg = ref_pipeline.EngineConfig(b_q=T, b_k=T, d=T, **kw)
        wl = _Bf16Workload(cfg)
        res = ref_pipeline.run(cfg, wl)
        p = f"r{ci}_"
        # unrounded generator draws, to pin SyntheticWorkload's RNG sequence
        raw = ref_pipeline.synthetic_workload(cfg)
        lp = raw.layer_params[-1]
        d[p + "w_probe"] = np.concatenate([lp.w_q[-1, -3:, :5].ravel(), lp.q_norm[0, :5],
                                           lp.k_norm[-1, -5:], lp.w_out[0, :3, -5:].ravel()])
        d[p + "x_probe"] = np.stack([raw.x(t)[-4:, :6] for t in range(cfg.steps)])
        d[p + "out"] = np.stack(res.outputs).astype(np.float16)
        d[p + "costs"] = np.array([[getattr(sc, k) for k in STEP_KEYS] for sc in res.step_costs],
                                  np.int64)
        d[p + "phase"] = np.array([sc.phase == "update" for sc in res.step_costs])
        for li, st in enumerate(res.states):
            d[p + f"l{li}_sc"] = np.stack([np.frombuffer(s.s_c, np.uint8) for s in st.symbols])
            d[p + f"l{li}_ss"] = np.stack([np.frombuffer(s.s_s, np.uint8) for s in st.symbols])
        r = res.report
        d[p + "report"] = np.array([r.attn_pairs_total, r.attn_pairs_skipped, r.gemm_q_macs_dense,
                                    r.gemm_q_macs_actual, r.gemm_o_macs_dense,
                                    r.gemm_o_macs_actual, r.gemm_o_bias_macs], np.int64)
        d[p + "speedups"] = np.array([r.sparsity, r.speedup_attention or 0.0, r.speedup_gemm_o])
    d["n_cases"] = np.array(len(RUN_CASES))
    np.savez_compressed(OUT / "run.npz", **d)


def api():
    """The reference's tile-level and policy building blocks on float32 inputs
    (not bf16-rounded: these device functions compute in float32/float64 like
    the reference), small d and blocks as the reference's own tests use them
    (attention.py:21-113, policy.py:21-178, tensor.py:33-126)."""
    from omniattn import tensor as ref_tensor

    d = {}
    rng = np.random.default_rng(7)
    # online softmax over three score blocks, then finalize
    rows, d_h = 24, 16
    st = ref_attn.OnlineSoftmaxState.fresh(rows, d_h)
    for b, cols in enumerate((8, 32, 5)):
        s_blk = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
        v_blk = rng.standard_normal((cols, d_h)).astype(np.float32)
        d[f"os{b}_scores"], d[f"os{b}_v"] = s_blk, v_blk
        st = ref_attn.online_softmax_update(st, s_blk, v_blk)
        d[f"os{b}_m"], d[f"os{b}_l"], d[f"os{b}_acc"] = st.m, st.l, st.acc
    d["os_final"] = ref_attn.online_softmax_finalize(st)
    # update_entry / forecast: 4 pushes at order 2 on a ragged tile
    e = None
    for t in range(4):
        o = rng.standard_normal((37, 12)).astype(np.float32)
        e = ref_attn.update_entry(e, o, 2)
        d[f"ue{t}_o"], d[f"ue{t}_stack"], d[f"ue{t}_valid"] = o, e.diff_stack, np.array(e.valid_orders)
        for k, n in ((1, 4), (3, 6)):
            for od in (0, 1, 2):
                d[f"ue{t}_fc_{k}_{n}_{od}"] = ref_attn.forecast(e, k, n, od)
    # tensor.py numerics
    x = rng.standard_normal((50, 24)).astype(np.float32) * 2
    w = (1 + 0.1 * rng.standard_normal(24)).astype(np.float32)
    d["t_x"], d["t_w"] = x, w
    d["t_rms"] = ref_tensor.rms_norm(x, w)
    pos = np.arange(50, dtype=np.float64) * 3 + 1
    d["t_pos"], d["t_rope"] = pos, ref_tensor.rope(x, pos)
    d["t_rope_vec"] = ref_tensor.rope(x[3], 7.0)
    d["t_softmax"] = ref_tensor.row_softmax(x)
    for pool in (1, 4, 7, 64):
        d[f"t_pool{pool}"] = ref_tensor.mean_pool_blocks(x, pool)
    a = rng.standard_normal((33, 20)).astype(np.float32)
    bm = rng.standard_normal((20, 9)).astype(np.float32)
    d["t_a"], d["t_b"], d["t_matmul"] = a, bm, ref_tensor.matmul(a, bm)
    q, k, v = (rng.standard_normal((40, 8)).astype(np.float32) for _ in range(3))
    d["t_q"], d["t_k"], d["t_v"] = q, k, v
    d["t_dense_attn"] = ref_tensor.dense_attention(q, k, v)
    # policy building blocks: several geometries, float32 q/k, small d
    cases = [(96, 8, 8, 8, 16), (100, 16, 4, 4, 9), (130, 4, 10, 5, 0), (256, 32, 8, 8, 40),
             (77, 12, 7, 7, 14)]
    for ci, (n, dd, pq_, pk_, n_text) in enumerate(cases):
        qc = rng.standard_normal((n, dd)).astype(np.float32)
        kc = (rng.standard_normal((n, dd)) * 1.5).astype(np.float32)
        m = ref_policy.compressed_attention(qc, kc, pq_, pk_, n_text)
        d[f"p{ci}_q"], d[f"p{ci}_k"] = qc, kc
        d[f"p{ci}_cfg"] = np.array([n, dd, pq_, pk_, n_text])
        d[f"p{ci}_map"], d[f"p{ci}_nt"] = m.p_tilde, np.array(m.n_t)
        c = ref_policy.vision_to_text_contribution(m)
        g = ref_policy.text_to_vision_guidance(m)
        d[f"p{ci}_contrib"], d[f"p{ci}_guid"] = c, g
        rows, cols = m.p_tilde.shape
        for ti, tau in enumerate((0.0, 0.3, 0.7, 1.0)):
            if rows == cols:
                d[f"p{ci}_cached{ti}"] = ref_policy.select_cached_blocks(c, g, tau)
            cbits = rng.random(rows) < 0.7
            d[f"p{ci}_cbits{ti}"] = cbits
            for guard in (True, False):
                d[f"p{ci}_keep{ti}_{int(guard)}"] = ref_policy.select_skip_blocks(m, cbits, tau * 0.6, guard=guard)
            d[f"p{ci}_degrade{ti}"] = ref_policy.degrade_to_full_cache(cbits, m.n_t, 0.25 * ti)
        if rows == cols and pq_ == pk_:
            for gi, (tq, tkv, sq, guard) in enumerate(((0.5, 0.3, 0.0, True), (0.8, 0.6, 0.5, False),
                                                      (0.2, 0.9, 0.1, True))):
                cb, sb = ref_policy.generate_masks(qc, kc, b_q=pq_, b_k=pk_, pool_n=1, n_text=n_text,
                                                   tau_q=tq, tau_kv=tkv, s_q=sq, guard=guard)
                d[f"p{ci}_gm{gi}_cfg"] = np.array([tq, tkv, sq, float(guard)])
                d[f"p{ci}_gm{gi}_cache"], d[f"p{ci}_gm{gi}_skip"] = cb, sb
    d["n_policy_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "api.npz", **d)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    if sys.argv[1:] == ["api"]:
        api()
        sys.exit(0)
    if sys.argv[1:] == ["run"]:
        pipeline_run()
        sys.exit(0)
    pipeline_run()
    policy()
    codec()
    attention()
    gemm_q()
    gemm_o()
    cache_push()
    api()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
