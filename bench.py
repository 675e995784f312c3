#!/usr/bin/env python
"""FlashOmni B200 hot-path benchmark (BASELINE.json metric).

A step = one dispatch step of the sparse hot path of one HunyuanVideo DiT
attention layer (C4: 33,024 tokens = 258 blocks of 128, 24 heads x 128,
d_model 3072): GEMM-Q (cached tiles dropped) -> sparse attention (cached
q-blocks and masked KV blocks skipped) -> GEMM-O dispatch (cached-head
K-blocks dropped, forecast bias added). Symbols are random 8-bit symbols in
the reference's random_masks rule (verify.py:29-44): 25% cached q-blocks, 50%
KV blocks skipped in active rows (62.5% pair sparsity). Inputs are resident in
HBM and larger than L2 (x, q, k, v, o are 203 MB each), so no flush is needed.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun): heads are sharded over ranks (C5): each rank runs its heads
and GEMM-O partial sums are all-reduced over NCCL inside the step.
"""

import argparse
import json
import os
import pathlib
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sparse attn/GEMM-Q/GEMM-O ms & speedup vs sparsity ratio, Hunyuan 33K tokens"
T = 128
CONFIGS = {
    "c4": dict(name="C4 HunyuanVideo attention layer, 33K tokens", seq=33024, heads=24, d_model=3072),
    "c1": dict(name="C1 single DiT attention layer, 4096 tokens", seq=4096, heads=24, d_model=3072),
    "c2": dict(name="C2 FLUX.1-dev joint attention, 4608 tokens", seq=4608, heads=24, d_model=3072),
    # C5: the C4 layer as a block stack (layer l's output is layer l+1's input);
    # 4 layers [choice], --layers overrides
    "c5": dict(name="C5 HunyuanVideo DiT block stack, 33K tokens", seq=33024, heads=24,
               d_model=3072, layers=4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cached", type=float, default=0.25, help="cached q-block ratio")
    ap.add_argument("--skip", type=float, default=0.5, help="KV block skip ratio in active rows")
    ap.add_argument("--interval", type=int, default=6)
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--elapsed", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also sweep sparsity (extra JSON key)")
    ap.add_argument("--layers", type=int, default=None, help="layers in the stack (c5: 4)")
    ap.add_argument("--eager", action="store_true",
                    help="launch the operators from Python each step instead of replaying "
                         "their CUDA graphs")
    return ap.parse_args()


def random_masks(rng, heads, t, cached_ratio, skip_ratio):
    """Vectorised verify.py:29-44 rule (pool_n = 1): cache density 1-cached,
    pair density 1-skip, >= 1 computed pair per active row, cached rows empty."""
    cache = rng.random((heads, t)) >= cached_ratio
    skip = rng.random((heads, t, t)) >= skip_ratio
    for h in range(heads):
        if not cache[h].any():
            cache[h, rng.integers(t)] = True
    empty = cache & ~skip.any(axis=2)
    hh, rr = np.nonzero(empty)
    skip[hh, rr, rng.integers(t, size=hh.size)] = True
    skip &= cache[:, :, None]
    return cache, skip


def peaks():
    """(bf16 burst TFLOP/s, bf16 sustained TFLOP/s, HBM GB/s, source) from the
    driver's MEASURED_PEAKS.json (keys as B200_PROFILING.md names them, at the
    top level or one level down), else the recipe's fallback."""
    fallback = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}
    p = ROOT / "MEASURED_PEAKS.json"
    if not p.exists():
        return (*fallback.values(), "fallback")
    d = json.loads(p.read_text())
    flat = dict(d)
    for v in d.values():
        if isinstance(v, dict):
            for k, x in v.items():
                flat.setdefault(k, x)
    got, src = [], "measured"
    for k, fb in fallback.items():
        v = flat.get(k)
        if isinstance(v, (int, float)) and v > 0:
            got.append(float(v))
        else:
            got.append(fb)
            src = "measured (fallback for missing keys)"
    return (*got, src)


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def _rows(self):
        self.f.flush()
        try:
            return [r for r in open(self.f.name).read().splitlines() if r.strip()]
        except OSError:
            return []

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        # nvidia-smi can take seconds to start: wait for its first sample so the
        # samples taken from here on cover the timed region
        t0 = time.time()
        while self.p is not None and not self._rows() and time.time() - t0 < 15:
            time.sleep(0.05)
        self.mark = max(len(self._rows()) - 1, 0)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            # one more sample taken at/after the end of the timed region
            n, t0 = len(self._rows()), time.time()
            while len(self._rows()) <= n and time.time() - t0 < 2:
                time.sleep(0.01)
            self.p.terminate()
            self.p.wait()

    def summary(self):
        rows = [r.split(",") for r in self._rows()[getattr(self, "mark", 0):]]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the reference CPU path on the host cores
# ---------------------------------------------------------------------------
def cpu_layer(args, cfg, cache_bits, skip_bits):
    """oracle.layer_cpu.CpuLayer: the reference's compiled attention kernel
    (oracle/_ref, built from /root/reference/.../_core.pyx) over one worker
    process per host core, plus the numpy GEMM-Q / GEMM-O of gemm.py."""
    from oracle.layer_cpu import CpuLayer

    return CpuLayer(cfg["seq"], cfg["heads"], cfg["d_model"], cache_bits, skip_bits,
                    seed=args.seed, order=args.order, elapsed=args.elapsed,
                    interval=args.interval)


def cpu_baseline(args, cfg, cache_bits, skip_bits, k=16):
    """Bounded sample for the B200 arm's line: slice 0 of a k-way interleaved
    partition of the layer (1/k of every head's active query blocks, 1/k of
    the GEMM tiles), scaled to the full layer by exact pair counts (attention)
    and by k (GEMMs)."""
    L = cpu_layer(args, cfg, cache_bits, skip_bits)
    try:
        L.run_slice(1, 256)  # warm the pool and the BLAS threads
        sec, parts, pairs = L.run_slice(0, k)
    finally:
        L.close()
    pairs_all = int(L.pairs_per_unit.sum())
    scale_attn = pairs_all / max(pairs, 1)
    full = {"attention": parts["attention"] * scale_attn * 1e3,
            "gemm_q": parts["gemm_q"] * k * 1e3, "gemm_o_dispatch": parts["gemm_o_dispatch"] * k * 1e3}
    sample = (f"1/{k} of the layer ({pairs} of {pairs_all} attention pairs, every {k}th active "
              f"(head, q-block) unit; 1/{k} of the GEMM-Q tiles and GEMM-O row blocks), "
              f"{sec:.1f} s measured, scaled to one full layer step by exact pair counts / {k}; "
              f"attention backend {L.backend} on {L.workers} worker processes")
    return sum(full.values()), sample, full, L


def cpu_threads():
    return os.cpu_count()


def run_reference(args, cfg, rank, world):
    """Reference arm: the reference CPU path on the host cores, rank 0 only.
    The K timed steps are the K slices of an interleaved partition of one
    layer step, so together they run the WHOLE layer exactly once; the value
    is their summed time (a measured full layer, not an extrapolation)."""
    if rank != 0:
        return
    rng = np.random.default_rng(args.seed)
    t = cfg["seq"] // T
    cache_bits, skip_bits = random_masks(rng, cfg["heads"], t, args.cached, args.skip)
    L = cpu_layer(args, cfg, cache_bits, skip_bits)
    try:
        for w in range(args.warmup):  # untimed: small slices of a 256-way partition
            L.run_slice(w, 256)
        total, parts_sum, pairs = 0.0, {}, 0
        for s in range(args.steps):
            sec, parts, p = L.run_slice(s, args.steps)
            total += sec
            pairs += p
            for k2, v2 in parts.items():
                parts_sum[k2] = parts_sum.get(k2, 0.0) + v2
    finally:
        L.close()
    nl = layers_of(args, cfg)
    v = total * 1e3 * nl
    assert pairs == int(L.pairs_per_unit.sum()), "the K slices must cover the layer exactly once"
    sample = (f"the whole layer step, as {args.steps} interleaved slices (one per timed step; "
              f"{pairs} attention pairs, all GEMM-Q tiles and GEMM-O row blocks); attention "
              f"backend {L.backend} on {L.workers} worker processes, GEMMs numpy/OpenBLAS")
    if nl > 1:
        sample += f"; one layer measured, x {nl} layers of the stack (same shapes and sparsity)"
    layers = [dict(cb=cache_bits, sb=skip_bits)] * nl
    parts_sum = {k: x * nl for k, x in parts_sum.items()}
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(v, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (N(0,1) tensors, random symbols)",
            "config": dict(config_json(args, cfg, world, layers),
                           launch="reference CPU path (compiled _core.pyx + numpy), no GPU"),
            "breakdown_ms": {k: round(x * 1e3, 3) for k, x in parts_sum.items()},
            "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cpu_threads(),
                             "kind": L.kind, "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def local_device():
    """This rank's GPU: LOCAL_RANK, or 0 for every rank under FO_BENCH_SHARE_GPU=1."""
    if os.environ.get("FO_BENCH_SHARE_GPU") == "1":
        return 0
    return int(os.environ.get("LOCAL_RANK", 0))


def layers_of(args, cfg):
    return args.layers if args.layers is not None else cfg.get("layers", 1)


def config_json(args, cfg, world, layers):
    H, t = cfg["heads"], cfg["seq"] // T
    computed = sum(int(sum(ly["sb"][h][ly["cb"][h]].sum() for h in range(H))) for ly in layers)
    L = len(layers)
    extra = {"layers": L} if L > 1 else {}
    return {"workload": cfg["name"], **extra, "seq": cfg["seq"], "heads": H, "head_dim": T,
            "d_model": cfg["d_model"], "b_q": T, "b_k": T, "pool_n": 1,
            "cached_ratio": args.cached, "kv_skip_ratio": args.skip,
            "pair_sparsity": round(1 - computed / (L * H * t * t), 4),
            "interval_n": args.interval, "order_d": args.order, "elapsed_k": args.elapsed,
            "symbols": "random (verify.py:29-44 rule), seed %d" % args.seed,
            "parallelism": "heads/%d" % world if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (x/q/k/v/o 203 MB each), no flush",
            "launch": ("eager Python calls" if getattr(args, "eager", True) else
                       "each operator replayed as a CUDA graph (as the engine runs steps)")}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args, cfg, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2509_25401_b200 as fo
    from paper_2509_25401_b200 import _lib

    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    group = dist.group.WORLD if world > 1 else None
    S, H, dm = cfg["seq"], cfg["heads"], cfg["d_model"]
    t = S // T
    L = layers_of(args, cfg)
    rng = np.random.default_rng(args.seed)
    heads = fo.shard_heads(H, world, rank)
    Hl = len(heads)
    g = torch.Generator(device=dev).manual_seed(args.seed)

    def randn(*shape, scale=1.0):
        return torch.randn(*shape, device=dev, generator=g) * scale

    x = randn(S, dm).bfloat16()
    dense_sym = fo.encode_symbols(np.ones((Hl, t), bool), np.ones((Hl, t, t), bool), 1)
    layers = []
    for li in range(L):
        # layer li: its own symbols (the next draws of the same rng), weights
        # (reference init, pipeline.py:145-159, packed once), cache and bias
        cb_l, sb_l = random_masks(rng, H, t, args.cached, args.skip)
        params = fo.LayerParams.from_reference(
            randn(H, dm, T, scale=dm ** -0.5), randn(H, dm, T, scale=dm ** -0.5),
            randn(H, dm, T, scale=dm ** -0.5), 1 + 0.05 * randn(H, T), 1 + 0.05 * randn(H, T),
            randn(H, T, dm, scale=T ** -0.5), heads=heads)
        k, v = fo.project_kv(x, params)
        sym = fo.encode_symbols(cb_l[heads], sb_l[heads], 1)
        cache = fo.FeatureCache(Hl, t, args.order, seq=S)
        for _ in range(args.order + 1):
            cache.push(randn(S, Hl, T).bfloat16())
        o_upd = randn(S, Hl, T).bfloat16()
        _, bias = fo.project_out_update(o_upd, params.w_out, sym, cache, args.order)
        _, bias_dense = fo.project_out_update(o_upd, params.w_out, dense_sym, cache, args.order)
        layers.append(dict(params=params, k=k, v=v, sym=sym, cache=cache, bias=bias,
                           bias_dense=bias_dense, cb=cb_l, sb=sb_l))
    cache_bits, skip_bits = layers[0]["cb"], layers[0]["sb"]
    params, k, v, cache = (layers[0][n] for n in ("params", "k", "v", "cache"))
    sym, bias, bias_dense = layers[0]["sym"], layers[0]["bias"], layers[0]["bias_dense"]
    q = torch.empty(S, Hl, T, dtype=torch.bfloat16, device=dev)
    o = torch.empty_like(q)
    outs = [torch.empty(S, dm, dtype=torch.bfloat16, device=dev) for _ in range(min(L, 2))]
    out = outs[0]
    torch.cuda.synchronize()

    def phase_fns(dense, li, xin, lo):
        ly = layers[li]
        sy = dense_sym if dense else ly["sym"]
        bs = ly["bias_dense"] if dense else ly["bias"]
        return [lambda: fo.project_q(xin, ly["params"].w_q, ly["params"].q_norm, sy, "dispatch",
                                     out=q, fill=None, check=False),
                lambda: fo.sparse_attention(q, ly["k"], ly["v"], sy, ly["cache"], None,
                                            args.elapsed, args.interval, args.order, mode="bias",
                                            out=o, fill=None, check=False),
                lambda: fo.project_out_dispatch(o, ly["params"].w_out, sy, bs, args.elapsed,
                                                args.interval, args.order, out=lo, check=False)]

    graphs = {}

    def phase_graphs(dense):
        """each layer's three operators as CUDA graphs (the engine replays its
        dispatch chains the same way, engine.py), captured once"""
        if dense not in graphs:
            cs = torch.cuda.Stream(device=dev)
            cs.wait_stream(torch.cuda.current_stream())
            gl, xin = [], x
            with torch.cuda.stream(cs):
                for li in range(L):
                    lo = outs[li % len(outs)]
                    gs = []
                    for fn in phase_fns(dense, li, xin, lo):
                        fn()  # first use outside capture (host-side tables, plans)
                        gr = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(gr, stream=cs):
                            fn()
                        gs.append(gr)
                    gl.append(gs)
                    xin = lo
            torch.cuda.current_stream().wait_stream(cs)
            torch.cuda.synchronize()
            graphs[dense] = gl
        return graphs[dense]

    def step(dense, ev=None):
        """one dispatch step through the stack; ev: per layer, 4 events"""
        gl = None if args.eager else phase_graphs(dense)
        xin = x
        for li in range(L):
            e = ev[li] if ev else None
            lo = outs[li % len(outs)]
            fns = phase_fns(dense, li, xin, lo) if gl is None else [g.replay for g in gl[li]]
            for k_ph in range(3):
                if e:
                    e[k_ph].record()
                fns[k_ph]()
            if group is not None:
                dist.all_reduce(lo, group=group)
            if e:
                e[3].record()
            xin = lo

    def timed(dense, steps, warm, clocks=None):
        for _ in range(warm):
            step(dense)
        evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(L)]
               for _ in range(steps)]
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()
        _lib.reset_launch_count()
        ctx = clocks if clocks is not None else _Null()
        with ctx:
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record()
            for s in range(steps):
                step(dense, evs[s])
            end.record()
            torch.cuda.synchronize()
        launches = _lib.launch_count() if args.eager else launches_per_step * steps
        if group is not None:
            dist.barrier()
        total = start.elapsed_time(end)
        # per-phase ms per step, summed over the layers
        parts = np.array([[sum(e[li][0].elapsed_time(e[li][1]) for li in range(L)),
                           sum(e[li][1].elapsed_time(e[li][2]) for li in range(L)),
                           sum(e[li][2].elapsed_time(e[li][3]) for li in range(L))]
                          for e in evs]).mean(axis=0)
        total_t = torch.tensor([total], device=dev)
        if group is not None:
            dist.all_reduce(total_t, op=dist.ReduceOp.MAX, group=group)
        return total_t.item() / steps, parts, launches

    # check once that the contract holds (errors are latched, not raised, while timing)
    step(False)
    fo._runtime.Status.default().check("bench warm-up")
    # kernels per step, counted on one eager step after the warm-up (graph replays
    # launch the same kernels)
    torch.cuda.synchronize()
    _lib.reset_launch_count()
    for fn_l in range(L):
        for fn in phase_fns(False, fn_l, x if fn_l == 0 else outs[(fn_l - 1) % len(outs)],
                            outs[fn_l % len(outs)]):
            fn()
    launches_per_step = _lib.launch_count()
    torch.cuda.synchronize()

    clocks = Clocks(dev.index) if rank == 0 else None
    ms, parts, launches = timed(False, args.steps, args.warmup, clocks)
    fo._runtime.Status.default().check("bench timed region")
    res = {"ms": ms, "parts": parts, "launches": launches}
    if not args.no_dense:
        dms, dparts, _ = timed(True, max(3, args.steps // 2), 2)
        res.update(dense_ms=dms, dense_parts=dparts)

    # e2e through the public API with host buffers: every step copies its x in
    # (pinned H2D) and its out back (D2H); pipeline.HostStepper overlaps step k's
    # compute with step k+1's input copy and step k-1's output copy
    e2e = None
    if not args.no_e2e and L == 1:
        state = fo.LayerState(params=params, cache=cache, symbols=sym, bias=bias)
        stepper = fo.HostStepper(state, S, dm, device=dev, group=group)
        x_host = [x.cpu().pin_memory() for _ in range(2)]
        out_host = [torch.empty(S, dm, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        for k in range(args.warmup):
            stepper.step(x_host[k & 1], out_host[k & 1], args.elapsed, args.interval, args.order)
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        _lib.reset_launch_count()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stepper.h2d)
        for k in range(args.steps):
            stepper.step(x_host[k & 1], out_host[k & 1], args.elapsed, args.interval, args.order)
        s1.record(stepper.d2h)
        torch.cuda.synchronize()
        e2e_launches = _lib.launch_count()
        et = torch.tensor([s0.elapsed_time(s1) / args.steps], device=dev)
        if group is not None:
            dist.all_reduce(et, op=dist.ReduceOp.MAX, group=group)
        fo._runtime.Status.default().check("bench e2e")
        e2e = {"value": round(et.item(), 3), "unit": "ms",
               "h2d_bytes_per_step": x.numel() * 2, "d2h_bytes_per_step": out.numel() * 2,
               "path": "pipeline.HostStepper -> dispatch_step (GEMM-Q, K/V projection, sparse "
                       "attention, GEMM-O dispatch); pinned host x in / out back every step, "
                       "copies overlapped with the neighbouring steps' compute",
               "gpu_launches_per_step": e2e_launches / args.steps}

    if rank != 0:
        return
    # ---------------- roofline of the dominant kernel (sparse attention)
    burst, sustained, hbm, src = peaks()
    computed = sum(int(sum(ly["sb"][h][ly["cb"][h]].sum() for h in heads)) for ly in layers)
    active = sum(int(ly["cb"][heads].sum()) for ly in layers)
    attn_flops = 4.0 * T * T * T * computed / L  # per launch (one per layer)
    # Q of active tiles, K and V of every (head, block), O of active tiles (bf16)
    attn_bytes = 2.0 * T * T * (2 * active / L + 2 * Hl * t)
    ach = attn_flops * L / (parts[1] * 1e-3) / 1e12
    kname = ("sparse_attention_kernel" if os.environ.get("FO_ATTN_IMPL") == "v1"
             else "sparse_attention_cs_kernel")
    traffic, traffic_src = ncu_traffic(kname, args)
    q_flops = 2.0 * dm * T * T * active
    o_flops = 2.0 * dm * T * T * active
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (N(0,1) activations, reference-init weights, random 8-bit symbols)",
        "config": config_json(args, cfg, world, layers),
        "breakdown_ms": {"gemm_q": round(parts[0], 4), "attention": round(parts[1], 4),
                         "gemm_o_dispatch": round(parts[2], 4)},
        "effective_tflops": {"gemm_q": round(q_flops / parts[0] / 1e9, 1),
                             "attention": round(ach, 1),
                             "gemm_o_dispatch": round(o_flops / parts[2] / 1e9, 1)},
        "gpu_launches": int(launches),
        # the timed region is ~0.1 s of back-to-back steps: the burst peak
        # applies (B200_PROFILING.md); the sustained-peak fraction is beside it
        "roofline": {"bound": "tensor", "achieved": round(ach, 1), "peak": burst,
                     "unit": "TFLOP/s", "frac": round(ach / burst, 4), "traffic": traffic,
                     "traffic_source": traffic_src, "kernel": kname,
                     "peak_source": f"{src} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                     "peak_sustained": sustained, "frac_sustained": round(ach / sustained, 4),
                     "algorithmic_flops_per_launch": attn_flops,
                     "algorithmic_hbm_bytes_per_launch": attn_bytes},
    }
    if "dense_ms" in res:
        dp = res["dense_parts"]
        s_attn = 1 - computed / (L * Hl * t * t)
        s_rows = 1 - active / (L * Hl * t)
        ideal = {"attention": 1 / (1 - s_attn), "gemm_q": 1 / (1 - s_rows),
                 "gemm_o_dispatch": 1 / (1 - s_rows)}
        sp = {"gemm_q": dp[0] / parts[0], "attention": dp[1] / parts[1],
              "gemm_o_dispatch": dp[2] / parts[2]}
        line["dense_ms"] = {"gemm_q": round(dp[0], 4), "attention": round(dp[1], 4),
                            "gemm_o_dispatch": round(dp[2], 4), "step": round(res["dense_ms"], 4)}
        line["speedup_vs_dense"] = {k2: round(v2, 3) for k2, v2 in sp.items()}
        line["speedup_vs_dense"]["step"] = round(res["dense_ms"] / ms, 3)
        line["ideal_speedup"] = {k2: round(v2, 3) for k2, v2 in ideal.items()}
        line["frac_sparsity_scaled_roofline"] = {k2: round(sp[k2] / ideal[k2], 3) for k2 in sp}
        n_int = args.interval
        line["gemm_o_amortized_ideal"] = round(n_int / (1 + (n_int - 1) * (1 - s_rows)), 3)
        dense_attn_tflops = 4.0 * T * T * T * L * Hl * t * t / (dp[1] * 1e-3) / 1e12
        line["dense_attention_tflops"] = round(dense_attn_tflops, 1)
    if clocks is not None:
        line["clocks"] = clocks.summary()
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu:
        cms, sample, cparts, CL = cpu_baseline(args, cfg, cache_bits, skip_bits)
        if L > 1:
            cms, cparts = cms * L, {k2: v2 * L for k2, v2 in cparts.items()}
            sample += f"; layer 0 sampled, x {L} layers of the stack"
        line["cpu_baseline"] = {"value": round(cms, 1), "unit": "ms", "cores": cpu_threads(),
                                "kind": CL.kind, "sample": sample,
                                "breakdown_ms": {k2: round(v2, 1) for k2, v2 in cparts.items()}}
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel, args):
    """DRAM bytes per launch of `kernel` from the committed ncu summary of the
    current kernels (profiles/ncu_current.json, written by
    tools/ncu_summary.py from a --set full capture of this bench's default
    workload). None when no capture of that kernel at this workload exists."""
    p = ROOT / "profiles" / "ncu_current.json"
    if not p.exists():
        return None, None
    try:
        d = json.loads(p.read_text())
        k = d["kernels"][kernel]
        w = d.get("workload", {})
        if (w.get("cached") not in (None, args.cached) or w.get("skip") not in (None, args.skip)
                or w.get("config", "c4") != args.config):
            return None, None
        return float(k["dram_bytes_per_launch"]), f"profiles/{d.get('source', 'ncu_current.json')}"
    except Exception:
        return None, None


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_device())
        # FO_BENCH_BACKEND=gloo with FO_BENCH_SHARE_GPU=1 runs N ranks on one GPU:
        # a functional check of the sharded path where only one GPU exists
        dist.init_process_group(os.environ.get("FO_BENCH_BACKEND", "nccl"))
    try:
        run_b200(args, cfg, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
