"""Sparse projections around the attention core, on the GPU (reference gemm.py).

GEMM-Q (project_q) skips the (block, head) output tiles whose cache symbol
is 0 — RMS norm and rotary encoding are token-local, so dropping rows is exact
and both run in the tcgen05 epilogue. GEMM-O runs in two stages: at update
steps (project_out_update) heads the next window will cache are projected once
into per-block bias stacks B_c[d]; dispatch steps (project_out_dispatch)
multiply only active heads and add the forecast sum_d c_d B_c[d].

Layouts: x bf16 [seq, d_model]; q/o bf16 [seq, heads, 128]; weights are packed
once (pack_w_q / pack_w_out) into the K-major layouts the TMA descriptors read.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, gemm_ref
from ._runtime import (TILE, Status, as_device, check_bsd, check_finite, check_out, require_cuda,
                       stream_ptr)
from .attention import check_elapsed, ctypes_floats, forecast_coefficients
from .errors import ParameterError, ShapeError, StateError
from .symbols import DeviceSymbols, ceil_div

ROPE_BASE = 10000.0


@dataclass
class GemmCounters:
    """Multiply-accumulate counts for the projection paths (gemm.py:22-35)."""

    q_macs_dense: int = 0
    q_macs_actual: int = 0
    o_macs_dense: int = 0
    o_macs_actual: int = 0
    o_bias_macs: int = 0


# ---------------------------------------------------------------------------
# weight packing and rotary tables (host prep, done once per layer / shape)
# ---------------------------------------------------------------------------
class PackedWeight:
    """A projection weight resident in HBM in the kernel's K-major layout."""

    def __init__(self, t, heads, d_model):
        self.t, self.heads, self.d_model = t, heads, d_model


def pack_w_q(w_q):
    """Reference w_q [heads, d_model, 128] -> bf16 [heads*128, d_model]."""
    if isinstance(w_q, PackedWeight):
        return w_q
    w = as_device(w_q, torch.float32, "w_q")
    if w.dim() != 3 or w.shape[2] != TILE:
        raise ShapeError(f"w_q: expected [heads, d_model, {TILE}], got {tuple(w.shape)}")
    heads, dm, _ = w.shape
    t = w.permute(0, 2, 1).reshape(heads * TILE, dm).to(torch.bfloat16).contiguous()
    return PackedWeight(t, heads, dm)


def pack_w_out(w_out):
    """Reference w_out [heads, 128, d_model] -> bf16 [d_model, heads*128]."""
    if isinstance(w_out, PackedWeight):
        return w_out
    w = as_device(w_out, torch.float32, "w_out")
    if w.dim() != 3 or w.shape[1] != TILE:
        raise ShapeError(f"w_out: expected [heads, {TILE}, d_model], got {tuple(w.shape)}")
    heads, _, dm = w.shape
    t = w.reshape(heads * TILE, dm).t().to(torch.bfloat16).contiguous()
    return PackedWeight(t, heads, dm)


_ROPE = {}


def rope_tables(seq, positions=None, device=None):
    """cos/sin of pos * base^(-2j/d) in float64 cast to float32, exactly as
    tensor.py:83-109 computes them. Returns fp32 [seq, 64] each (cached)."""
    key = (int(seq), None if positions is None else np.asarray(positions).tobytes(), str(device))
    if key not in _ROPE:
        pos = np.arange(seq, dtype=np.float64) if positions is None else np.asarray(positions, np.float64)
        if pos.shape != (seq,):
            raise ShapeError("rope: need one position per row")
        j = np.arange(TILE // 2, dtype=np.float64)
        theta = ROPE_BASE ** (-2.0 * j / TILE)
        ang = pos[:, None] * theta
        dev = device or "cuda"
        _ROPE[key] = (torch.from_numpy(np.cos(ang).astype(np.float32)).to(dev),
                      torch.from_numpy(np.sin(ang).astype(np.float32)).to(dev))
    return _ROPE[key]


def _norm(norm_weight, heads):
    w = as_device(norm_weight, torch.float32, "norm_weight")
    if tuple(w.shape) != (heads, TILE):
        raise ShapeError(f"norm weight shape {tuple(w.shape)} != {(heads, TILE)}")
    return w


# ---------------------------------------------------------------------------
# GEMM-Q
# ---------------------------------------------------------------------------
def project_q(x, w_q, norm_weight, symbols, phase, *, b_q=TILE, positions=None, eps=1e-6,
              counters=None, fill=0.0, out=None, rope=True, stream=None, status=None, check=True,
              plan=None):
    """Per-head query projection -> RMS norm -> rotary encoding (gemm.py:44-93).

    Update phase projects every tile; dispatch phase only the (block, head)
    tiles whose cache symbol is 1. Skipped tiles keep `fill` (pass NaN to trap
    illegal reads; fill=None leaves `out` untouched). norm_weight=None skips
    the RMS norm and rope=False the rotary encoding (the plain V projection).
    The reference's own convention (numpy arrays, one SymbolBuffer per head,
    any b_q / head dim; out [heads, n, d]) runs gemm_ref.project_q.
    """
    if not isinstance(w_q, PackedWeight) and gemm_ref.is_reference_call(
            x, symbols, b_q, np.shape(w_q)[-1]):
        return gemm_ref.project_q(x, w_q, norm_weight, symbols, phase, b_q=b_q,
                                  positions=positions, eps=eps, counters=counters,
                                  fill=0.0 if fill is None else fill)
    require_cuda()
    if phase not in ("update", "dispatch"):
        raise ParameterError(f"unknown phase {phase!r}")
    if b_q != TILE:
        raise ParameterError(f"the sm_100a kernels tile blocks of {TILE} tokens")
    w = pack_w_q(w_q)
    x = as_device(x, torch.bfloat16, "x")
    if x.dim() != 2:
        raise ShapeError(f"x: expected a 2-D matrix, got shape {tuple(x.shape)}")
    n, dm = x.shape
    if dm != w.d_model:
        raise ShapeError(f"x width {dm} != projection input {w.d_model}")
    heads = w.heads
    t_q = ceil_div(n, TILE)
    if check:  # gemm.py:64 as_matrix(x)
        check_finite(x, "x", status, stream=stream)
    nw = _norm(norm_weight, heads) if norm_weight is not None else None
    cs, sn = rope_tables(n, positions, x.device) if rope else (None, None)
    if out is None:
        out = torch.full((n, heads, TILE), 0.0 if fill is None else float(fill),
                         dtype=torch.bfloat16, device=x.device)
    else:
        check_out(out, "out", (n, heads, TILE), device=x.device)
    if phase == "dispatch":
        if symbols is None or symbols.heads != heads or symbols.rows != t_q:
            raise ShapeError(f"symbols must cover {heads} heads x {t_q} blocks")
        if plan is None:
            plan = symbols.plan(status=status, stream=stream, check=check)
    else:
        plan = None
    _lib.call("fo_gemm_q", x.data_ptr(), n, dm, w.t.data_ptr(), heads, TILE, _lib.ptr(nw),
              _lib.ptr(cs), _lib.ptr(sn), float(eps), None if plan is None else plan.ptr(),
              1 if phase == "update" else 0, out.data_ptr(), stream_ptr(stream))
    if counters is not None:
        counters.q_macs_dense += heads * n * dm * TILE
        if phase == "update":
            counters.q_macs_actual += heads * n * dm * TILE
        else:
            rows = 0
            for h, i in plan.gq_items():
                rows += min(TILE, n - int(i) * TILE)
            counters.q_macs_actual += rows * dm * TILE
    return out


def pack_w_qkv(w_q, w_k, w_v):
    """[W_q^T; W_k^T; W_v^T] bf16 [3*heads*128, d_model] for the fused
    projection (one weight, one TMA map)."""
    q, k, v = pack_w_q(w_q), pack_w_q(w_k), pack_w_q(w_v)
    if not (q.heads == k.heads == v.heads and q.d_model == k.d_model == v.d_model):
        raise ShapeError("w_q / w_k / w_v disagree on heads or d_model")
    return PackedWeight(torch.cat([q.t, k.t, v.t], 0).contiguous(), q.heads, q.d_model)


def project_qkv(x, w_qkv, q_norm, k_norm, symbols, phase, *, positions=None, eps=1e-6,
                q_out=None, k_out=None, v_out=None, fill=None, stream=None, status=None,
                check=True, plan=None):
    """The dispatch step's three projections (pipeline.py:223-234 with
    gemm.py:44-93) in ONE launch that reads x once: q = rope(rms_norm(x W_q))
    for the active tiles (every tile in the update phase), k = rope(rms_norm(x
    W_k)) and v = x W_v densely. w_qkv: pack_w_qkv(...). Returns (q, k, v)."""
    require_cuda()
    if phase not in ("update", "dispatch"):
        raise ParameterError(f"unknown phase {phase!r}")
    x = as_device(x, torch.bfloat16, "x")
    if x.dim() != 2:
        raise ShapeError(f"x: expected a 2-D matrix, got shape {tuple(x.shape)}")
    n, dm = x.shape
    if dm != w_qkv.d_model:
        raise ShapeError(f"x width {dm} != projection input {w_qkv.d_model}")
    heads = w_qkv.heads
    if tuple(w_qkv.t.shape) != (3 * heads * TILE, dm):
        raise ShapeError("w_qkv: expected the packed [W_q; W_k; W_v] (pack_w_qkv)")
    t_q = ceil_div(n, TILE)
    if check:  # gemm.py:64 as_matrix(x)
        check_finite(x, "x", status, stream=stream)
    qn, kn = _norm(q_norm, heads), _norm(k_norm, heads)
    cs, sn = rope_tables(n, positions, x.device)
    outs = []
    for name, o in (("q_out", q_out), ("k_out", k_out), ("v_out", v_out)):
        if o is None:
            # q's skipped tiles keep `fill`; k and v are written everywhere
            f = fill if (name == "q_out" and fill is not None) else 0.0
            o = torch.full((n, heads, TILE), float(f), dtype=torch.bfloat16, device=x.device)
        else:
            check_out(o, name, (n, heads, TILE), device=x.device)
        outs.append(o)
    if phase == "dispatch":
        if symbols is None or symbols.heads != heads or symbols.rows != t_q:
            raise ShapeError(f"symbols must cover {heads} heads x {t_q} blocks")
        if plan is None:
            plan = symbols.plan(status=status, stream=stream, check=check)
    else:
        plan = None
    _lib.call("fo_gemm_qkv", x.data_ptr(), n, dm, w_qkv.t.data_ptr(), heads, TILE, qn.data_ptr(),
              kn.data_ptr(), cs.data_ptr(), sn.data_ptr(), float(eps),
              None if plan is None else plan.ptr(), 1 if phase == "update" else 0,
              outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), stream_ptr(stream))
    return tuple(outs)


# ---------------------------------------------------------------------------
# GEMM-O
# ---------------------------------------------------------------------------
@dataclass
class CachedBias:
    """Output-projected contribution of to-be-cached heads (gemm.py:96-107).

    stacks: bf16 [order+1, seq, d_model] — row block i of stacks[d] is the
    reference's stacks[i][d]; orders int32 [t_q] (device) counts populated
    levels; symbols are the cache symbols the bias was built under (their
    decoded active-head matrix is the reference's active_heads).
    """

    stacks: torch.Tensor
    orders: torch.Tensor
    symbols: DeviceSymbols
    order_d: int

    @property
    def active_heads(self):
        active, _ = self.symbols.decoded()
        return active.t().bool().cpu().numpy()


def project_out_update(o_heads, w_out, symbols_next, cache, order_d, *, b_q=TILE, counters=None,
                       out=None, bias=None, stream=None, status=None, check=True, plan=None):
    """Update-step output projection, two stages in one pass (gemm.py:110-175).
    Returns (out bf16 [seq, d_model], CachedBias). The reference's convention
    (o_heads [heads, n, d], one SymbolBuffer per head, any b_q / head dim)
    runs gemm_ref.project_out_update and returns its ReferenceCachedBias."""
    if not isinstance(w_out, PackedWeight) and gemm_ref.is_reference_call(
            o_heads, symbols_next, b_q, np.shape(w_out)[1]):
        return gemm_ref.project_out_update(o_heads, w_out, symbols_next, cache, order_d, b_q=b_q,
                                           counters=counters)
    require_cuda()
    if b_q != TILE:
        raise ParameterError(f"the sm_100a kernels tile blocks of {TILE} tokens")
    o = check_bsd(o_heads, "o_heads")
    n, heads = o.shape[0], o.shape[1]
    w = pack_w_out(w_out)
    if w.heads != heads:
        raise ShapeError(f"w_out has {w.heads} heads, o has {heads}")
    dm = w.d_model
    t_q = ceil_div(n, TILE)
    if order_d < 0 or order_d > 3:
        raise ParameterError(f"order_d must be in [0, 3], got {order_d}")
    if cache is None or (cache.heads, cache.n_blocks) != (heads, t_q) or cache.stacks is None:
        raise StateError("update projection needs the refreshed feature cache")
    if order_d > cache.order:
        raise ParameterError(f"order_d {order_d} exceeds the cache order {cache.order}")
    if symbols_next.heads != heads or symbols_next.rows != t_q:
        raise ShapeError(f"symbols must cover {heads} heads x {t_q} blocks")
    st = status or Status.default()
    if plan is None:
        plan = symbols_next.plan(valid=cache.valid, valid_version=cache.version, order_d=order_d,
                                 status=st, stream=stream, check=check)
    if out is None:
        out = torch.empty(n, dm, dtype=torch.bfloat16, device=o.device)
    else:
        check_out(out, "out", (n, dm), device=o.device)
    if bias is not None:
        check_out(bias.stacks, "bias.stacks", (order_d + 1, n, dm), device=o.device)
        check_out(bias.orders, "bias.orders", (t_q,), dtype=torch.int32, device=o.device)
        stacks = bias.stacks
    else:
        stacks = torch.empty(order_d + 1, n, dm, dtype=torch.bfloat16, device=o.device)
    # the cache stacks are [cache.order+1, seq, H*128]; the kernel addresses slot d < order_d+1
    _lib.call("fo_gemm_o_update", o.data_ptr(), cache.stacks.data_ptr(), w.t.data_ptr(), n, heads,
              TILE, dm, order_d, plan.ptr(), out.data_ptr(), stacks.data_ptr(), st.ptr(),
              stream_ptr(stream))
    if bias is not None:
        bias.orders.copy_(plan.orders_tensor())
        orders = bias.orders
    else:
        orders = plan.orders_tensor().clone()
    if check:
        st.check("project_out_update")
    if counters is not None:
        counters.o_macs_dense += heads * n * TILE * dm
        counters.o_macs_actual += heads * n * TILE * dm
        hm = plan.hmask()
        ords = orders.cpu().numpy()
        for i in range(t_q):
            ncached = heads - bin(int(hm[i])).count("1")
            rows = min(TILE, n - i * TILE)
            if ncached:
                counters.o_bias_macs += ncached * (int(ords[i]) - 1) * rows * TILE * dm
    return out, CachedBias(stacks=stacks, orders=orders, symbols=symbols_next, order_d=order_d)


def project_out_dispatch(o_heads, w_out, symbols, bias, elapsed_k, interval_n, order_d, *, b_q=TILE,
                         counters=None, out=None, stream=None, status=None, check=True, plan=None,
                         blocks=None, max_sms=0):
    """Dispatch-step output projection (gemm.py:178-229): active heads plus the
    forecast of the cached-head bias stacks. blocks=(b0, b1) computes only the
    rows of query blocks [b0, b1) (the rest of `out` is untouched) on at most
    max_sms SMs (0 = all): the row chunks the multi-GPU step overlaps with the
    all-reduce (pipeline.dispatch_step). A ReferenceCachedBias or the
    reference's convention runs gemm_ref.project_out_dispatch."""
    if isinstance(bias, gemm_ref.ReferenceCachedBias) or (
            not isinstance(w_out, PackedWeight) and gemm_ref.is_reference_call(
                o_heads, symbols, b_q, np.shape(w_out)[1])):
        return gemm_ref.project_out_dispatch(o_heads, w_out, symbols, bias, elapsed_k, interval_n,
                                             order_d, b_q=b_q, counters=counters)
    require_cuda()
    if b_q != TILE:
        raise ParameterError(f"the sm_100a kernels tile blocks of {TILE} tokens")
    o = check_bsd(o_heads, "o_heads")
    n, heads = o.shape[0], o.shape[1]
    w = pack_w_out(w_out)
    dm = w.d_model
    t_q = ceil_div(n, TILE)
    if bias is None:
        raise StateError("dispatch projection requires the update-step bias")
    check_elapsed(elapsed_k, interval_n)
    if symbols.heads != heads or symbols.rows != t_q:
        raise ShapeError(f"symbols must cover {heads} heads x {t_q} blocks")
    st = status or Status.default()
    if bias.symbols is not symbols:
        # stale-symbol check (gemm.py:205-209) on the device
        _lib.call("fo_check_active_match", symbols.s_c.data_ptr(), bias.symbols.s_c.data_ptr(),
                  heads, t_q, symbols.pool_n, st.ptr(), stream_ptr(stream))
        if check:
            st.check("project_out_dispatch")
    if plan is None:
        plan = symbols.plan(status=st, stream=stream, check=check)
    coef = ctypes_floats(forecast_coefficients(elapsed_k, interval_n, order_d + 1))
    if bias.stacks.dim() != 3 or bias.stacks.shape[0] < min(order_d, bias.order_d) + 1:
        raise ShapeError(f"bias.stacks {tuple(bias.stacks.shape)} holds fewer than "
                         f"{min(order_d, bias.order_d) + 1} orders")
    check_out(bias.stacks, "bias.stacks", (bias.stacks.shape[0], n, dm), device=o.device)
    check_out(bias.orders, "bias.orders", (t_q,), dtype=torch.int32, device=o.device)
    if out is None:
        out = torch.empty(n, dm, dtype=torch.bfloat16, device=o.device)
    else:
        check_out(out, "out", (n, dm), device=o.device)
    b0, b1 = (0, t_q) if blocks is None else (int(blocks[0]), int(blocks[1]))
    _lib.call("fo_gemm_o_dispatch_rows", o.data_ptr(), w.t.data_ptr(), bias.stacks.data_ptr(),
              bias.orders.data_ptr(), n, heads, TILE, dm, min(order_d, bias.order_d),
              ctypes.addressof(coef), plan.ptr(), b0, b1, int(max_sms), out.data_ptr(),
              stream_ptr(stream))
    if counters is not None:
        counters.o_macs_dense += heads * sum(min(TILE, n - i * TILE) for i in range(b0, b1)) * TILE * dm
        hm = plan.hmask()
        ords = bias.orders.cpu().numpy()
        for i in range(b0, b1):
            rows = min(TILE, n - i * TILE)
            counters.o_macs_actual += bin(int(hm[i])).count("1") * rows * TILE * dm
            if ords[i]:
                counters.o_bias_macs += min(order_d + 1, int(ords[i])) * rows * dm
    return out
