"""The reference's per-head GEMM signatures (reference gemm.py:44-229), on the GPU.

`project_q`, `project_out_update` and `project_out_dispatch` accept the
reference's calling convention too: numpy arrays, head-major o [heads, n, d],
one SymbolBuffer per head and any block size / head dim. Those calls land here
and follow the reference step for step, in float32, with every product on the
device (`fo_matmul_f32`), the RMS norm and rotary encoding on the device
kernels of tensor.py, and the reference's shapes for the returned objects
(`ReferenceCachedBias`: one stack per block, orders, active heads). The
layer-level calls (device bf16 [S, H, 128], DeviceSymbols) keep the tcgen05
kernels of gemm.py; this module is the compatibility surface of the drop-in,
not the hot path.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._runtime import require_cuda, stream_ptr
from .attention import forecast_coefficients
from .errors import ParameterError, ShapeError, StateError
from .symbols import DeviceSymbols, ceil_div
from .tensor import rms_norm, rope

DTYPE = np.float32


def is_reference_call(a, symbols, b_q, d):
    """The reference convention: host arrays, a per-head symbol list, or a
    geometry the tcgen05 kernels do not tile (b_q != 128, head dim != 128)."""
    return (not isinstance(a, torch.Tensor) or isinstance(symbols, (list, tuple))
            or b_q != 128 or d != 128)


def _f32(a, name, ndim=None, finite=True):
    host = not isinstance(a, torch.Tensor)
    t = torch.as_tensor(np.asarray(a, dtype=DTYPE)) if host else a
    t = t.to("cuda", torch.float32).contiguous()
    if ndim is not None and t.dim() != ndim:
        raise ShapeError(f"{name}: expected a {ndim}-D array, got shape {tuple(t.shape)}")
    if finite and not bool(torch.isfinite(t).all()):
        raise ParameterError(f"{name}: contains NaN or Inf")
    return t, host


def _mm(a, b, c, accumulate):
    """c (+)= a @ b, fp32 row-major, on the device (views must be row-contiguous)."""
    m, k = a.shape
    n = b.shape[1]
    _lib.call("fo_matmul_f32", a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
              1 if accumulate else 0, stream_ptr(None))


def _active(symbols, heads, t_q):
    """gemm.py:38-41 _active_blocks for every head: bool [t_q, heads]."""
    syms = list(symbols) if isinstance(symbols, (list, tuple)) else symbols
    if isinstance(syms, DeviceSymbols):
        ds = syms
    else:
        if len(syms) != heads:
            raise ShapeError(f"{len(syms)} symbol buffers for {heads} heads")
        for s in syms:
            if s.rows != t_q:
                raise ShapeError(f"symbols have {s.rows} rows, expected {t_q}")
        ds = DeviceSymbols.from_buffers(syms)
    if ds.rows != t_q:
        raise ShapeError(f"symbols have {ds.rows} rows, expected {t_q}")
    act, _ = ds.decoded()
    return act.t().bool().cpu().numpy()


def _rows(active_blocks, b_q, n):
    starts = np.flatnonzero(active_blocks) * b_q
    if not starts.size:
        return np.empty(0, dtype=np.int64)
    return np.concatenate([np.arange(s, min(s + b_q, n)) for s in starts])


def project_q(x, w_q, norm_weight, symbols, phase, *, b_q, positions=None, eps=1e-6,
              counters=None, fill=0.0):
    """gemm.py:44-93: out [heads, n, d]; rows of cached blocks hold `fill`."""
    require_cuda()
    xt, host = _f32(x, "x", 2)
    w, _ = _f32(w_q, "w_q", 3, finite=False)
    if phase not in ("update", "dispatch"):
        raise ParameterError(f"unknown phase {phase!r}")
    heads, d_model, d = w.shape
    n = xt.shape[0]
    if xt.shape[1] != d_model:
        raise ShapeError(f"x width {xt.shape[1]} != projection input {d_model}")
    nw, _ = _f32(norm_weight, "norm_weight", 2, finite=False)
    pos = np.arange(n) if positions is None else np.asarray(positions)
    t_q = ceil_div(n, b_q)
    act = None if phase == "update" else _active(symbols, heads, t_q)
    out = torch.full((heads, n, d), float(fill), dtype=torch.float32, device="cuda")
    for h in range(heads):
        rows = np.arange(n) if phase == "update" else _rows(act[:, h], b_q, n)
        if rows.size:
            ri = torch.from_numpy(rows).cuda()
            y = torch.empty(rows.size, d, dtype=torch.float32, device="cuda")
            _mm(xt.index_select(0, ri).contiguous(), w[h].contiguous(), y, False)
            y = rope(rms_norm(y, nw[h], eps), pos[rows])
            out[h].index_copy_(0, ri, y)
        if counters is not None:
            counters.q_macs_dense += n * d_model * d
            counters.q_macs_actual += int(rows.size) * d_model * d
    return out.cpu().numpy() if host else out


@dataclass
class ReferenceCachedBias:
    """The reference's CachedBias (gemm.py:96-107): stacks[i][d] is block i's
    d-th bias level [rows, d_model] (shape [0, ...] without cached heads),
    orders[i] its populated levels, active_heads [t_q, heads]."""

    stacks: list
    orders: np.ndarray
    active_heads: np.ndarray


def _entry_stack(cache, h, i):
    e = cache.device_entry(h, i) if getattr(cache, "per_entry", False) else cache.entry(h, i)
    if e is None:
        return None
    st = e.diff_stack
    return st if isinstance(st, torch.Tensor) else torch.from_numpy(np.asarray(st, DTYPE)).cuda()


def project_out_update(o_heads, w_out, symbols_next, cache, order_d, *, b_q, counters=None):
    """gemm.py:110-175: (out [n, d_model], ReferenceCachedBias)."""
    require_cuda()
    o, host = _f32(o_heads, "o_heads", 3, finite=False)
    w, _ = _f32(w_out, "w_out", 3, finite=False)
    heads, n, d = o.shape
    d_model = w.shape[2]
    t_q = ceil_div(n, b_q)
    act = _active(symbols_next, heads, t_q)
    stacks, orders = [], np.zeros(t_q, dtype=int)
    out = torch.zeros(n, d_model, dtype=torch.float32, device="cuda")
    for i in range(t_q):
        r0, r1 = i * b_q, min(i * b_q + b_q, n)
        nr = r1 - r0
        cached = np.flatnonzero(~act[i])
        if cached.size:
            n_orders = min(order_d + 1, min(cache.valid_orders(int(h), i) for h in cached))
            if n_orders < 1:
                raise StateError(f"block {i}: a to-be-cached head has a cold cache")
            stack = torch.zeros(n_orders, nr, d_model, dtype=torch.float32, device="cuda")
            for h in cached:
                st = _entry_stack(cache, int(h), i)
                for dd in range(n_orders):
                    _mm(st[dd].contiguous(), w[h].contiguous(), stack[dd], True)
            stacks.append(stack)
            orders[i] = n_orders
            out[r0:r1] += stack[0]
            if counters is not None:
                counters.o_macs_actual += cached.size * nr * d * d_model
                counters.o_bias_macs += cached.size * (n_orders - 1) * nr * d * d_model
        else:
            stacks.append(torch.zeros(0, nr, d_model, dtype=torch.float32, device="cuda"))
        for h in np.flatnonzero(act[i]):
            _mm(o[h, r0:r1].contiguous(), w[h].contiguous(), out[r0:r1], True)
            if counters is not None:
                counters.o_macs_actual += nr * d * d_model
    if counters is not None:
        counters.o_macs_dense += heads * n * d * d_model
    if host:
        return out.cpu().numpy(), ReferenceCachedBias([s.cpu().numpy() for s in stacks], orders, act)
    return out, ReferenceCachedBias(stacks, orders, act)


def project_out_dispatch(o_heads, w_out, symbols, bias, elapsed_k, interval_n, order_d, *, b_q,
                         counters=None):
    """gemm.py:178-229: active heads plus the forecast of the bias stacks."""
    require_cuda()
    o, host = _f32(o_heads, "o_heads", 3, finite=False)
    w, _ = _f32(w_out, "w_out", 3, finite=False)
    heads, n, d = o.shape
    d_model = w.shape[2]
    t_q = ceil_div(n, b_q)
    if bias is None:
        raise StateError("dispatch projection requires the update-step bias")
    if interval_n < 1 or not 1 <= elapsed_k <= interval_n - 1:
        raise ParameterError(f"elapsed_k={elapsed_k} outside [1, {interval_n - 1}]")
    act = _active(symbols, heads, t_q)
    if not np.array_equal(act, np.asarray(bias.active_heads, bool)):
        raise StateError("bias was generated under different cache symbols")
    out = torch.zeros(n, d_model, dtype=torch.float32, device="cuda")
    for i in range(t_q):
        r0, r1 = i * b_q, min(i * b_q + b_q, n)
        nr = r1 - r0
        for h in np.flatnonzero(act[i]):
            _mm(o[h, r0:r1].contiguous(), w[h].contiguous(), out[r0:r1], True)
            if counters is not None:
                counters.o_macs_actual += nr * d * d_model
        if bias.orders[i]:
            n_orders = min(order_d + 1, int(bias.orders[i]))
            coeffs = forecast_coefficients(elapsed_k, interval_n, n_orders)
            st = bias.stacks[i]
            st = st if isinstance(st, torch.Tensor) else torch.from_numpy(np.asarray(st, DTYPE)).cuda()
            for dd in range(n_orders):
                out[r0:r1] += float(coeffs[dd]) * st[dd]
            if counters is not None:
                counters.o_bias_macs += n_orders * nr * d_model
    if counters is not None:
        counters.o_macs_dense += heads * n * d * d_model
    return out.cpu().numpy() if host else out
