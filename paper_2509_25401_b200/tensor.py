"""Dense reference numerics on the device (reference tensor.py:1-126).

The reference keeps its ground-truth helpers here: float32 matrices, a stable
row softmax, the dense attention oracle, token-wise RMS normalisation,
interleaved rotary encoding and block mean pooling, all accumulating in
float64 and rounding once. The same functions run here on the GPU:
`mean_pool_blocks`, `rms_norm`, `rope` and `row_softmax` are sm_100a kernels
(csrc/fo_numerics.cu) that follow numpy's summation orders, so they match the
reference bit for bit; `matmul` and the two products inside `dense_attention`
are float64 cuBLAS GEMMs rounded to float32 (numpy's float64 BLAS has no fixed
order either). These are the operator API's dense helpers, not the layer's hot
path.

Inputs may be numpy arrays (the reference's calling convention; results come
back as numpy float32) or torch tensors (results stay on the device).
"""

import numpy as np
import torch

from . import _lib
from ._runtime import require_cuda, stream_ptr
from .errors import ParameterError, ShapeError

DTYPE = np.float32
ROPE_BASE = 10000.0


def _dev(a, name, ndim=None, check_finite=False):
    """(fp32 contiguous CUDA tensor, came-from-numpy flag)."""
    require_cuda()
    host = not isinstance(a, torch.Tensor)
    t = torch.as_tensor(np.asarray(a, dtype=DTYPE)) if host else a
    t = t.to("cuda" if host or not t.is_cuda else t.device, torch.float32).contiguous()
    if ndim is not None and t.dim() != ndim:
        raise ShapeError(f"{name}: expected a {ndim}-D matrix, got shape {tuple(t.shape)}")
    if check_finite and not bool(torch.isfinite(t).all()):
        raise ParameterError(f"{name}: contains NaN or Inf")
    return t, host


def _ret(t, host):
    return t.cpu().numpy() if host else t


def as_matrix(a, name="matrix", check_finite=True):
    """tensor.py:19-30: a C-contiguous float32 2-D matrix, finite unless told otherwise."""
    t, host = _dev(a, name, ndim=2, check_finite=check_finite)
    return _ret(t, host)


def matmul(a, b):
    """tensor.py:33-39: float64 product rounded to float32 (cuBLAS DGEMM)."""
    ta, host = _dev(a, "a", 2, True)
    tb, _ = _dev(b, "b", 2, True)
    if ta.shape[1] != tb.shape[0]:
        raise ShapeError(f"matmul: inner dims differ ({tuple(ta.shape)} x {tuple(tb.shape)})")
    return _ret((ta.double() @ tb.double()).float(), host)


def row_softmax(s):
    """tensor.py:42-47: per-row max subtraction, float64 exp and numpy's
    pairwise row sum, rounded to float32 (fo_row_softmax)."""
    t, host = _dev(s, "scores", 2, True)
    out = torch.empty_like(t)
    _lib.call("fo_row_softmax", t.data_ptr(), t.shape[0], t.shape[1], out.data_ptr(),
              stream_ptr())
    return _ret(out, host)


def dense_attention(q, k, v):
    """tensor.py:50-65: softmax(q kᵀ / sqrt(d)) v, the oracle every sparse path
    is checked against. Scores in float64 (cuBLAS), softmax and the final
    float64 product as the reference rounds them."""
    tq, host = _dev(q, "q", 2, True)
    tk, _ = _dev(k, "k", 2, True)
    tv, _ = _dev(v, "v", 2, True)
    if not (tq.shape[1] == tk.shape[1] == tv.shape[1]) or tk.shape[0] != tv.shape[0]:
        raise ShapeError(f"attention operands inconsistent: q{tuple(tq.shape)} k{tuple(tk.shape)} "
                         f"v{tuple(tv.shape)}")
    d = tq.shape[1]
    scores = ((tq.double() @ tk.double().T) / np.sqrt(d)).float().contiguous()
    p = row_softmax(scores)
    return _ret((p.double() @ tv.double()).float(), host)


def rms_norm(x, weight, eps=1e-6):
    """tensor.py:68-80: y = x * w / sqrt(mean(x^2) + eps) along the last axis,
    mean in float64 (fo_rms_norm)."""
    tx, host = _dev(x, "x")
    tw, _ = _dev(weight, "weight")
    if tx.shape[-1] != tw.shape[-1]:
        raise ShapeError(f"rms_norm: dim mismatch {tx.shape[-1]} vs {tw.shape[-1]}")
    d = tx.shape[-1]
    out = torch.empty_like(tx)
    _lib.call("fo_rms_norm", tx.data_ptr(), tw.data_ptr(), tx.numel() // max(d, 1), d, float(eps),
              out.data_ptr(), stream_ptr())
    return _ret(out, host)


def rope_angles(position, d, rows=None):
    """cos/sin of position * base^(-2j/d) in float64, cast once to float32
    (tensor.py:96-101); [rows, d/2] each."""
    pos = np.asarray(position, dtype=np.float64)
    if rows is not None and pos.ndim == 0:
        pos = np.broadcast_to(pos, (rows,))
    j = np.arange(d // 2, dtype=np.float64)
    ang = pos[..., None] * (ROPE_BASE ** (-2.0 * j / d))
    return np.cos(ang).astype(DTYPE), np.sin(ang).astype(DTYPE)


def rope(x, position):
    """tensor.py:83-109: interleaved pairwise rotations (fo_rope). A vector
    with a scalar position, or a matrix with one position per row."""
    tx, host = _dev(x, "x")
    d = tx.shape[-1]
    if d % 2 != 0:
        raise ShapeError(f"rope: feature dim must be even, got {d}")
    pos = np.asarray(position.cpu() if isinstance(position, torch.Tensor) else position,
                     dtype=np.float64)
    if tx.dim() == 2 and pos.ndim == 0:
        pos = np.broadcast_to(pos, (tx.shape[0],))
    if tx.dim() == 2 and pos.shape != (tx.shape[0],):
        raise ShapeError("rope: need one position per row")
    if tx.dim() > 2 or (tx.dim() == 1 and pos.ndim != 0):
        raise ShapeError("rope: expected a vector with a scalar position or a matrix")
    c, s = rope_angles(pos, d)
    tc = torch.from_numpy(np.ascontiguousarray(c)).to(tx.device)
    ts = torch.from_numpy(np.ascontiguousarray(s)).to(tx.device)
    n = 1 if tx.dim() == 1 else tx.shape[0]
    out = torch.empty_like(tx)
    _lib.call("fo_rope", tx.data_ptr(), tc.data_ptr(), ts.data_ptr(), n, d, out.data_ptr(),
              stream_ptr())
    return _ret(out, host)


def mean_pool_blocks(x, pool):
    """tensor.py:112-126: mean of consecutive row blocks of `pool` rows (the
    trailing partial block over its actual length), float64 sums (fo_mean_pool_blocks)."""
    tx, host = _dev(x, "x", 2, True)
    if pool < 1:
        raise ParameterError(f"pool must be >= 1, got {pool}")
    n, d = tx.shape
    out = torch.empty(-(-n // pool), d, dtype=torch.float32, device=tx.device)
    _lib.call("fo_mean_pool_blocks", tx.data_ptr(), n, d, int(pool), out.data_ptr(), stream_ptr())
    return _ret(out, host)
