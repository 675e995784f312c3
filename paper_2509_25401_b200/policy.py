"""Update-step mask policy on the GPU (reference policy.py).

At every update step the reference pools each head's fresh q/k into
compressed blocks, scores them, and derives the next window's cache mask
(which query blocks are recomputed) and skip mask (which key blocks each
computed row reads) — policy.py:196-234, called head by head from
pipeline.py:254-266. Here all heads run in one C-ABI call
(`fo_generate_masks`, csrc/fo_policy.cu) whose decisions match the
reference's float32/float64 numpy bit for bit, and the result feeds
`encode_symbols` without leaving the device.

generate_masks_heads takes the engine's bf16 activations (another dtype is
rounded to bf16 first, so its decisions are the reference's on the
bf16-rounded tensors). The per-head reference signature `generate_masks` and
the building blocks (compressed_attention, select_cached_blocks, ...) run the
same kernels stage by stage in the caller's precision: float32 inputs are
pooled as float32, bit-for-bit the reference's decisions.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._runtime import TILE, as_device, check_bsd, check_finite, require_cuda, stream_ptr
from .errors import ParameterError, ShapeError
from .symbols import ceil_div, encode_symbols

_workspaces = {}


def _workspace(seq, heads, pool_n, device):
    """Per-device scratch, grown on demand (stream-ordered reuse: one policy
    call per update step)."""
    nbytes = int(_lib.load().fo_policy_workspace_bytes(seq, heads, pool_n))
    ws = _workspaces.get(device)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _workspaces[device] = ws
    return ws


def ramp_threshold(tau_target, step, warmup_steps):
    """Linear warmup from 0 to the target threshold (policy.py:181-187)."""
    if step < 0:
        raise ParameterError(f"step must be >= 0, got {step}")
    if warmup_steps <= 0:
        return tau_target
    return tau_target * min(1.0, step / warmup_steps)


def generate_masks_heads(q, k, *, pool_n, n_text, tau_q, tau_kv, s_q=0.0, guard=True,
                         cache_out=None, skip_out=None, stream=None, check=True):
    """All heads at once: q, k bf16 [S, H, 128] on the device ->
    (cache_bits u8 [H, t_q], skip_bits u8 [H, t_q, t_q]), True = compute."""
    q = check_bsd(as_device(q, torch.bfloat16, "q"), "q")
    k = check_bsd(as_device(k, torch.bfloat16, "k"), "k", seq=q.shape[0], heads=q.shape[1])
    S, H = q.shape[0], q.shape[1]
    if pool_n < 1:
        raise ParameterError(f"pool_n must be >= 1, got {pool_n}")
    t_q = ceil_div(S, TILE)
    cb = cache_out if cache_out is not None else torch.empty(H, t_q, dtype=torch.uint8,
                                                             device=q.device)
    sb = skip_out if skip_out is not None else torch.empty(H, t_q, t_q, dtype=torch.uint8,
                                                           device=q.device)
    if tuple(cb.shape) != (H, t_q) or tuple(sb.shape) != (H, t_q, t_q):
        raise ShapeError("generate_masks: output buffers have the wrong shape")
    if check:  # policy.py:46-47 as_matrix(q), as_matrix(k)
        check_finite(q, "q", stream=stream)
        check_finite(k, "k", stream=stream)
    ws = _workspace(S, H, pool_n, q.device)
    _lib.call("fo_generate_masks", q.data_ptr(), k.data_ptr(), S, H, int(n_text), int(pool_n),
              float(tau_q), float(tau_kv), float(s_q), 1 if guard else 0, cb.data_ptr(),
              sb.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr(stream))
    return cb, sb


def generate_masks(q, k, *, b_q, b_k, pool_n, n_text, tau_q, tau_kv, s_q=0.0, guard=True):
    """Reference signature for one head (policy.py:196-234): q, k [n, d] ->
    block-granularity (cache_bits [t_q], skip_bits [t_q, t_kv]), True =
    compute; numpy in -> numpy out. The reference's composition of its building
    blocks, every stage on the device (the per-stage kernels below) in the
    caller's precision: float32 inputs are pooled as float32 (bit-for-bit the
    reference's decisions), bf16 tensors as bf16. Any b_q / b_k and d <= 128;
    the batched engine path is generate_masks_heads."""
    host = not isinstance(q, torch.Tensor)
    qt = torch.as_tensor(np.asarray(q, dtype=np.float32)) if host else q
    kt = torch.as_tensor(np.asarray(k, dtype=np.float32)) if not isinstance(k, torch.Tensor) else k
    if qt.dim() != 2 or kt.dim() != 2:
        raise ShapeError(f"q/k must be 2-D, got {tuple(qt.shape)} / {tuple(kt.shape)}")
    if pool_n < 1 or b_q < 1 or b_k < 1:
        raise ParameterError(f"pool_n, b_q and b_k must be >= 1, got {pool_n}, {b_q}, {b_k}")
    n = qt.shape[0]
    m = compressed_attention(qt.cuda(), kt.cuda(), pool_n * b_q, pool_n * b_k, n_text)
    rows, cols = m.p_tilde.shape
    if rows != cols:
        raise ParameterError(
            f"cache selection needs a square compressed map, got {rows}x{cols}; "
            "choose b_q/b_k so query and key grids align")
    contribution, guidance = _block_scores(m)
    cached = select_cached_blocks(contribution, guidance, tau_q)
    comp_cache = torch.ones(rows, dtype=torch.bool, device=cached.device)
    comp_cache[m.n_t:] = ~cached
    comp_cache = degrade_to_full_cache(comp_cache, m.n_t, s_q)
    comp_skip = select_skip_blocks(m, comp_cache, tau_kv, guard=guard)
    t_q, t_kv = ceil_div(n, b_q), ceil_div(kt.shape[0], b_k)
    cache_bits = comp_cache.repeat_interleave(pool_n)[:t_q]  # expand_blocks (policy.py:190-193)
    skip_bits = comp_skip.repeat_interleave(pool_n, 0)[:t_q].repeat_interleave(pool_n, 1)[:, :t_kv]
    if host:
        return cache_bits.cpu().numpy(), skip_bits.cpu().numpy()
    return cache_bits, skip_bits


# ---------------------------------------------------------------------------
# The reference's policy building blocks (policy.py:21-178), one device stage
# per call (csrc/fo_policy.cu: the same kernels generate_masks_heads fuses).
# numpy in -> numpy out (the reference convention), torch in -> torch out.


@dataclass(frozen=True)
class CompressedAttnMap:
    """Row-stochastic attention map over compressed blocks (policy.py:21-41);
    n_t leading compressed blocks hold text tokens. p_tilde may be a numpy
    array or a CUDA tensor [rows, cols] (one head) / [heads, rows, cols]."""

    p_tilde: object
    n_t: int

    def __post_init__(self):
        p = self.p_tilde
        shape = tuple(p.shape)
        if len(shape) not in (2, 3) or (isinstance(p, np.ndarray) and len(shape) != 2):
            raise ShapeError(f"compressed map must be 2-D, got {shape}")
        if not 0 <= self.n_t < shape[-2]:
            raise ParameterError(f"n_t={self.n_t} must leave at least one vision row "
                                 f"(map has {shape[-2]} rows)")
        sums = p.sum(axis=-1) if isinstance(p, np.ndarray) else p.double().sum(-1)
        ok = (np.allclose(sums, 1.0, atol=1e-5) if isinstance(p, np.ndarray)
              else bool(((sums - 1.0).abs() <= 1e-5 + 1e-8).all()))
        if not ok:
            raise ParameterError("compressed map rows must each sum to 1")


def _heads_layout(x, name):
    """[n, d] (one head) or [n, H, d] -> (fp32/bf16 CUDA [n, H, 128] zero-padded,
    is_f32, d, came-from-numpy)."""
    require_cuda()
    host = not isinstance(x, torch.Tensor)
    t = torch.as_tensor(np.asarray(x, dtype=np.float32)) if host else x
    if not t.is_cuda:
        t = t.cuda()
    if t.dtype not in (torch.float32, torch.bfloat16):
        t = t.float()
    if t.dim() == 2:
        t = t[:, None, :]
    if t.dim() != 3:
        raise ShapeError(f"{name}: expected a 2-D matrix, got shape {tuple(x.shape)}")
    d = t.shape[2]
    if d > TILE:
        raise ShapeError(f"{name}: head dim {d} exceeds {TILE}")
    if not bool(torch.isfinite(t).all()):  # as_matrix (tensor.py:19-30)
        raise ParameterError(f"{name}: contains NaN or Inf")
    if d < TILE:
        t = torch.nn.functional.pad(t, (0, TILE - d))
    return t.contiguous(), t.dtype == torch.float32, d, host


def compressed_attention(q, k, pool_q, pool_k, n_text):
    """policy.py:44-55: mean-pool q/k rows into compressed tokens (float64
    sums), score them in float64 / sqrt(d) and row-softmax the map
    (fo_policy_compressed_map). q, k: [n, d] (or [n, heads, d] for every head)."""
    tq, f32q, d, host = _heads_layout(q, "q")
    tk, f32k, dk, _ = _heads_layout(k, "k")
    if d != dk:
        raise ShapeError(f"q/k feature dims differ: {d} vs {dk}")
    if tq.shape[1] != tk.shape[1]:
        raise ShapeError(f"q/k head counts differ: {tq.shape[1]} vs {tk.shape[1]}")
    if f32q != f32k:
        tq, tk = tq.float(), tk.float()
    if pool_q < 1 or pool_k < 1:
        raise ParameterError(f"pool must be >= 1, got {min(pool_q, pool_k)}")
    H = tq.shape[1]
    rows, cols = ceil_div(tq.shape[0], pool_q), ceil_div(tk.shape[0], pool_k)
    p = torch.empty(H, rows, cols, dtype=torch.float32, device=tq.device)
    nb = int(_lib.load().fo_policy_map_workspace_bytes(tq.shape[0], tk.shape[0], H, pool_q, pool_k))
    ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=tq.device)
    _lib.call("fo_policy_compressed_map", tq.data_ptr(), tk.data_ptr(),
              1 if tq.dtype == torch.float32 else 0, tq.shape[0], tk.shape[0], H, d, int(pool_q),
              int(pool_k), p.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr(None))
    single = (q.dim() if isinstance(q, torch.Tensor) else np.ndim(q)) == 2
    out = p[0] if single else p
    return CompressedAttnMap(p_tilde=out.cpu().numpy() if host else out,
                             n_t=ceil_div(n_text, pool_q))


def _map_dev(m):
    p = m.p_tilde
    host = isinstance(p, np.ndarray)
    t = torch.as_tensor(np.ascontiguousarray(p, dtype=np.float32)).cuda() if host else p.float()
    single = t.dim() == 2
    return (t[None] if single else t).contiguous(), host, single


def _block_scores(m):
    t, host, single = _map_dev(m)
    H, rows, cols = t.shape
    c = torch.empty(H, cols - m.n_t, dtype=torch.float64, device=t.device)
    g = torch.empty(H, rows - m.n_t, dtype=torch.float64, device=t.device)
    _lib.call("fo_policy_block_scores", t.data_ptr(), H, rows, cols, m.n_t, c.data_ptr(),
              g.data_ptr(), stream_ptr(None))

    def back(x):
        x = x[0] if single else x
        return x.cpu().numpy() if host else x
    return back(c), back(g)


def vision_to_text_contribution(m):
    """policy.py:58-65: per vision block, the mass text rows place on it
    (float32 column sums, float64 out)."""
    return _block_scores(m)[0]


def text_to_vision_guidance(m):
    """policy.py:68-77: per vision block, the re-softmaxed text-to-vision mass
    summed over text rows (float64 out)."""
    return _block_scores(m)[1]


def select_cached_blocks(contribution, guidance, tau_q):
    """policy.py:93-111: vision blocks in both ascending-score prefixes within
    tau_q of their totals (stable order, float64 cumsums). True = cached."""
    host = not isinstance(contribution, torch.Tensor)
    c = torch.as_tensor(np.asarray(contribution, dtype=np.float64)) if host else contribution.double()
    g = torch.as_tensor(np.asarray(guidance, dtype=np.float64)) if not isinstance(
        guidance, torch.Tensor) else guidance.double()
    if tuple(c.shape) != tuple(g.shape):
        raise ShapeError(f"score vectors differ: {tuple(c.shape)} vs {tuple(g.shape)}")
    if not 0.0 <= tau_q <= 1.0:
        raise ParameterError(f"tau_q must be in [0, 1], got {tau_q}")
    require_cuda()
    single = c.dim() == 1
    c2 = (c[None] if single else c).cuda().contiguous()
    g2 = (g[None] if single else g).cuda().contiguous()
    out = torch.zeros(c2.shape, dtype=torch.uint8, device=c2.device)
    _lib.call("fo_policy_select_cached", c2.data_ptr(), g2.data_ptr(), c2.shape[0], c2.shape[1],
              float(tau_q), out.data_ptr(), stream_ptr(None))
    out = out.bool()
    out = out[0] if single else out
    return out.cpu().numpy() if host else out


def select_skip_blocks(m, cache_bits, tau_kv, guard=True):
    """policy.py:124-159: per computed row, skip the lowest-mass key blocks
    within the absolute budget tau_kv (text columns and the diagonal exempt
    under guard; an unprotected row keeps its highest-mass block). Returns
    the compressed keep mask, True = compute the pair."""
    if not 0.0 <= tau_kv <= 1.0:
        raise ParameterError(f"tau_kv must be in [0, 1], got {tau_kv}")
    t, host, single = _map_dev(m)
    H, rows, cols = t.shape
    cb = torch.as_tensor(np.asarray(cache_bits, dtype=bool)) if not isinstance(
        cache_bits, torch.Tensor) else cache_bits
    want = (rows,) if single else (H, rows)
    if tuple(cb.shape) != want:
        raise ShapeError(f"cache bits shape {tuple(cb.shape)} != {want}")
    cbd = cb.to(device=t.device, dtype=torch.uint8).reshape(H, rows).contiguous()
    keep = torch.empty(H, rows, cols, dtype=torch.uint8, device=t.device)
    _lib.call("fo_policy_select_skip", t.data_ptr(), cbd.data_ptr(), H, rows, cols, m.n_t,
              float(tau_kv), 1 if guard else 0, keep.data_ptr(), stream_ptr(None))
    keep = keep.bool()
    keep = keep[0] if single else keep
    return keep.cpu().numpy() if host else keep


def degrade_to_full_cache(cache_bits, n_t, s_q):
    """policy.py:162-178: if the computed fraction of vision blocks is below
    s_q, cache them all (text blocks stay computed). A bit vector per head;
    torch tensors are decided on the device."""
    if not 0.0 <= s_q <= 1.0:
        raise ParameterError(f"s_q must be in [0, 1], got {s_q}")
    if isinstance(cache_bits, torch.Tensor):
        cb = cache_bits.bool()
        vision = cb[..., n_t:]
        if vision.shape[-1] == 0:
            return cb
        low = vision.double().mean(-1, keepdim=True) < s_q
        out = cb.clone()
        out[..., n_t:] = vision & ~low
        return out
    cb = np.asarray(cache_bits, dtype=bool)
    vision = cb[n_t:]
    if vision.size == 0:
        return cb
    if vision.mean() < s_q:
        out = cb.copy()
        out[n_t:] = False
        return out
    return cb


@dataclass(frozen=True)
class MaskPolicy:
    """The policy fields of the reference PipelineConfig (pipeline.py:40-70)."""

    n_text: int
    tau_q: float
    tau_kv: float
    pool_n: int = 1
    s_q: float = 0.0
    guard: bool = True
    warmup: int = 0

    def __post_init__(self):
        if self.pool_n < 1:
            raise ParameterError(f"pool_n must be >= 1, got {self.pool_n}")
        if self.warmup < 0:
            raise ParameterError("warmup must be >= 0")
        for name in ("tau_q", "tau_kv", "s_q"):
            v = getattr(self, name)
            if not 0.0 <= v <= 1.0:
                raise ParameterError(f"{name} must be in [0, 1], got {v}")

    def symbols(self, q, k, t, stream=None):
        """Next window's DeviceSymbols from this update step's q/k at step t."""
        tq = ramp_threshold(self.tau_q, t, self.warmup)
        tkv = ramp_threshold(self.tau_kv, t, self.warmup)
        cb, sb = generate_masks_heads(q, k, pool_n=self.pool_n, n_text=self.n_text, tau_q=tq,
                                      tau_kv=tkv, s_q=self.s_q, guard=self.guard, stream=stream,
                                      check=False)
        return encode_symbols(cb, sb, self.pool_n, stream=stream, check=False)
