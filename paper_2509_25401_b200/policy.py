"""Update-step mask policy on the GPU (reference policy.py).

At every update step the reference pools each head's fresh q/k into
compressed blocks, scores them, and derives the next window's cache mask
(which query blocks are recomputed) and skip mask (which key blocks each
computed row reads) — policy.py:196-234, called head by head from
pipeline.py:254-266. Here all heads run in one C-ABI call
(`fo_generate_masks`, csrc/fo_policy.cu) whose decisions match the
reference's float32/float64 numpy bit for bit, and the result feeds
`encode_symbols` without leaving the device.

Inputs are the engine's bf16 activations: q and k given in another dtype
(e.g. the reference's float32) are rounded to bf16 before pooling, so the
decisions are bit-for-bit those the reference makes on the bf16-rounded
tensors (the fixtures in tests/golden/policy.npz are bf16-representable).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._runtime import TILE, as_device, check_bsd, check_finite, stream_ptr
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
    block-granularity numpy (cache_bits [t_q], skip_bits [t_q, t_kv]), True =
    compute. The sm_100a kernels fix b_q = b_k = d = 128."""
    if b_q != TILE or b_k != TILE:
        raise ParameterError(f"b_q/b_k must be {TILE} for the sm_100a kernels, got {b_q}/{b_k}")
    qt, kt = torch.as_tensor(np.asarray(q)), torch.as_tensor(np.asarray(k))
    if qt.dim() != 2 or kt.dim() != 2:
        raise ShapeError(f"q/k must be 2-D, got {tuple(qt.shape)} / {tuple(kt.shape)}")
    if qt.shape[1] != kt.shape[1]:
        raise ShapeError(f"q/k feature dims differ: {qt.shape[1]} vs {kt.shape[1]}")
    if qt.shape[0] != kt.shape[0]:
        raise ParameterError("cache selection needs a square compressed map; q and k lengths differ")
    cb, sb = generate_masks_heads(qt[:, None, :], kt[:, None, :], pool_n=pool_n, n_text=n_text,
                                  tau_q=tau_q, tau_kv=tau_kv, s_q=s_q, guard=guard)
    return cb[0].bool().cpu().numpy(), sb[0].bool().cpu().numpy()


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
