"""The sm_100a backend behind the reference tile-kernel protocol.

Implements the contract of reference _kernels/pyref.py:14-48 and
_kernels/_core.pyx:14-101 — masked_block_attention(q, k, v, active,
pair_bits, b_q, b_k, scale, out) -> computed pair count — on the tcgen05
sparse-attention kernel: the decoded bits are packed on the device (K1), the
schedule is planned on the device, and only rows of active blocks are
written back into the caller's `out`. Inputs are rounded to bf16 (the
engine's arithmetic type); head dims below 128 are zero-padded, which leaves
q.k and the attended values unchanged Other block sizes run the fp32 tile
kernel (fo_masked_block_attention_f32), so the reference's own small-block
kernel tests hold at their 1e-5 tolerance.
"""

import numpy as np
import torch

from .. import _lib
from .._runtime import TILE, Status, require_cuda, stream_ptr
from ..errors import ConsistencyError, ParameterError, ShapeError

NAME = "b200"


def masked_block_attention(q, k, v, active, pair_bits, b_q, b_k, scale, out):
    if b_q != TILE or b_k != TILE:
        # any other block size (the reference's own kernel tests use 4-16): the
        # fp32 tile kernel, which keeps the reference's float32 arithmetic
        from ..attention import masked_block_attention_f32

        return masked_block_attention_f32(q, k, v, active, pair_bits, b_q, b_k, scale, out)
    require_cuda()
    q = np.ascontiguousarray(q, dtype=np.float32)
    n, d = q.shape
    if d > TILE:
        raise ParameterError(f"head dim {d} > {TILE}")
    t_q = -(-n // TILE)
    active = np.asarray(active, dtype=np.uint8).reshape(-1)
    pair_bits = np.asarray(pair_bits, dtype=np.uint8)
    if active.shape != (t_q,) or pair_bits.shape != (t_q, t_q):
        raise ShapeError(f"mask shapes {active.shape}/{pair_bits.shape} for {t_q} blocks")

    def dev(a):
        t = torch.zeros(n, 1, TILE, dtype=torch.bfloat16, device="cuda")
        t[:, 0, :d] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
        return t

    qd, kd, vd = dev(q), dev(k), dev(v)
    from ..symbols import encode_symbols

    st = Status()
    sym = encode_symbols(torch.from_numpy(active[None]), torch.from_numpy(pair_bits[None]), 1,
                         status=st)
    plan = sym.plan(status=st, check=False)
    res = torch.zeros(n, 1, TILE, dtype=torch.bfloat16, device="cuda")
    pairs = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.call("fo_sparse_attention", qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), n, 1, TILE,
              sym.s_s.data_ptr(), t_q, t_q, 1, plan.ptr(), float(scale), 0, res.data_ptr(), None,
              None, 0, pairs.data_ptr(), st.ptr(), stream_ptr())
    bits = int(st.t.item())
    if bits & _lib.ST_CONSISTENCY:
        raise ConsistencyError("active query block has every key block skipped")
    _lib.raise_status(bits, "masked_block_attention")
    rows = np.repeat(active.astype(bool), TILE)[:n]
    out[rows] = res[:, 0, :d].float().cpu().numpy()[rows]
    return int(pairs.item())
