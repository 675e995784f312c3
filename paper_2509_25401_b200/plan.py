"""Per-layer schedule derived from the symbols on the GPU (fo_plan).

One single-CTA kernel turns the packed symbols into everything the hot-path
kernels consume: attention work items (head, q-block, #KV blocks) sorted
longest-first, the GEMM-Q tile list, per-block active-head masks for GEMM-O,
cached-bias orders, and the mask-predicted pair counts. It also performs the
reference's contract checks: an active query block with no key block
(ConsistencyError, pyref.py:43-46) and a cached tile with a cold cache
(StateError, attention.py:208-211 / gemm.py:150-153).
"""

import ctypes

import numpy as np
import torch

from . import _lib
from ._runtime import Status, stream_ptr


class Plan:
    def __init__(self, ws, heads, rows, dense):
        self.ws = ws
        self.heads, self.rows, self.dense = heads, rows, dense
        offs = (ctypes.c_size_t * 7)()
        _lib.load().fo_plan_offsets(heads, rows, offs)
        self.offsets = [int(o) for o in offs]

    @classmethod
    def build(cls, sym, valid=None, order_d=0, dense=False, status=None, stream=None, check=True,
              ws=None):
        """ws: optional preallocated workspace, rewritten in place (the engine's
        static per-layer plans, so captured CUDA graphs keep valid pointers)."""
        nbytes = _lib.load().fo_plan_workspace_bytes(sym.heads, sym.rows)
        if ws is None:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=sym.s_c.device)
        elif ws.numel() < nbytes or ws.dtype != torch.uint8:
            raise ValueError(f"plan workspace needs {nbytes} uint8 bytes")
        st = status or Status.default()
        _lib.call("fo_plan", sym.s_c.data_ptr(), sym.s_s.data_ptr(), sym.heads, sym.rows, sym.cols,
                  sym.pool_n, int(bool(dense)), _lib.ptr(valid), int(order_d), ws.data_ptr(),
                  st.ptr(), stream_ptr(stream))
        if check:
            st.check("plan")
        return cls(ws, sym.heads, sym.rows, dense)

    def ptr(self):
        return self.ws.data_ptr()

    def _view(self, k, dtype, n):
        itemsize = torch.tensor([], dtype=dtype).element_size()
        return self.ws[self.offsets[k]:self.offsets[k] + n * itemsize].view(dtype)

    # host-side inspection (synchronising; used by counters and tests)
    def counts(self):
        return self._view(0, torch.int32, 8).cpu().numpy()

    def items(self):
        n = int(self.counts()[0])
        it = self._view(1, torch.int32, 2 * self.heads * self.rows).view(-1, 2)[:n].cpu().numpy()
        return np.stack([it[:, 0] >> 20, it[:, 0] & 0xFFFFF, it[:, 1]], axis=1)

    def pair_items(self):
        """True when each attention item (h, i) covers query blocks i and i + 1
        on the two CTAs of a cluster (pool_n even: they share a skip row)."""
        return bool(int(self.counts()[4]))

    def gq_items(self):
        n = int(self.counts()[1])
        it = self._view(2, torch.int32, self.heads * self.rows)[:n].cpu().numpy()
        return np.stack([it >> 20, it & 0xFFFFF], axis=1)

    def hmask(self):
        return self._view(3, torch.int64, self.rows).cpu().numpy().view(np.uint64)

    def orders_tensor(self):
        return self._view(4, torch.int32, self.rows)

    def pairs_pred(self):
        return self._view(5, torch.int64, self.heads).cpu().numpy()

    def schedule(self):
        """Attention schedule: int32 [n_waves, slots], the item index (into
        items()) each CTA (each CTA pair when pair_items()) runs in each wave,
        -1 for none."""
        lib = _lib.load()
        off = int(lib.fo_plan_schedule_offset(self.heads, self.rows))
        n_waves, ctas = int(self.counts()[6]), int(self.counts()[5])
        n = n_waves * ctas
        return self.ws[off:off + 4 * n].view(torch.int32).cpu().numpy().reshape(n_waves, ctas)

    def gq_jobs(self):
        """GEMM-Q CTA-pair jobs (counts[7]): rows (i0, i1 or -1, h, n256, h2); n256
        jobs cover heads h and h2 as one N=256 tile, the others head h alone
        (h2 = 0)."""
        n = int(self.counts()[7])
        it = self._view(6, torch.int32, 2 * n).view(-1, 2).cpu().numpy()
        x, y = it[:, 0], it[:, 1]
        return np.stack([x & 0xFFFF, (x >> 16) - 1, y & 0xFF, (y >> 8) & 1, (y >> 16) & 0xFF],
                        axis=1)
