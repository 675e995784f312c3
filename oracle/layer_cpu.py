"""The reference CPU path of one dispatch step, timed on the host (BASELINE /
REFERENCE-ARM INFRASTRUCTURE ONLY — bench.py's cpu_baseline and --impl
reference legs; never on the product path).

One dispatch step of the layer (pipeline.py:291-326, the GEMM-Q -> sparse
attention -> GEMM-O dispatch chain) on fp32 numpy tensors of the bench's
shape, cut into `k` interleaved slices so a run of k steps covers the whole
layer exactly once (slice s takes every k-th unit):

  attention  the reference's own compiled kernel (_core.pyx:14-101, built
             from /root/reference by oracle/build_ref.py; the backend
             omniattn picks by default when it is built, _kernels/__init__.py:28-33)
             — or, when that is absent, the numpy restatement of pyref.py:14-48.
             The kernel holds the GIL (one head at a time in the reference), so
             the (head, query-block) units are spread over one worker process
             per host core.
  GEMM-Q     gemm.py:44-93 (numpy, OpenBLAS threads), active tiles of the slice
  GEMM-O     gemm.py:178-229 (numpy), the slice's row blocks, all heads

Work units are (head, active query block) for attention and GEMM-Q and row
blocks for GEMM-O; the partition is by unit index, so every slice carries
~1/k of each.
"""

import multiprocessing as mp
import os
import time

import numpy as np

from . import forecast_coefficients, project_out_dispatch, project_q

T = 128
_W = {}  # worker globals (inherited through fork)


def _attn_task(task):
    h, blocks = task
    core = _W["core"]
    q, k, v = _W["q"][h], _W["k"][h], _W["v"][h]
    act = np.zeros(_W["t"], np.uint8)
    act[blocks] = 1
    out = _W["out"]
    if core is not None:
        return core.masked_block_attention(q, k, v, act, _W["pairs"][h], T, T,
                                           np.float32(1 / np.sqrt(T)), out)
    from . import masked_block_attention

    return masked_block_attention(q, k, v, act, _W["pairs"][h], T, T, 1 / np.sqrt(T), out)


class CpuLayer:
    def __init__(self, seq, heads, d_model, cache_bits, skip_bits, seed=0, workers=None,
                 order=1, elapsed=1, interval=6, backend="auto"):
        from . import build_ref

        self.S, self.H, self.dm = seq, heads, d_model
        self.t = seq // T
        self.cache_bits, self.skip_bits = cache_bits, skip_bits
        self.order, self.elapsed, self.interval = order, elapsed, interval
        core = None
        if backend in ("auto", "compiled") and build_ref.available():
            core = build_ref.load_core()
        elif backend == "compiled":
            raise ImportError("the reference's compiled kernel is not built")
        self.kind = "reference" if core is not None else "port"
        self.backend = "compiled (reference _core.pyx)" if core is not None else "python (numpy port of pyref.py)"
        self.workers = workers or os.cpu_count() or 1
        rng = np.random.default_rng(seed)
        f32 = np.float32
        self.q = rng.standard_normal((heads, seq, T), dtype=f32)
        self.k = rng.standard_normal((heads, seq, T), dtype=f32)
        self.v = rng.standard_normal((heads, seq, T), dtype=f32)
        self.x = rng.standard_normal((seq, d_model), dtype=f32)
        self.w_q = (rng.standard_normal((heads, d_model, T), dtype=f32) * f32(d_model ** -0.5))
        self.norm = (1 + 0.05 * rng.standard_normal((heads, T))).astype(f32)
        self.w_out = (rng.standard_normal((heads, T, d_model), dtype=f32) * f32(T ** -0.5))
        self.o = rng.standard_normal((heads, seq, T), dtype=f32)
        self.n_ord = order + 1
        self.bias = rng.standard_normal((self.n_ord, seq, d_model), dtype=f32)
        self.orders = np.where((~cache_bits).any(axis=0), self.n_ord, 0)
        # attention / GEMM-Q units (head-major, block order) and GEMM-O row blocks
        hh, ii = np.nonzero(cache_bits)
        self.units = np.stack([hh, ii], axis=1)
        self.pairs_per_unit = skip_bits[hh, ii].sum(axis=1)
        _W.update(core=core, q=self.q, k=self.k, v=self.v, t=self.t,
                  pairs=[np.ascontiguousarray(skip_bits[h].astype(np.uint8)) for h in range(heads)],
                  out=np.zeros((seq, T), np.float32))
        self.pool = mp.get_context("fork").Pool(self.workers) if self.workers > 1 else None

    def close(self):
        if self.pool is not None:
            self.pool.terminate()
            self.pool.join()
            self.pool = None

    # ------------------------------------------------------------------ slices
    def slice_units(self, s, k):
        return self.units[s::k]

    def _attn_tasks(self, units):
        """Group a slice's units by head and split them into ~4 tasks per worker."""
        tasks = []
        n_target = max(1, 4 * self.workers)
        chunk = max(1, -(-len(units) // n_target))
        for h in np.unique(units[:, 0]):
            blocks = units[units[:, 0] == h, 1]
            for c in range(0, len(blocks), chunk):
                tasks.append((int(h), blocks[c:c + chunk]))
        return tasks

    def run_slice(self, s, k):
        """Time slice s of k. Returns (seconds, parts dict, computed pairs)."""
        units = self.slice_units(s, k)
        tasks = self._attn_tasks(units)
        t0 = time.perf_counter()
        if self.pool is not None:
            pairs = sum(self.pool.map(_attn_task, tasks, chunksize=1))
        else:
            pairs = sum(_attn_task(tk) for tk in tasks)
        t1 = time.perf_counter()
        # GEMM-Q on a contiguous (head-major) 1/k of the active tiles: the
        # reference loops heads (gemm.py:44-93), so a slice spans 1-2 heads and
        # allocates only their output planes
        n = len(self.units)
        gq = self.units[s * n // k:(s + 1) * n // k]
        hs = np.unique(gq[:, 0])
        if hs.size:
            active = np.zeros((hs.size, self.t), bool)
            active[np.searchsorted(hs, gq[:, 0]), gq[:, 1]] = True
            project_q(self.x, self.w_q[hs], self.norm[hs], active, T)
        t2 = time.perf_counter()
        # GEMM-O dispatch on the slice's row blocks, all heads (gemm.py:178-229)
        blocks = np.arange(s, self.t, k)
        rows = np.concatenate([np.arange(b * T, b * T + T) for b in blocks])
        bias = [self.bias[:, b * T:b * T + T] for b in blocks]
        project_out_dispatch(self.o[:, rows], self.w_out, self.cache_bits[:, blocks].T, bias,
                             self.orders[blocks], self.elapsed, self.interval, self.order, T)
        t3 = time.perf_counter()
        return t3 - t0, {"attention": t1 - t0, "gemm_q": t2 - t1, "gemm_o_dispatch": t3 - t2}, pairs


__all__ = ["CpuLayer", "forecast_coefficients"]
