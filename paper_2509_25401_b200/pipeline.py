"""One DiT attention layer on the GPU: the callers of the hot path.

Mirrors reference pipeline.py:223-326. update_step refreshes the feature
cache and the GEMM-O bias and computes the step densely; dispatch_step runs
the sparse chain GEMM-Q -> sparse attention (mode="bias") -> GEMM-O dispatch
against the governing update step's symbols. The next window's symbols come
from the GPU mask policy (policy.MaskPolicy, reference policy.py) or from the
caller.

Multi-GPU: heads are sharded across ranks (shard_heads). GEMM-Q and K/V are
column-parallel, attention and the cache are per head, GEMM-O is row-parallel
and its partial outputs (each rank's heads, including each rank's partial
cached bias) are summed by one all-reduce — exact by linearity of the
projection and the forecast.
"""

import functools
import os
from dataclasses import dataclass

import torch

from ._runtime import TILE, Status, as_device
from .attention import FeatureCache, dense_attention_update, sparse_attention
from .errors import ParameterError, StateError
from .gemm import (pack_w_out, pack_w_q, pack_w_qkv, project_out_dispatch, project_out_update,
                   project_q, project_qkv)
from .symbols import ceil_div


@dataclass
class LayerParams:
    """Packed bf16 weights of one layer (reference LayerParams, pipeline.py:115-122)."""

    w_q: object
    w_k: object
    w_v: object
    q_norm: torch.Tensor
    k_norm: torch.Tensor
    w_out: object

    @classmethod
    def from_reference(cls, w_q, w_k, w_v, q_norm, k_norm, w_out, heads=None):
        """Pack reference-layout weights ([H, dm, D] / [H, D, dm], any device).
        heads: optional index list to keep (head-sharded rank)."""
        def sel(a):
            a = torch.as_tensor(a)
            return a if heads is None else a[list(heads)]
        return cls(w_q=pack_w_q(sel(w_q)), w_k=pack_w_q(sel(w_k)), w_v=pack_w_q(sel(w_v)),
                   q_norm=as_device(sel(q_norm), torch.float32, "q_norm"),
                   k_norm=as_device(sel(k_norm), torch.float32, "k_norm"),
                   w_out=pack_w_out(sel(w_out)))

    @property
    def heads(self):
        return self.w_q.heads

    @property
    def w_qkv(self):
        """[W_q; W_k; W_v] packed once for the fused projection (None above
        32 heads per rank, where the three launches are used)."""
        if not hasattr(self, "_w_qkv"):
            fused = self.heads <= 32 and os.environ.get("FO_FUSED_QKV", "1") != "0"
            self._w_qkv = pack_w_qkv(self.w_q, self.w_k, self.w_v) if fused else None
        return self._w_qkv


@dataclass
class LayerState:
    params: LayerParams
    cache: FeatureCache
    symbols: object = None
    bias: object = None


def shard_heads(heads, world, rank):
    """Contiguous head range owned by `rank` (heads must divide evenly)."""
    if heads % world:
        raise ParameterError(f"{heads} heads do not shard evenly over {world} ranks")
    per = heads // world
    return list(range(rank * per, (rank + 1) * per))


def project_kv(x, params, *, eps=1e-6, k_out=None, v_out=None, stream=None, check=True):
    """Dense K (RMS norm + RoPE) and V projections (pipeline.py:223-234) on the
    GEMM-Q kernel in dense mode."""
    k = project_q(x, params.w_k, params.k_norm, None, "update", eps=eps, out=k_out, fill=None,
                  stream=stream, check=check)
    v = project_q(x, params.w_v, None, None, "update", rope=False, out=v_out, fill=None,
                  stream=stream, check=False)  # same x, checked once
    return k, v


def _allreduce(out, group):
    if group is not None:
        import torch.distributed as dist

        dist.all_reduce(out, group=group)
    return out


def _nvtx(name):
    """An NVTX range around a layer step (the C-ABI entry points inside carry
    their own ranges), for nsys / ncu --nvtx filtering."""
    def wrap(fn):
        @functools.wraps(fn)
        def ranged(*args, **kwargs):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()
        return ranged
    return wrap


@_nvtx("fo.update_step")
def update_step(state, x, symbols_next, order_d, *, group=None, check=True, policy=None, t=0):
    """Refresh symbols, cache and bias; compute the step densely
    (pipeline.py:244-288). The next window's symbols come from `policy`
    (a MaskPolicy, run on this step's q/k at step t, pipeline.py:254-266)
    when symbols_next is None, else from the caller."""
    x = as_device(x, torch.bfloat16, "x")
    p = state.params
    if p.w_qkv is not None:  # q, k, v in one launch (one read of x)
        q, k, v = project_qkv(x, p.w_qkv, p.q_norm, p.k_norm, None, "update", check=check)
    else:
        q = project_q(x, p.w_q, p.q_norm, None, "update", fill=None, check=check)
        k, v = project_kv(x, p, check=False)
    if symbols_next is None:
        if policy is None:
            raise ParameterError("update_step needs symbols_next or a MaskPolicy")
        symbols_next = policy.symbols(q, k, t)
    o = dense_attention_update(q, k, v, state.cache, check=check)
    out, bias = project_out_update(o, p.w_out, symbols_next, state.cache, order_d, check=check)
    state.symbols = symbols_next
    state.bias = bias
    return _allreduce(out, group)


_COMM = {}


def _comm_stream(device):
    if device not in _COMM:
        _COMM[device] = torch.cuda.Stream(device=device)
    return _COMM[device]


def _dispatch_out_allreduce(o, p, state, elapsed_k, interval_n, order_d, out, group, chunks, check,
                            comm_sms):
    """GEMM-O dispatch in `chunks` row chunks, each chunk's all-reduce issued on
    a side stream as soon as its rows are written, so the transfer of chunk c
    overlaps the projection of chunk c + 1 (the reduction is per row, so the
    chunked sum equals the whole one). comm_sms SMs are left to the
    collective's kernels while the projection of the next chunk runs."""
    import torch.distributed as dist

    n = o.shape[0]
    t_q = ceil_div(n, TILE)
    if out is None:
        out = torch.empty(n, p.w_out.d_model, dtype=torch.bfloat16, device=o.device)
    chunks = max(1, min(int(chunks), t_q))
    bounds = [t_q * c // chunks for c in range(chunks + 1)]
    main = torch.cuda.current_stream(o.device)
    comm = _comm_stream(o.device)
    sms = 0
    if chunks > 1 and comm_sms > 0:
        sms = max(2, torch.cuda.get_device_properties(o.device).multi_processor_count - comm_sms)
    works = []
    for c in range(chunks):
        b0, b1 = bounds[c], bounds[c + 1]
        project_out_dispatch(o, p.w_out, state.symbols, state.bias, elapsed_k, interval_n, order_d,
                             out=out, blocks=(b0, b1), max_sms=sms, check=check and c == 0)
        ev = torch.cuda.Event()
        ev.record(main)
        comm.wait_event(ev)
        with torch.cuda.stream(comm):
            works.append(dist.all_reduce(out[b0 * TILE:min(b1 * TILE, n)], group=group,
                                         async_op=True))
    for w in works:
        w.wait()
    main.wait_stream(comm)
    return out


@_nvtx("fo.dispatch_step")
def dispatch_step(state, x, elapsed_k, interval_n, order_d, *, group=None, check=True, fill=None,
                  bufs=None, chunks=1, comm_sms=0):
    """Sparse execution against the governing symbols (pipeline.py:291-326).
    bufs: optional dict of preallocated q/k/v/o/out tensors (graph capture).
    With a process group, chunks > 1 overlaps GEMM-O row chunks with the
    all-reduce of the previous chunk (_dispatch_out_allreduce)."""
    if state.symbols is None or state.bias is None:
        raise StateError("dispatch step before any update step")
    x = as_device(x, torch.bfloat16, "x")
    p = state.params
    b = bufs or {}
    if p.w_qkv is not None:  # q (active tiles), k and v in one launch (one read of x)
        q, k, v = project_qkv(x, p.w_qkv, p.q_norm, p.k_norm, state.symbols, "dispatch",
                              q_out=b.get("q"), k_out=b.get("k"), v_out=b.get("v"), fill=fill,
                              check=check)
    else:
        q = project_q(x, p.w_q, p.q_norm, state.symbols, "dispatch", fill=fill, out=b.get("q"),
                      check=check)
        k, v = project_kv(x, p, k_out=b.get("k"), v_out=b.get("v"), check=False)
    o = sparse_attention(q, k, v, state.symbols, state.cache, None, elapsed_k, interval_n, order_d,
                         mode="bias", fill=fill, out=b.get("o"), check=check)
    if group is not None and chunks > 1:
        return _dispatch_out_allreduce(o, p, state, elapsed_k, interval_n, order_d, b.get("out"),
                                       group, chunks, check, comm_sms)
    out = project_out_dispatch(o, p.w_out, state.symbols, state.bias, elapsed_k, interval_n,
                               order_d, out=b.get("out"), check=check)
    return _allreduce(out, group)


def new_layer_state(params, seq, order_d):
    t_q = ceil_div(seq, TILE)
    return LayerState(params=params, cache=FeatureCache(params.heads, t_q, order_d, seq=seq))


class HostStepper:
    """Dispatch steps on host-resident activations with the PCIe copies
    overlapped across steps: step k+1's input copy (H2D stream) and step k-1's
    output copy (D2H stream) run while step k computes. Every step still moves
    its own x in and its own out back; device buffers are double-buffered and
    ordered by CUDA events, so no step reads a buffer the next copy is filling.
    """

    def __init__(self, state, seq, d_model, device=None, group=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.state, self.group = state, group
        H = state.params.heads
        self.h2d, self.d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        self.x = [torch.empty(seq, d_model, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.out = [torch.empty(seq, d_model, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.bufs = {n: torch.empty(seq, H, TILE, dtype=torch.bfloat16, device=dev)
                     for n in ("q", "k", "v", "o")}
        ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        self.x_ready, self.x_free, self.out_ready, self.out_free = ev(), ev(), ev(), ev()
        self.k = 0

    def step(self, x_host, out_host, elapsed_k, interval_n, order_d):
        """Enqueue one step (asynchronous; out_host is valid after synchronize)."""
        b = self.k & 1
        comp = torch.cuda.current_stream()
        if self.k >= 2:
            self.h2d.wait_event(self.x_free[b])
        with torch.cuda.stream(self.h2d):
            self.x[b].copy_(x_host, non_blocking=True)
            self.x_ready[b].record(self.h2d)
        comp.wait_event(self.x_ready[b])
        if self.k >= 2:
            comp.wait_event(self.out_free[b])
        bufs = dict(self.bufs, out=self.out[b])
        dispatch_step(self.state, self.x[b], elapsed_k, interval_n, order_d, group=self.group,
                      check=False, bufs=bufs)
        self.x_free[b].record(comp)
        self.out_ready[b].record(comp)
        self.d2h.wait_event(self.out_ready[b])
        with torch.cuda.stream(self.d2h):
            out_host.copy_(self.out[b], non_blocking=True)
            self.out_free[b].record(self.d2h)
        self.k += 1
