"""Symbol-guided sparse attention and the feature cache, on the GPU.

Mirrors reference pkg/src/omniattn/attention.py: each query block either runs
compute-on-demand (online softmax over the key blocks its skip row allows) or
cache-then-reuse (its tile is forecast from stored finite differences, or left
alone in mode="bias" where the output projection covers it). The batched form
processes every head of a layer in one launch: q, k, v are bf16 [seq, heads,
128] CUDA tensors and `symbols` is a DeviceSymbols. The per-head reference
signature (numpy q[n, d] + SymbolBuffer) is accepted too and adapted onto the
batched kernel.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._runtime import TILE, Status, check_bsd, check_finite, check_out, require_cuda, stream_ptr
from .errors import ConsistencyError, ParameterError, ShapeError, StateError
from .symbols import DeviceSymbols, SymbolBuffer, ceil_div

DTYPE = np.float32


def forecast_coefficients(elapsed_k, interval_n, n_orders):
    """(k/N)^d / d! in float32 (attention.py:88-93)."""
    x = elapsed_k / interval_n
    return np.array([x**d / math.factorial(d) for d in range(n_orders)], dtype=DTYPE)


def check_elapsed(elapsed_k, interval_n):
    if interval_n < 1 or not 1 <= elapsed_k <= interval_n - 1:
        raise ParameterError(f"elapsed_k={elapsed_k} outside [1, {interval_n - 1}]")


@dataclass
class AttnCounters:
    """Instrumentation for one attention call (attention.py:138-147)."""

    pairs_total: int = 0
    pairs_computed: int = 0

    @property
    def pairs_skipped(self):
        return self.pairs_total - self.pairs_computed


@dataclass
class CacheEntry:
    """Host view of one (head, block) entry (attention.py:58-69)."""

    diff_stack: np.ndarray
    valid_orders: int = 0


class FeatureCache:
    """Per (head, query block) backward-difference stacks for one layer, in HBM.

    stacks: bf16 [order+1, seq, heads*128] — slot d holds the d-th backward
    difference of every tile, laid out like the attention output so the GEMM-O
    update reads it with the same TMA descriptor shape. valid: int32 [heads,
    n_blocks] valid orders per entry (attention.py:116-135). Storage is
    allocated on the first push (the sequence length comes from the tiles).
    """

    def __init__(self, heads, n_blocks, order, seq=None, device=None):
        if order < 0:
            raise ParameterError(f"order must be >= 0, got {order}")
        require_cuda()
        self.heads, self.n_blocks, self.order = int(heads), int(n_blocks), int(order)
        self.device = device or "cuda"
        self.valid = torch.zeros(self.heads, self.n_blocks, dtype=torch.int32, device=self.device)
        self.stacks = None
        self.seq = None
        self.version = 0  # bumped on every push; keys the cached plans
        # per-entry mode: a cache that receives per-tile updates before any
        # sequence length is known keeps, like the reference (attention.py:
        # 116-135), one fp32 device stack per (head, block) at any tile shape
        self._entries = None
        if seq is not None:
            self._alloc(seq)

    @property
    def per_entry(self):
        """True once the cache holds per-entry fp32 stacks (any tile shape)."""
        return self._entries is not None

    def _alloc(self, seq):
        if self._entries is not None:
            raise StateError("this cache holds per-entry tiles; layer pushes need a cache made "
                             "with seq=")
        if self.order > 3:
            raise ParameterError(f"order must be in [0, 3] for the HBM stacks, got {self.order}")
        if ceil_div(seq, TILE) != self.n_blocks:
            raise ShapeError(f"seq {seq} gives {ceil_div(seq, TILE)} blocks, cache has {self.n_blocks}")
        self.seq = int(seq)
        self.stacks = torch.zeros(self.order + 1, self.seq, self.heads * TILE, dtype=torch.bfloat16,
                                  device=self.device)

    def ensure(self, seq):
        if self.stacks is None:
            self._alloc(seq)
        elif seq != self.seq:
            raise ShapeError(f"tile rows {seq} != cached {self.seq}")

    def push(self, o, select=None, stream=None, check=True):
        """Push fresh outputs o [seq, heads, 128] into every (selected) entry."""
        o = check_bsd(o, "o", heads=self.heads)
        if check:  # update_entry's as_matrix(o_new) (attention.py:73)
            check_finite(o, "tile", stream=stream)
        self.ensure(o.shape[0])
        sel = None
        if select is not None:
            sel = torch.as_tensor(select, dtype=torch.uint8).to(self.device).contiguous()
            if tuple(sel.shape) != (self.heads, self.n_blocks):
                raise ShapeError(f"select shape {tuple(sel.shape)} != {(self.heads, self.n_blocks)}")
        _lib.call("fo_cache_push", o.data_ptr(), self.stacks.data_ptr(), self.valid.data_ptr(),
                  self.seq, self.heads, TILE, self.n_blocks, self.order, _lib.ptr(sel),
                  stream_ptr(stream))
        self.version += 1
        self._sel_keep = sel  # keep alive until the launch retires

    def update(self, head, block, o_new):
        """Reference signature (attention.py:128-131): push one tile o_new
        (numpy or torch) into entry (head, block). A cache made with seq= takes
        [rows, 128] tiles into its HBM stacks (one tile-sized launch,
        fo_cache_push_tile; nothing synchronises for device tiles); a cache
        without one keeps per-entry fp32 device stacks at any tile shape
        (fo_update_entry), as the reference does."""
        if isinstance(o_new, torch.Tensor):
            tile = o_new
            if tile.dim() == 2 and not bool(torch.isfinite(tile).all()):
                raise ParameterError("tile: contains NaN or Inf")
        else:
            arr = np.asarray(o_new, dtype=np.float32)
            if arr.ndim == 2 and not np.isfinite(arr).all():
                raise ParameterError("tile: contains NaN or Inf")
            tile = torch.from_numpy(np.ascontiguousarray(arr))
        if not (0 <= head < self.heads and 0 <= block < self.n_blocks):
            raise IndexError(f"entry ({head}, {block}) outside ({self.heads}, {self.n_blocks})")
        if self.stacks is None:  # no seq given: per-entry fp32 stacks, any tile shape
            if self._entries is None:
                self._entries = [[None] * self.n_blocks for _ in range(self.heads)]
            e = update_entry(self._entries[head][block],
                             tile.to(self.device, torch.float32).contiguous(), self.order)
            self._entries[head][block] = e
            self.valid[head, block] = e.valid_orders
            self.version += 1
            return
        if tile.dim() != 2 or tile.shape[1] != TILE:
            raise ShapeError(f"tile shape {tuple(tile.shape)}; head_dim must be {TILE}")
        rows = min(TILE, self.seq - block * TILE)
        if tile.shape[0] != rows:
            raise ShapeError(f"tile shape {tuple(tile.shape)} != cached ({rows}, {TILE})")
        t = tile.to(self.device, torch.bfloat16).contiguous()
        _lib.call("fo_cache_push_tile", t.data_ptr(), self.stacks.data_ptr(), self.valid.data_ptr(),
                  self.seq, self.heads, TILE, self.n_blocks, self.order, int(head), int(block),
                  stream_ptr(None))
        self.version += 1

    def valid_orders(self, head, block):
        if self._entries is not None:
            e = self._entries[head][block]
            return 0 if e is None else int(e.valid_orders)
        return int(self.valid[head, block].item())

    def device_entry(self, head, block):
        """Per-entry mode: the entry with its device fp32 stack (or None)."""
        return None if self._entries is None else self._entries[head][block]

    def entry(self, head, block):
        if self._entries is not None:
            e = self._entries[head][block]
            if e is None:
                return None
            return CacheEntry(diff_stack=e.diff_stack.cpu().numpy(), valid_orders=e.valid_orders)
        if self.valid_orders(head, block) < 1:
            return None
        r0 = block * TILE
        rows = min(TILE, self.seq - r0)
        st = self.stacks[:, r0:r0 + rows, head * TILE:(head + 1) * TILE].float().cpu().numpy()
        return CacheEntry(diff_stack=st, valid_orders=self.valid_orders(head, block))


# ---------------------------------------------------------------------------
# Tile-level building blocks of the reference API (attention.py:21-113), on
# the device (csrc/fo_numerics.cu). numpy in -> numpy out, torch in -> torch.


def _f32(a, name=None, finite=False):
    host = not isinstance(a, torch.Tensor)
    require_cuda()
    t = torch.as_tensor(np.asarray(a, dtype=DTYPE)) if host else a
    t = t.to("cuda" if host or not t.is_cuda else t.device, torch.float32).contiguous()
    if finite and not bool(torch.isfinite(t).all()):
        raise ParameterError(f"{name}: contains NaN or Inf")
    return t, host


def _back(t, host):
    return t.cpu().numpy() if host else t


@dataclass
class OnlineSoftmaxState:
    """Running max, normalizer and unnormalized accumulator per query row
    (attention.py:21-36)."""

    m: object
    l: object
    acc: object

    @classmethod
    def fresh(cls, rows, d):
        return cls(m=np.full(rows, -np.inf, dtype=DTYPE), l=np.zeros(rows, dtype=DTYPE),
                   acc=np.zeros((rows, d), dtype=DTYPE))


def online_softmax_update(state, scores, v_block):
    """Fold one score block into the running softmax state (attention.py:39-49),
    one CTA per row (fo_online_softmax_update)."""
    s, host = _f32(scores)
    v, _ = _f32(v_block)
    m, _ = _f32(state.m)
    l, _ = _f32(state.l)
    acc, _ = _f32(state.acc)
    if s.dim() != 2 or v.dim() != 2 or acc.dim() != 2:
        raise ShapeError("online_softmax_update: scores, v_block and acc must be 2-D")
    rows, cols = s.shape
    d = v.shape[1]
    if v.shape[0] != cols or tuple(acc.shape) != (rows, d) or m.numel() != rows or l.numel() != rows:
        raise ShapeError(f"online_softmax_update: scores {tuple(s.shape)}, v {tuple(v.shape)}, "
                         f"acc {tuple(acc.shape)}, m/l {m.numel()}/{l.numel()}")
    m_o, l_o, acc_o = torch.empty_like(m), torch.empty_like(l), torch.empty_like(acc)
    _lib.call("fo_online_softmax_update", m.data_ptr(), l.data_ptr(), acc.data_ptr(), s.data_ptr(),
              v.data_ptr(), rows, cols, d, m_o.data_ptr(), l_o.data_ptr(), acc_o.data_ptr(),
              stream_ptr(None))
    return OnlineSoftmaxState(m=_back(m_o, host), l=_back(l_o, host), acc=_back(acc_o, host))


def online_softmax_finalize(state):
    """Normalize the accumulator, diag(l)^-1 acc (attention.py:52-55); an empty
    row (l <= 0) raises ConsistencyError."""
    acc, host = _f32(state.acc)
    l, _ = _f32(state.l)
    if acc.dim() != 2 or l.numel() != acc.shape[0]:
        raise ShapeError("online_softmax_finalize: acc must be [rows, d] with one l per row")
    out = torch.empty_like(acc)
    st = Status.default()
    st.check("online_softmax_finalize")
    _lib.call("fo_online_softmax_finalize", acc.data_ptr(), l.data_ptr(), acc.shape[0],
              acc.shape[1], out.data_ptr(), st.ptr(), stream_ptr(None))
    bits = int(st.t.item())
    if bits:
        st.t.zero_()
        raise ConsistencyError("softmax state finalized with an empty row")
    return _back(out, host)


def update_entry(entry, o_new, order):
    """Push a fresh tile output, shifting differences one level deeper
    (attention.py:71-85): stack[0] = o_new, stack[d] = stack[d-1] - old[d-1]
    for d < valid = min(old valid + 1, order + 1) (fo_update_entry)."""
    o, host = _f32(o_new, "tile", finite=True)
    if o.dim() != 2:
        raise ShapeError(f"tile: expected a 2-D matrix, got shape {tuple(o.shape)}")
    if order < 0:
        raise ParameterError(f"order must be >= 0, got {order}")
    stack = torch.empty((order + 1,) + tuple(o.shape), dtype=torch.float32, device=o.device)
    old, old_valid = None, 0
    if entry is not None:
        old, _ = _f32(entry.diff_stack)
        if tuple(old.shape[1:]) != tuple(o.shape):
            raise ShapeError(f"tile shape {tuple(o.shape)} != cached {tuple(old.shape[1:])}")
        old_valid = min(int(entry.valid_orders), old.shape[0])
    _lib.call("fo_update_entry", None if old is None else old.data_ptr(), old_valid, o.data_ptr(),
              o.numel(), int(order), stack.data_ptr(), stream_ptr(None))
    valid = 1 if entry is None else min(int(entry.valid_orders) + 1, order + 1)
    return CacheEntry(diff_stack=_back(stack, host), valid_orders=valid)


def forecast(entry, elapsed_k, interval_n, order_d):
    """Extrapolate a cached tile elapsed_k steps past its last update
    (attention.py:96-113): sum_{d < min(order_d+1, valid)} c_d * stack[d]
    (fo_forecast_entry). StateError for a cold entry, then ParameterError for
    elapsed_k outside [1, N-1], in the reference's order."""
    if entry is None or entry.valid_orders < 1:
        raise StateError("forecast requested from a cold cache entry")
    check_elapsed(elapsed_k, interval_n)
    st, host = _f32(entry.diff_stack)
    n_orders = min(order_d + 1, int(entry.valid_orders))
    coef = forecast_coefficients(elapsed_k, interval_n, n_orders)
    c = (ctypes.c_float * len(coef))(*coef.tolist())
    tile = st[0].numel()
    out = torch.empty(tuple(st.shape[1:]), dtype=torch.float32, device=st.device)
    _lib.call("fo_forecast_entry", st.data_ptr(), tile, n_orders, ctypes.addressof(c),
              out.data_ptr(), stream_ptr(None))
    return _back(out, host)


# ---------------------------------------------------------------------------
def _as_matrix(a, name, finite=True):
    """tensor.py:19-30 as_matrix: C-contiguous float32 2-D, finite unless opted out."""
    m = np.ascontiguousarray(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                             dtype=DTYPE)
    if m.ndim != 2:
        raise ShapeError(f"{name}: expected a 2-D matrix, got shape {m.shape}")
    if finite and not np.isfinite(m).all():
        raise ParameterError(f"{name}: contains NaN or Inf")
    return m


def masked_block_attention_f32(q, k, v, active, pair_bits, b_q, b_k, scale, out):
    """The reference tile-kernel protocol (pyref.py:14-48) at any block size and
    head dim <= 256, in fp32 on the GPU (fo_masked_block_attention_f32): writes
    the rows of active blocks into `out` (numpy [n, d]) and returns the computed
    pair count; an active block with no key block raises ConsistencyError."""
    require_cuda()
    q, k, v = (torch.from_numpy(_as_matrix(a, nm, finite=False)).cuda()
               for a, nm in ((q, "q"), (k, "k"), (v, "v")))
    n, d = q.shape
    if tuple(k.shape) != (n, d) or tuple(v.shape) != (n, d):
        raise ShapeError(f"q/k/v shapes {tuple(q.shape)}/{tuple(k.shape)}/{tuple(v.shape)} differ")
    if d > 256:
        raise ParameterError(f"head dim {d} > 256")
    t_q, t_kv = ceil_div(n, b_q), ceil_div(n, b_k)
    act = torch.as_tensor(np.asarray(active, dtype=np.uint8).reshape(-1)).cuda()
    pb = torch.as_tensor(np.ascontiguousarray(pair_bits, dtype=np.uint8)).cuda()
    if tuple(act.shape) != (t_q,) or tuple(pb.shape) != (t_q, t_kv):
        raise ShapeError(f"mask shapes {tuple(act.shape)}/{tuple(pb.shape)} for {t_q}x{t_kv} blocks")
    res = torch.from_numpy(np.ascontiguousarray(out, dtype=DTYPE)).cuda()
    pairs = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = Status()
    _lib.call("fo_masked_block_attention_f32", q.data_ptr(), k.data_ptr(), v.data_ptr(), n, d,
              act.data_ptr(), pb.data_ptr(), int(b_q), int(b_k), float(scale), res.data_ptr(),
              pairs.data_ptr(), st.ptr(), stream_ptr(None))
    bits = int(st.t.item())
    if bits & _lib.ST_CONSISTENCY:
        raise ConsistencyError("active query block has every key block skipped")
    _lib.raise_status(bits, "masked_block_attention")
    out[...] = res.cpu().numpy()
    return int(pairs.item())


def _per_head_general(q, k, v, symbols, cache, head, elapsed_k, interval_n, order_d, b_q, b_k,
                      mode, counters, fill):
    """Reference per-head signature at any block size / head dim, fp32
    (attention.py:150-221, step for step): the symbols decode on the GPU, the
    tile kernel is fo_masked_block_attention_f32 and cached blocks take their
    forecast from the cache's per-entry device stacks (fo_forecast_entry)."""
    q = _as_matrix(q, "q", finite=False)
    k = _as_matrix(k, "k")
    v = _as_matrix(v, "v")
    if mode not in ("materialize", "bias"):
        raise ParameterError(f"unknown mode {mode!r}")
    n, d = q.shape
    t_q, t_kv = ceil_div(n, b_q), ceil_div(n, b_k)
    if (symbols.rows, symbols.cols) != (t_q, t_kv):
        raise ShapeError(f"symbols dimensioned {symbols.rows}x{symbols.cols}, "
                         f"expected {t_q}x{t_kv}")
    sym = symbols if isinstance(symbols, DeviceSymbols) else DeviceSymbols.from_buffers([symbols])
    act_d, pair_d = sym.decoded()
    active = act_d[0].cpu().numpy()
    read_rows = np.repeat(active.astype(bool), b_q)[:n]
    if not np.isfinite(q[read_rows]).all():
        raise ParameterError("q: active-block rows contain NaN or Inf")
    out = np.full((n, d), fill, dtype=DTYPE)
    pairs = masked_block_attention_f32(q, k, v, active, pair_d[0].cpu().numpy(), b_q, b_k,
                                       1.0 / math.sqrt(d), out)
    for i in np.flatnonzero(active == 0):
        entry = None
        if cache is not None:
            entry = cache.device_entry(head, i) if cache.per_entry else cache.entry(head, i)
        if entry is None or entry.valid_orders < 1:
            raise StateError(f"query block {i} is cached but the cache is cold")
        if mode == "materialize":
            f = forecast(entry, elapsed_k, interval_n, order_d)
            f = f.cpu().numpy() if isinstance(f, torch.Tensor) else f
            out[i * b_q:i * b_q + f.shape[0]] = f
    if counters is not None:
        counters.pairs_total += t_q * t_kv
        counters.pairs_computed += pairs
    return out


def _per_head_adapter(q, k, v, symbols, cache, head, elapsed_k, interval_n, order_d, b_q, b_k,
                      mode, counters, fill):
    """Reference per-head signature: numpy [n, d] in, numpy fp32 out."""
    q, k, v = (torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)) for a in (q, k, v))
    if q.dim() != 2:
        raise ShapeError(f"q: expected a 2-D matrix, got shape {tuple(q.shape)}")
    if q.shape[1] != TILE:
        raise ParameterError(f"the B200 engine is built for head_dim {TILE}, got {q.shape[1]}")
    dev = "cuda"
    qd, kd, vd = (a.to(dev, torch.bfloat16).unsqueeze(1) for a in (q, k, v))
    sym = symbols if isinstance(symbols, DeviceSymbols) else DeviceSymbols.from_buffers([symbols])
    sub = None
    if cache is not None:
        sub = FeatureCache(1, cache.n_blocks, cache.order, seq=cache.seq)
        sub.valid.copy_(cache.valid[head:head + 1])
        if cache.stacks is not None:
            sub.stacks.copy_(cache.stacks[:, :, head * TILE:(head + 1) * TILE])
    out = torch.full_like(qd, float(fill), dtype=torch.bfloat16)
    res = sparse_attention(qd, kd, vd, sym, sub, None, elapsed_k, interval_n, order_d, b_q=b_q,
                           b_k=b_k, mode=mode, counters=counters, out=out)
    arr = res[:, 0].float().cpu().numpy()
    if fill is not None and np.isnan(fill):
        # rows never written keep the caller's placeholder exactly
        active, _ = sym.decoded()
        rows = np.repeat(active[0].cpu().numpy().astype(bool), TILE)[: arr.shape[0]]
        if mode == "bias":
            arr[~rows] = np.nan
    return arr


def sparse_attention(q, k, v, symbols, cache, head, elapsed_k, interval_n, order_d, *, b_q=TILE,
                     b_k=TILE, mode="materialize", counters=None, backend=None, fill=0.0, out=None,
                     stream=None, status=None, check=True, plan=None, pairs=None):
    """Symbol-guided attention for every head of a layer (attention.py:150-221).

    q, k, v: bf16 [seq, heads, 128] on the GPU. symbols: DeviceSymbols.
    cache: FeatureCache or None. mode="bias" leaves cached tiles untouched in
    `out` (pre-filled with `fill` when `out` is not given); mode="materialize"
    writes their forecast. Returns out [seq, heads, 128] bf16.
    check=False defers the device contract checks (errors stay latched in the
    status word) so the call never synchronises. plan overrides the cached
    schedule (the engine's static plans); pairs is an optional int64 [heads]
    device accumulator of computed pairs (no host read).
    """
    if backend is not None and getattr(backend, "NAME", "b200") != "b200":
        raise ParameterError("this engine runs only its sm_100a kernels")
    if isinstance(q, np.ndarray) or isinstance(symbols, SymbolBuffer):
        # the reference's per-head numpy signature: 128-token blocks at head dim
        # 128 run on the tcgen05 kernel; any other shape (or a per-entry cache)
        # on the fp32 tile kernel
        if (b_q != TILE or b_k != TILE or np.shape(q)[-1] != TILE
                or (cache is not None and cache.per_entry)):
            return _per_head_general(q, k, v, symbols, cache, head, elapsed_k, interval_n,
                                     order_d, b_q, b_k, mode, counters, fill)
        if mode not in ("materialize", "bias"):
            raise ParameterError(f"unknown mode {mode!r}")
        return _per_head_adapter(q, k, v, symbols, cache, head, elapsed_k, interval_n, order_d,
                                 b_q, b_k, mode, counters, fill)
    if mode not in ("materialize", "bias"):
        raise ParameterError(f"unknown mode {mode!r}")
    if b_q != TILE or b_k != TILE:
        raise ParameterError(f"the sm_100a kernels tile blocks of {TILE} tokens (b_q=b_k={TILE})")
    require_cuda()
    q = check_bsd(q, "q")
    seq, heads = q.shape[0], q.shape[1]
    k = check_bsd(k, "k", seq, heads)
    v = check_bsd(v, "v", seq, heads)
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.dtype != torch.bfloat16 or not t.is_cuda:
            raise ParameterError(f"{name}: expected a CUDA bf16 tensor")
    t_q = ceil_div(seq, TILE)
    if (symbols.rows, symbols.cols) != (t_q, t_q):
        raise ShapeError(f"symbols dimensioned {symbols.rows}x{symbols.cols}, expected {t_q}x{t_q}")
    if symbols.heads != heads:
        raise ShapeError(f"symbols for {symbols.heads} heads, q has {heads}")
    st = status or Status.default()
    if cache is not None:
        if cache.per_entry:
            raise StateError("a per-entry cache (no seq=) serves the per-head signature only")
        if (cache.heads, cache.n_blocks) != (heads, t_q):
            raise ShapeError("feature cache geometry does not match q")
        valid, vver = cache.valid, cache.version
    else:
        # no cache at all: any cached block is a cold-cache StateError
        valid, vver = _zeros_valid(heads, t_q, q.device), -1
    if plan is None:
        plan = symbols.plan(valid=valid, valid_version=vver, order_d=order_d, status=st,
                            stream=stream, check=check)
    if mode == "materialize" and (interval_n < 1 or not 1 <= elapsed_k <= interval_n - 1):
        # the reference validates elapsed_k inside forecast(), i.e. only for a
        # cached block and after its cold-cache StateError (attention.py:104-107,
        # 208-216): all-active symbols with any elapsed_k are legal
        if int(plan.counts()[1]) < heads * t_q:
            st.check("sparse_attention")
            check_elapsed(elapsed_k, interval_n)
    if check:
        # as_matrix (tensor.py:19-30): q only on the rows it reads (attention.py:176-196)
        check_finite(q, "q: active-block rows", st, plan=plan, stream=stream)
        check_finite(k, "k", st, stream=stream)
        check_finite(v, "v", st, stream=stream)
    if out is None:
        out = torch.full((seq, heads, TILE), float(fill) if fill is not None else 0.0,
                         dtype=torch.bfloat16, device=q.device)
    else:
        check_out(out, "out", (seq, heads, TILE), device=q.device)
    if pairs is None and counters is not None:
        pairs = torch.zeros(heads, dtype=torch.int64, device=q.device)
    if mode == "materialize" and cache is not None and cache.stacks is not None:
        # one launch: computed tiles + the cached tiles' OP_reuse fused in (K2r)
        coef = ctypes_floats(forecast_coefficients(elapsed_k, interval_n, order_d + 1))
        _lib.call("fo_sparse_attention_reuse", q.data_ptr(), k.data_ptr(), v.data_ptr(), seq,
                  heads, TILE, symbols.s_s.data_ptr(), symbols.rows, symbols.cols, symbols.pool_n,
                  plan.ptr(), 1.0 / math.sqrt(TILE), cache.stacks.data_ptr(),
                  cache.valid.data_ptr(), min(order_d, cache.order), ctypes.addressof(coef),
                  out.data_ptr(), _lib.ptr(pairs), st.ptr(), stream_ptr(stream))
    else:
        # mode="bias" (cached rows untouched), or nothing cached can be read: the
        # plan has latched a cold-cache StateError for any cached tile
        _lib.call("fo_sparse_attention", q.data_ptr(), k.data_ptr(), v.data_ptr(), seq, heads,
                  TILE, symbols.s_s.data_ptr(), symbols.rows, symbols.cols, symbols.pool_n,
                  plan.ptr(), 1.0 / math.sqrt(TILE), 0, out.data_ptr(), None, None, order_d,
                  _lib.ptr(pairs), st.ptr(), stream_ptr(stream))
    if check:
        st.check("sparse_attention")
    if counters is not None:
        counters.pairs_total += heads * t_q * t_q
        counters.pairs_computed += int(pairs.sum().item())
    return out


def dense_attention_update(q, k, v, cache, *, out=None, counters=None, stream=None, status=None,
                           check=True):
    """Update-step attention (pipeline.py:268-278): dense over every pair, and
    the epilogue pushes each fresh tile into the cache's difference stacks in
    place (K2u) — no separate cache pass."""
    require_cuda()
    q = check_bsd(q, "q")
    seq, heads = q.shape[0], q.shape[1]
    k = check_bsd(k, "k", seq, heads)
    v = check_bsd(v, "v", seq, heads)
    t_q = ceil_div(seq, TILE)
    if cache is not None:
        if (cache.heads, cache.n_blocks) != (heads, t_q):
            raise ShapeError("feature cache geometry does not match q")
        cache.ensure(seq)
    st = status or Status.default()
    plan = _dense_plan(heads, t_q, q.device, st, stream)
    if check:
        for name, t in (("q", q), ("k", k), ("v", v)):
            check_finite(t, name, st, stream=stream)
    if out is None:
        out = torch.empty(seq, heads, TILE, dtype=torch.bfloat16, device=q.device)
    else:
        check_out(out, "out", (seq, heads, TILE), device=q.device)
    pairs = torch.zeros(heads, dtype=torch.int64, device=q.device) if counters is not None else None
    _lib.call("fo_sparse_attention", q.data_ptr(), k.data_ptr(), v.data_ptr(), seq, heads, TILE,
              plan.sym.s_s.data_ptr(), t_q, t_q, 1, plan.ptr(), 1.0 / math.sqrt(TILE),
              1 if cache is not None else 0,
              out.data_ptr(), None if cache is None else cache.stacks.data_ptr(),
              None if cache is None else cache.valid.data_ptr(),
              0 if cache is None else cache.order, _lib.ptr(pairs), st.ptr(), stream_ptr(stream))
    if cache is not None:
        cache.version += 1
    if check:
        st.check("dense_attention_update")
    if counters is not None:
        counters.pairs_total += heads * t_q * t_q
        counters.pairs_computed += int(pairs.sum().item())
    return out


# ---------------------------------------------------------------------------
_DENSE = {}
_ZEROS = {}


def _zeros_valid(heads, t_q, device):
    key = (heads, t_q, str(device))
    if key not in _ZEROS:
        _ZEROS[key] = torch.zeros(heads, t_q, dtype=torch.int32, device=device)
    return _ZEROS[key]


def _dense_plan(heads, t_q, device, status, stream):
    """Plan with every (head, block) active and every key block (update step)."""
    key = (heads, t_q, str(device))
    pl = _DENSE.get(key)
    if pl is None:
        from .symbols import encode_symbols

        sym = encode_symbols(torch.ones(heads, t_q, dtype=torch.uint8, device=device),
                             torch.ones(heads, t_q, t_q, dtype=torch.uint8, device=device), 1)
        pl = sym.plan(dense=True, status=status, stream=stream)
        pl.sym = sym
        _DENSE[key] = pl
    return pl


def ctypes_floats(arr):
    a = np.zeros(4, np.float32)
    a[: len(arr)] = arr
    return (ctypes.c_float * 4)(*a.tolist())
