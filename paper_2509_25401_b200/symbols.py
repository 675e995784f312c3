"""Compact sparse symbols: byte-packed block masks, packed and decoded on the GPU.

Format (identical to reference pkg/src/omniattn/symbols.py:1-25): one bit per
compressed group of `pool_n` blocks, MSB-first within a byte, zero-padded; each
compressed skip-mask row starts on a byte boundary. Compressed cache bits
[1,1,1,0,0] pack to the single byte 224.

Two containers:
  SymbolBuffer   host bytes for one head, with the 16-byte little-endian wire
                 header (rows, cols, pool_n, version) of symbols.py:84-142.
  DeviceSymbols  every head of a layer resident in HBM: s_c uint8 [H, sc_len],
                 s_s uint8 [H, comp_rows, row_stride] — byte-identical to the
                 concatenation of the per-head buffers. This is what the kernels
                 read; their prologues decode it on the fly.
Packing (K1, fo_encode_symbols) and decoding (fo_decode_symbols, the same
device decoders the attention/GEMM prologues use) run on the GPU.
"""

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._runtime import Status, as_device, require_cuda, stream_ptr
from .errors import BoundsError, ConsistencyError, ShapeError

SYMBOL_FORMAT_VERSION = 1
_HEADER = struct.Struct("<4I")


def ceil_div(a, b):
    return -(-a // b)


@dataclass(frozen=True)
class SymbolBuffer:
    """Byte-packed cache/skip symbols for one attention head (symbols.py:84-142)."""

    s_c: bytes
    s_s: bytes
    rows: int
    cols: int
    pool_n: int

    def __post_init__(self):
        if len(self.s_c) != ceil_div(self.comp_rows, 8):
            raise ConsistencyError(
                f"s_c length {len(self.s_c)} != expected {ceil_div(self.comp_rows, 8)}"
            )
        if len(self.s_s) != self.comp_rows * self.row_stride:
            raise ConsistencyError(
                f"s_s length {len(self.s_s)} != expected {self.comp_rows * self.row_stride}"
            )

    @property
    def comp_rows(self):
        return ceil_div(self.rows, self.pool_n)

    @property
    def comp_cols(self):
        return ceil_div(self.cols, self.pool_n)

    @property
    def row_stride(self):
        return ceil_div(self.comp_cols, 8)

    def to_bytes(self):
        header = _HEADER.pack(self.rows, self.cols, self.pool_n, SYMBOL_FORMAT_VERSION)
        return header + self.s_c + self.s_s

    @classmethod
    def from_bytes(cls, data):
        if len(data) < _HEADER.size:
            raise ConsistencyError("symbol blob shorter than header")
        rows, cols, pool_n, version = _HEADER.unpack_from(data)
        if version != SYMBOL_FORMAT_VERSION:
            raise ConsistencyError(f"unsupported symbol format version {version}")
        comp_rows = ceil_div(rows, pool_n)
        n_c = ceil_div(comp_rows, 8)
        n_s = comp_rows * ceil_div(ceil_div(cols, pool_n), 8)
        if len(data) != _HEADER.size + n_c + n_s:
            raise ConsistencyError("symbol blob length inconsistent with header")
        return cls(s_c=bytes(data[_HEADER.size:_HEADER.size + n_c]),
                   s_s=bytes(data[_HEADER.size + n_c:]), rows=rows, cols=cols, pool_n=pool_n)


class DeviceSymbols:
    """All heads' symbols of one layer, resident on the GPU."""

    def __init__(self, s_c, s_s, rows, cols, pool_n):
        self.rows, self.cols, self.pool_n = int(rows), int(cols), int(pool_n)
        if self.pool_n < 1:
            raise ConsistencyError(f"pool_n must be >= 1, got {pool_n}")
        self.heads = int(s_c.shape[0])
        if tuple(s_c.shape) != (self.heads, self.sc_len):
            raise ConsistencyError(f"s_c shape {tuple(s_c.shape)} != {(self.heads, self.sc_len)}")
        if tuple(s_s.shape) != (self.heads, self.comp_rows, self.row_stride):
            raise ConsistencyError(
                f"s_s shape {tuple(s_s.shape)} != {(self.heads, self.comp_rows, self.row_stride)}")
        self.s_c = s_c.contiguous()
        self.s_s = s_s.contiguous()
        self._decoded = None
        self._plans = {}

    comp_rows = property(lambda self: ceil_div(self.rows, self.pool_n))
    comp_cols = property(lambda self: ceil_div(self.cols, self.pool_n))
    row_stride = property(lambda self: ceil_div(self.comp_cols, 8))
    sc_len = property(lambda self: ceil_div(self.comp_rows, 8))

    # ------------------------------------------------------------ conversions
    @classmethod
    def from_buffers(cls, buffers, device=None):
        """Upload per-head SymbolBuffers (all with equal geometry)."""
        buffers = list(buffers)
        if not buffers:
            raise ShapeError("no symbol buffers")
        b0 = buffers[0]
        for b in buffers:
            if (b.rows, b.cols, b.pool_n) != (b0.rows, b0.cols, b0.pool_n):
                raise ShapeError("symbol buffers of one layer must share rows/cols/pool_n")
        require_cuda()
        sc = np.frombuffer(b"".join(b.s_c for b in buffers), np.uint8).reshape(len(buffers), -1)
        ss = np.frombuffer(b"".join(b.s_s for b in buffers), np.uint8).reshape(
            len(buffers), b0.comp_rows, b0.row_stride)
        dev = device or "cuda"
        return cls(torch.from_numpy(sc.copy()).to(dev), torch.from_numpy(ss.copy()).to(dev),
                   b0.rows, b0.cols, b0.pool_n)

    def to_buffers(self):
        sc = self.s_c.cpu().numpy()
        ss = self.s_s.cpu().numpy()
        return [SymbolBuffer(s_c=sc[h].tobytes(), s_s=ss[h].tobytes(), rows=self.rows,
                             cols=self.cols, pool_n=self.pool_n) for h in range(self.heads)]

    def head(self, h):
        return DeviceSymbols(self.s_c[h:h + 1], self.s_s[h:h + 1], self.rows, self.cols, self.pool_n)

    def select_heads(self, idx):
        """Symbols of a subset of heads (head-sharded ranks)."""
        idx = torch.as_tensor(idx, dtype=torch.long, device=self.s_c.device)
        return DeviceSymbols(self.s_c.index_select(0, idx), self.s_s.index_select(0, idx),
                             self.rows, self.cols, self.pool_n)

    # ------------------------------------------------------------ device decode
    def decoded(self, stream=None):
        """(active uint8 [H, rows], pair_bits uint8 [H, rows, cols]) decoded on
        the GPU by the kernels' prologue decoders (symbols.py:163-198)."""
        if self._decoded is None:
            active = torch.empty(self.heads, self.rows, dtype=torch.uint8, device=self.s_c.device)
            pairs = torch.empty(self.heads, self.rows, self.cols, dtype=torch.uint8,
                                device=self.s_c.device)
            _lib.call("fo_decode_symbols", self.s_c.data_ptr(), self.s_s.data_ptr(), self.heads,
                      self.rows, self.cols, self.pool_n, active.data_ptr(), pairs.data_ptr(),
                      stream_ptr(stream))
            self._decoded = (active, pairs)
        return self._decoded

    def plan(self, valid=None, valid_version=None, order_d=0, dense=False, status=None,
             stream=None, check=True):
        """Schedule derived from the symbols. Symbols only change at update
        steps, so the plan is cached and reused by every dispatch step of the
        window; `valid_version` (the feature cache's update counter) keys it."""
        from .plan import Plan

        key = (None if valid is None else (valid.data_ptr(), valid_version),
               int(order_d), bool(dense))
        pl = self._plans.get(key)
        if pl is None:
            pl = Plan.build(self, valid=valid, order_d=order_d, dense=dense, status=status,
                            stream=stream, check=check)
            self._plans[key] = pl
        return pl

    def invalidate(self):
        self._plans.clear()
        self._decoded = None


# ---------------------------------------------------------------------------
# encoders (K1 on device)
# ---------------------------------------------------------------------------
def encode_symbols(cache_bits, skip_bits, pool_n, status=None, stream=None, check=True, out=None):
    """Pack every head at once. cache_bits [H, rows], skip_bits [H, rows, cols]
    (bool/uint8, any device) -> DeviceSymbols. Mirrors build_symbols
    (symbols.py:145-160) including its ConsistencyError for mixed pool groups."""
    if pool_n < 1:
        raise ConsistencyError(f"pool_n must be >= 1, got {pool_n}")
    cb = as_device(cache_bits, torch.uint8, "cache mask")
    sb = as_device(skip_bits, torch.uint8, "skip mask")
    if cb.dim() == 1:
        cb = cb.unsqueeze(0)
    if sb.dim() == 2:
        sb = sb.unsqueeze(0)
    if cb.dim() != 2:
        raise ShapeError(f"cache mask: expected [heads, rows], got {tuple(cb.shape)}")
    if sb.dim() != 3:
        raise ShapeError(f"skip mask: expected [heads, rows, cols], got {tuple(sb.shape)}")
    heads, rows = cb.shape
    if sb.shape[0] != heads or sb.shape[1] != rows:
        raise ShapeError(f"skip mask has {sb.shape[1]} rows, cache mask has {rows}")
    cols = sb.shape[2]
    comp_rows, comp_cols = ceil_div(rows, pool_n), ceil_div(cols, pool_n)
    if out is not None:
        # rewrite a resident DeviceSymbols in place (static buffers of the engine)
        if (out.heads, out.rows, out.cols, out.pool_n) != (heads, rows, cols, pool_n):
            raise ShapeError("encode_symbols: out geometry differs from the masks")
        s_c, s_s = out.s_c, out.s_s
        out.invalidate()
    else:
        s_c = torch.empty(heads, ceil_div(comp_rows, 8), dtype=torch.uint8, device=cb.device)
        s_s = torch.empty(heads, comp_rows, ceil_div(comp_cols, 8), dtype=torch.uint8,
                          device=cb.device)
    st = status or Status.default()
    _lib.call("fo_encode_symbols", cb.data_ptr(), sb.data_ptr(), heads, rows, cols, pool_n,
              s_c.data_ptr(), s_s.data_ptr(), st.ptr(), stream_ptr(stream))
    if check:
        st.check("encode_symbols")
    return out if out is not None else DeviceSymbols(s_c, s_s, rows, cols, pool_n)


def _bits(bits, ndim, name):
    arr = np.asarray(bits)
    if arr.ndim != ndim:
        raise ShapeError(f"{name}: expected {ndim}-D bit array, got shape {arr.shape}")
    return arr.astype(bool)


def build_symbols(cache_bits, skip_bits, pool_n):
    """Reference-signature encoder for one head (symbols.py:145-160): packs on
    the GPU and returns the host SymbolBuffer."""
    cb = _bits(cache_bits, 1, "cache mask")
    sb = _bits(skip_bits, 2, "skip mask")
    if sb.shape[0] != cb.shape[0]:
        raise ShapeError(f"skip mask has {sb.shape[0]} rows, cache mask has {cb.shape[0]}")
    if pool_n < 1:
        raise ConsistencyError(f"pool_n must be >= 1, got {pool_n}")
    return encode_symbols(cb[None], sb[None], pool_n).to_buffers()[0]


def encode_cache_mask(bits, pool_n):
    """symbols.py:65-70 on the GPU: bytes of one packed cache-mask row."""
    b = _bits(bits, 1, "cache mask")
    return build_symbols(b, np.zeros((b.size, 1), bool), pool_n).s_c


def encode_skip_mask(bits, pool_n):
    """symbols.py:73-81 on the GPU: concatenated byte-aligned skip rows."""
    b = _bits(bits, 2, "skip mask")
    if pool_n < 1:
        raise ConsistencyError(f"pool_n must be >= 1, got {pool_n}")
    # cache bits must be pool-uniform too; use all-ones so only the skip mask is checked
    return build_symbols(np.ones(b.shape[0], bool), b, pool_n).s_s


# ---------------------------------------------------------------------------
# reference-signature decoders (answers come from the device decoder)
# ---------------------------------------------------------------------------
def _device_view(buf):
    if isinstance(buf, DeviceSymbols):
        return buf
    cache = getattr(buf, "_fo_device", None)
    if cache is None:
        cache = DeviceSymbols.from_buffers([buf])
        object.__setattr__(buf, "_fo_device", cache)
    return cache


def decode_spatial(buf, i, head=0):
    """Cache bit for query block i: 1 = compute, 0 = reuse (symbols.py:163-168)."""
    if not 0 <= i < buf.rows:
        raise BoundsError(f"block index {i} out of range [0, {buf.rows})")
    active, _ = _device_view(buf).decoded()
    return int(active[head, i].item())


def decode_reduction(buf, i, j, head=0):
    """Skip bit for pair (i, j): 1 = compute (symbols.py:171-180)."""
    if not 0 <= i < buf.rows:
        raise BoundsError(f"query block {i} out of range [0, {buf.rows})")
    if not 0 <= j < buf.cols:
        raise BoundsError(f"key block {j} out of range [0, {buf.cols})")
    _, pairs = _device_view(buf).decoded()
    return int(pairs[head, i, j].item())


def decode_run(buf, comp_row, head=0):
    """One compressed skip row expanded to per-block bits (symbols.py:183-198)."""
    comp_rows = ceil_div(buf.rows, buf.pool_n)
    if not 0 <= comp_row < comp_rows:
        raise BoundsError(f"compressed row {comp_row} out of range [0, {comp_rows})")
    _, pairs = _device_view(buf).decoded()
    return pairs[head, comp_row * buf.pool_n].cpu().numpy().astype(np.uint8)
