// K1: sparse-symbol pack / decode and the per-layer schedule ("plan") kernels.
//
// Packing replaces the Python per-bit loops of reference symbols.py:39-81
// (_compress_groups, _pack_row, encode_cache_mask, encode_skip_mask): one warp
// per compressed row, lanes = compressed columns, __ballot_sync + __brev gives
// the MSB-first bytes. Decoding (symbols.py:163-198) lives in fo_common.cuh and
// is shared by every kernel prologue; fo_decode_symbols_kernel exposes it so the
// decoded bits can be checked bit-for-bit against the reference.
#include "fo_internal.cuh"

// 1: GEMM-Q jobs pair heads per block (fixed pairs first, then the lone heads
// among themselves); 0: fixed head pairs (2p, 2p+1) only
#ifndef FO_GQ_REPAIR
#define FO_GQ_REPAIR 1
#endif

namespace fo {

// ---------------------------------------------------------------------------
// encode
// ---------------------------------------------------------------------------
// One warp per (head, compressed row). Row -1 encodes s_c (the cache mask).
__global__ void encode_symbols_kernel(const uint8_t* __restrict__ cache_bits,  // [H, rows]
                                      const uint8_t* __restrict__ skip_bits,   // [H, rows, cols]
                                      int H, int rows, int cols, int pool_n,
                                      uint8_t* __restrict__ s_c,  // [H, sc_len]
                                      uint8_t* __restrict__ s_s,  // [H, comp_rows, row_stride]
                                      uint32_t* status) {
  const int comp_rows = ceil_div_d(rows, pool_n), comp_cols = ceil_div_d(cols, pool_n);
  const int sc_len = ceil_div_d(comp_rows, 8), row_stride = ceil_div_d(comp_cols, 8);
  const int warps_per_head = comp_rows + 1;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= H * warps_per_head) return;
  const int h = gw / warps_per_head;
  const int r = gw % warps_per_head - 1;  // -1 -> s_c
  if (r < 0) {
    // cache mask: collapse groups along the only axis (symbols.py:39-53)
    const uint8_t* cb = cache_bits + (size_t)h * rows;
    for (int base = 0; base < comp_rows; base += 32) {
      int c = base + lane;
      uint32_t bit = 0;
      if (c < comp_rows) {
        int r0 = c * pool_n, r1 = min(r0 + pool_n, rows);
        uint32_t v0 = cb[r0] != 0;
        for (int rr = r0 + 1; rr < r1; ++rr)
          if ((cb[rr] != 0) != v0) raise_status(status, ST_CONSISTENCY);
        bit = v0;
      }
      uint32_t m = __brev(__ballot_sync(0xffffffffu, bit));
      if (lane < 4) {
        int byte = (base >> 3) + lane;
        if (byte < sc_len) s_c[(size_t)h * sc_len + byte] = (uint8_t)(m >> (24 - 8 * lane));
      }
    }
    return;
  }
  // skip mask row r: every pool_n x pool_n group must be uniform (symbols.py:73-81)
  const uint8_t* sb = skip_bits + (size_t)h * rows * cols;
  const int r0 = r * pool_n, r1 = min(r0 + pool_n, rows);
  uint8_t* out = s_s + ((size_t)h * comp_rows + r) * row_stride;
  for (int base = 0; base < comp_cols; base += 32) {
    int c = base + lane;
    uint32_t bit = 0;
    if (c < comp_cols) {
      int c0 = c * pool_n, c1 = min(c0 + pool_n, cols);
      uint32_t v0 = sb[(size_t)r0 * cols + c0] != 0;
      for (int rr = r0; rr < r1; ++rr)
        for (int cc = c0; cc < c1; ++cc)
          if ((sb[(size_t)rr * cols + cc] != 0) != v0) raise_status(status, ST_CONSISTENCY);
      bit = v0;
    }
    uint32_t m = __brev(__ballot_sync(0xffffffffu, bit));
    if (lane < 4) {
      int byte = (base >> 3) + lane;
      if (byte < row_stride) out[byte] = (uint8_t)(m >> (24 - 8 * lane));
    }
  }
}

// ---------------------------------------------------------------------------
// decode (exposes the kernels' prologue decoders for bit-exact checks)
// ---------------------------------------------------------------------------
__global__ void decode_symbols_kernel(const uint8_t* __restrict__ s_c, const uint8_t* __restrict__ s_s,
                                      int H, int rows, int cols, int pool_n,
                                      uint8_t* __restrict__ active,      // [H, rows]
                                      uint8_t* __restrict__ pair_bits) {  // [H, rows, cols]
  const int comp_rows = ceil_div_d(rows, pool_n), comp_cols = ceil_div_d(cols, pool_n);
  const int sc_len = ceil_div_d(comp_rows, 8), row_stride = ceil_div_d(comp_cols, 8);
  const size_t total = (size_t)H * rows * cols;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    int j = (int)(idx % cols);
    int i = (int)((idx / cols) % rows);
    int h = (int)(idx / ((size_t)cols * rows));
    pair_bits[idx] = (uint8_t)decode_reduction(s_s + (size_t)h * comp_rows * row_stride, row_stride,
                                               i, j, pool_n);
    if (j == 0) active[(size_t)h * rows + i] = (uint8_t)decode_spatial(s_c + (size_t)h * sc_len, i, pool_n);
  }
}

// ---------------------------------------------------------------------------
// plan: one CTA turns the symbols of a layer into the schedules the hot-path
// kernels consume. Everything here is integer work on a few KB.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024, 1)
plan_kernel(const uint8_t* __restrict__ s_c, const uint8_t* __restrict__ s_s, int H, int rows,
            int cols, int pool_n, int dense, const int32_t* __restrict__ valid, int order_d,
            int ctas, int pair_items, PlanView pv, uint32_t* status) {
  // Attention items are ordered head-major, longest rows first within a head:
  // CTAs stride through the list together, so the K/V of the ~1-2 heads in
  // flight stay L2-resident while per-CTA work stays balanced.
  extern __shared__ int plan_smem[];
  const int nseg = (H * (cols + 2) + 3072) * (int)sizeof(int) <= 160 * 1024 ? H : 1;
  int* hist = plan_smem;                   // [nseg][cols + 2] -> exclusive offsets
  int* scan = hist + nseg * (cols + 2);    // [1024]
  __shared__ unsigned int s_pairs[64];  // per-head pairs <= 2048 x 2048: 32-bit (native shared atomics)
  const int comp_rows = ceil_div_d(rows, pool_n), comp_cols = ceil_div_d(cols, pool_n);
  const int sc_len = ceil_div_d(comp_rows, 8), row_stride = ceil_div_d(comp_cols, 8);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int total = H * rows;
  auto seg = [&](int h) { return nseg == 1 ? 0 : h; };
  // CTA-pair attention (pool_n even, sparse): query blocks 2c and 2c+1 share one
  // compressed skip row, so one item (h, 2c) covers both (one per CTA of a
  // cluster, K/V multicast); the schedule then has `ctas` = clusters slots
  const bool pair = pair_items != 0;
  auto scheduled = [&](int i) { return !pair || (i & 1) == 0; };

  for (int c = tid; c < nseg * (cols + 2); c += nt) hist[c] = 0;
  for (int h = tid; h < 64; h += nt) s_pairs[h] = 0;
  __syncthreads();

  auto is_active = [&](int h, int i) -> int {
    return dense ? 1 : (int)decode_spatial(s_c + (size_t)h * sc_len, i, pool_n);
  };

  // pass 1: histogram of per-row KV counts, head masks, checks
  for (int i = tid; i < rows; i += nt) {
    unsigned long long m = 0;
    int min_valid = 1 << 30;
    bool any_cached = false;
    for (int h = 0; h < H; ++h) {
      int a = is_active(h, i);
      if (a) {
        m |= 1ull << h;
      } else {
        any_cached = true;
        if (valid) min_valid = min(min_valid, valid[(size_t)h * rows + i]);
      }
    }
    pv.hmask[i] = m;
    // n_orders for the GEMM-O cached bias of block i (gemm.py:140-153)
    int no = 0;
    if (any_cached) {
      no = valid ? min(order_d + 1, min_valid) : order_d + 1;
      if (no < 1) raise_status(status, ST_STATE);
    }
    pv.orders[i] = no;
  }
  // per-(head, block) KV counts, computed once and kept in the plan scratch for
  // pass 2. The row's bytes are loaded 8 at a time before use, so a
  // row costs a few load latencies instead of one per byte.
  int* kvc = pv.scratch;
  for (int idx = tid; idx < total; idx += nt) {
    const int h = idx / rows, i = idx % rows;
    int c = -1;
    if (dense) {
      c = cols;
    } else if (is_active(h, i)) {
      const uint8_t* row = s_s + ((size_t)h * comp_rows + i / pool_n) * row_stride;
      c = 0;
      for (int b0 = 0; b0 < row_stride; b0 += 8) {
        uint32_t by[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) by[k] = (b0 + k < row_stride) ? row[b0 + k] : 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int b = b0 + k;
          if (b >= row_stride) break;
          uint32_t byte = by[k];
          const int nvalid = min(8, comp_cols - b * 8);
          byte &= (0xFFu << (8 - nvalid)) & 0xFFu;  // padding bits (decode_run truncates)
          if (pool_n == 1) {
            c += __popc(byte);
          } else {
            while (byte) {
              const int kk = __clz(byte) - 24;  // MSB-first bit index
              byte &= ~(0x80u >> kk);
              c += min(pool_n, cols - (b * 8 + kk) * pool_n);
            }
          }
        }
      }
    }
    kvc[idx] = c;
  }
  __syncthreads();
  for (int idx = tid; idx < total; idx += nt) {
    int h = idx / rows, i = idx % rows;
    if (is_active(h, i)) {
      int cnt = kvc[idx];
      if (cnt == 0) {
        // active query block with every key block skipped (pyref.py:43-46)
        raise_status(status, ST_CONSISTENCY);
      } else {
        if (scheduled(i)) atomicAdd(&hist[seg(h) * (cols + 2) + cnt], 1);
        atomicAdd(&s_pairs[h], (unsigned int)cnt);
      }
    } else if (valid && valid[(size_t)h * rows + i] < 1) {
      // cached tile with a cold cache (attention.py:208-211)
      raise_status(status, ST_STATE);
    }
  }
  __syncthreads();
  // exclusive scan: segment-major, descending KV count within a segment. One
  // warp per segment scans it in 32-wide chunks (shuffle scan), then the
  // segment totals are scanned and added back (a single-thread walk over
  // H*(cols+1) counters took ~100 us at C4).
  {
    const int wid = tid >> 5, ln = tid & 31, nw = nt >> 5;
    int* seg_tot = scan;  // [nseg] (scan[] is free until pass 3)
    for (int g = wid; g < nseg; g += nw) {
      int run = 0;
      for (int c0 = cols; c0 >= 1; c0 -= 32) {
        const int c = c0 - ln;
        const int v = c >= 1 ? hist[g * (cols + 2) + c] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (ln >= o) x += y;
        }
        if (c >= 1) hist[g * (cols + 2) + c] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (ln == 0) seg_tot[g] = run;
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int g = 0; g < nseg; ++g) {
        const int n = seg_tot[g];
        seg_tot[g] = run;
        run += n;
      }
      pv.counts[0] = run;  // attention items
    }
    __syncthreads();
    for (int e = tid; e < nseg * (cols + 2); e += nt) {
      const int g = e / (cols + 2), c = e - g * (cols + 2);
      if (c >= 1 && c <= cols) hist[e] += seg_tot[g];
    }
  }
  for (int h = tid; h < H; h += nt) pv.pairs_pred[h] = (long long)s_pairs[h];
  __syncthreads();
  // pass 2: scatter attention items (sorted by KV count, descending)
  for (int idx = tid; idx < total; idx += nt) {
    const int cnt = kvc[idx];  // -1 cached, 0 empty (flagged above)
    if (cnt > 0 && scheduled(idx % rows)) {
      const int h = idx / rows, i = idx % rows;
      int pos = atomicAdd(&hist[seg(h) * (cols + 2) + cnt], 1);
      pv.items[pos] = make_int2((h << 20) | i, cnt);
    }
  }
  // pass 2b: balanced attention schedule. The item list is cut into waves of
  // `ctas` consecutive items (head-major order keeps the K/V of the heads in
  // flight L2-resident); within a wave the longest item goes to the CTA with
  // the least work so far (LPT per wave). Static round-robin leaves a 3-5%
  // spread of per-CTA work at C4 (simulated), this ~1-3%, and with the
  // virtual head start below ~0.4%.
  __syncthreads();
  {
    const int n_items = pv.counts[0];
    const int P = ctas;  // <= 256 (checked by fo_plan): 4 threads per bin
    int* bin_load = scan;           // [P] tiles assigned so far (scan[] is free until pass 3)
    int* bin_of_rank = plan_smem + nseg * (cols + 2) + 1024;  // [P] (see the smem size in fo_plan)
    int* wave_len = bin_of_rank + 1024;                         // [P] item lengths of the wave
    // n_items % P CTAs get one item more than the rest. They start with a
    // virtual item of average length (removed before the last wave), so every
    // wave's LPT hands them shorter items and the extra item does not become
    // the makespan (C4 bench symbols, simulated: 2.9% -> 0.4% over the mean).
    const int r_last = n_items % P;
    __shared__ int s_tiles;
    if (tid == 0) s_tiles = 0;
    __syncthreads();
    if (r_last) {
      int loc = 0;
      for (int e = tid; e < n_items; e += nt) loc += pv.items[e].y;
      atomicAdd(&s_tiles, loc);
    }
    __syncthreads();
    const int head_start = r_last ? (s_tiles + n_items / 2) / n_items : 0;
    for (int b = tid; b < P; b += nt) bin_load[b] = b < r_last ? head_start : 0;
    __syncthreads();
    const int n_waves = ceil_div_d(n_items, P);
    if (tid < min(P, n_items)) wave_len[tid] = pv.items[tid].y;
    __syncthreads();
    for (int k = 0; k < n_waves; ++k) {
      if (r_last && k == n_waves - 1) {
        if (tid < r_last) bin_load[tid] -= head_start;
        __syncthreads();
      }
      const int base = k * P, m = min(P, n_items - base);
      // the next wave's lengths are loaded while this one is ranked
      const int nbase = base + P;
      const int next_len = (tid < min(P, n_items - nbase)) ? pv.items[nbase + tid].y : 0;
      // ranks are counted by 4 threads per element (quarter ranges, shuffle sum)
      const int e = tid >> 2, qq = tid & 3, span = (P + 3) >> 2;
      const int lo4 = qq * span, hi4 = min(P, lo4 + span);
      int my_rank = 0;
      if (e < P) {  // rank of bin e by (load, index)
        const int my_load = bin_load[e];
#pragma unroll 8
        for (int b = lo4; b < hi4; ++b) {
          const int l = bin_load[b];
          my_rank += (l < my_load) || (l == my_load && b < e);
        }
      }
      my_rank += __shfl_xor_sync(0xffffffffu, my_rank, 1);
      my_rank += __shfl_xor_sync(0xffffffffu, my_rank, 2);
      __syncthreads();
      if (e < P && qq == 0) bin_of_rank[my_rank] = e;
      __syncthreads();
      int r = 0;
      if (e < m) {  // rank of item e by (length desc, index)
        const int len = wave_len[e];
        const int hi_u = min(m, hi4);
#pragma unroll 8
        for (int u = lo4; u < hi_u; ++u) {
          const int lu = wave_len[u];
          r += (lu > len) || (lu == len && u < e);
        }
      }
      r += __shfl_xor_sync(0xffffffffu, r, 1);
      r += __shfl_xor_sync(0xffffffffu, r, 2);
      if (qq == 0) {
        if (e < m) {
          const int b = bin_of_rank[r];
          pv.att_sched[base + b] = base + e;
          bin_load[b] += wave_len[e];
        } else if (e < P) {
          // bins ranked past the wave's items get nothing this wave (last wave only)
          pv.att_sched[base + bin_of_rank[e]] = -1;
        }
      }
      __syncthreads();
      if (tid < min(P, n_items - nbase)) wave_len[tid] = next_len;
      __syncthreads();
    }
    if (tid == 0) {
      pv.counts[6] = n_waves;
      pv.counts[4] = pair ? 1 : 0;  // attention items cover CTA pairs (2c, 2c+1)
      pv.counts[5] = P;             // schedule slots per wave
    }
  }
  __syncthreads();
  // pass 3: GEMM-Q tile list in (block, head) order: compaction via block scan
  const int per = ceil_div_d(total, nt);
  const int lo = min(total, tid * per), hi = min(total, lo + per);
  int local = 0;
  for (int idx = lo; idx < hi; ++idx) {
    int i = idx / H, h = idx % H;
    local += is_active(h, i);
  }
  scan[tid] = local;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {
    int v = tid >= off ? scan[tid - off] : 0;
    __syncthreads();
    scan[tid] += v;
    __syncthreads();
  }
  const int n_active = scan[nt - 1];
  int pos = scan[tid] - local;
  int pos_c = n_active + (lo - pos);  // cached tiles follow the active ones, same order
  for (int idx = lo; idx < hi; ++idx) {
    int i = idx / H, h = idx % H;
    if (is_active(h, i))
      pv.gq_items[pos++] = (h << 20) | i;
    else
      pv.gq_items[pos_c++] = (h << 20) | i;
  }
  if (tid == nt - 1) {
    pv.counts[1] = n_active;
    pv.counts[2] = 0;  // fused-forecast cursor and CTA count (attention, materialize mode)
    pv.counts[3] = 0;
  }
  // pass 4: GEMM-Q jobs, all for the CTA-pair kernel (one launch). Every active
  // tile is in exactly one job and no cached tile is computed. By default
  // (FO_GQ_REPAIR) head pairs are chosen per block, below; the fallback uses
  // the fixed pairs p = (2p, 2p+1) (the last head alone when H is odd): the
  // blocks where both heads are active form N=256 jobs and the blocks where
  // only one is active N=128 jobs of that head; each of the three lists is cut
  // into jobs of two blocks (one per CTA; the last may hold one). Jobs are then
  // ordered by cost class and first block (counting sort), so the jobs in
  // flight share x tiles in L2.
  __syncthreads();  // pass 3 read scan[]; hmask (pass 1) is visible block-wide
  const int avail = nseg * (cols + 2) + 3072;  // ints of plan_smem free after pass 2
  const int W = (rows + 31) >> 5;                // 32-block words of a block bitmask
  const int ntypes = H * (H - 1) / 2;            // unordered head pairs (h1 < h2)
  int2* tmp = pv.gq_jobs + gq_jobs_cap(H, rows);  // unsorted jobs
  if (H >= 2 && (ntypes + H) * W + ntypes + H <= avail && FO_GQ_REPAIR) {
    // Head pairs chosen per block (FO_GQ_REPAIR). The fixed pairs (2p, 2p+1)
    // active together are kept; the heads whose partner is cached are paired
    // among themselves in head order, so a block with, say, heads 3 and 6
    // alone still yields an N = 256 tile. Blocks sharing a head pair are then
    // cut into two-block jobs (in block order); a pair type with an odd block
    // count hands its last block's two heads to the per-head single lists,
    // which are cut into N = 128 jobs (the last may hold one block). At random
    // 25 / 50 / 75 / 90% cached maps over 258 blocks this puts 93 / 89 / 78 /
    // 42% of the active tiles in N = 256 jobs (fixed pairs: 74 / 48 / 23 / 7%).
    unsigned* tmask = reinterpret_cast<unsigned*>(plan_smem);  // [ntypes][W] blocks per pair type
    unsigned* smask = tmask + ntypes * W;                       // [H][W] single-head blocks
    int* tcnt = reinterpret_cast<int*>(smask + H * W);          // [ntypes] jobs -> offsets
    int* hcnt = tcnt + ntypes;                                  // [H] jobs -> offsets
    auto tri = [&](int a, int b) { return a * (2 * H - a - 1) / 2 + (b - a - 1); };
    auto untri = [&](int t, int& a, int& b) {
      a = 0;
      while (t >= H - 1 - a) {
        t -= H - 1 - a;
        ++a;
      }
      b = a + 1 + t;
    };
    for (int e = tid; e < (ntypes + H) * W; e += nt) tmask[e] = 0u;
    __syncthreads();
    for (int i = tid; i < rows; i += nt) {
      const unsigned long long m = pv.hmask[i];
      const unsigned bit = 1u << (i & 31);
      const int w = i >> 5;
      int pend = -1;  // a head whose fixed partner is cached, waiting for a partner
      for (int a = 0; a < H; a += 2) {
        const bool xa = (m >> a) & 1ull, xb = a + 1 < H && ((m >> (a + 1)) & 1ull);
        if (xa && xb) {
          atomicOr(&tmask[tri(a, a + 1) * W + w], bit);
          continue;
        }
        const int lone = xa ? a : (xb ? a + 1 : -1);
        if (lone < 0) continue;
        if (pend < 0) {
          pend = lone;
        } else {
          atomicOr(&tmask[tri(pend, lone) * W + w], bit);
          pend = -1;
        }
      }
      if (pend >= 0) atomicOr(&smask[pend * W + w], bit);
    }
    __syncthreads();
    for (int t = tid; t < ntypes; t += nt) {
      int c = 0, last = -1;
      for (int w = 0; w < W; ++w) {
        const unsigned v = tmask[t * W + w];
        if (v) {
          c += __popc(v);
          last = w * 32 + 31 - __clz(v);
        }
      }
      if (c & 1) {  // the last block's two heads become single-head entries
        int a, b;
        untri(t, a, b);
        const unsigned bit = 1u << (last & 31);
        tmask[t * W + (last >> 5)] &= ~bit;
        atomicOr(&smask[a * W + (last >> 5)], bit);
        atomicOr(&smask[b * W + (last >> 5)], bit);
        --c;
      }
      tcnt[t] = c >> 1;
    }
    __syncthreads();
    for (int h = tid; h < H; h += nt) {
      int c = 0;
      for (int w = 0; w < W; ++w) c += __popc(smask[h * W + w]);
      hcnt[h] = (c + 1) >> 1;
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int t = 0; t < ntypes + H; ++t) {  // tcnt and hcnt are contiguous
        const int c = tcnt[t];
        tcnt[t] = run;
        run += c;
      }
      pv.counts[7] = run;
    }
    __syncthreads();
    for (int t = tid; t < ntypes + H; t += nt) {
      int pos = tcnt[t];
      const bool pair_t = t < ntypes;
      const unsigned* mk = pair_t ? tmask + t * W : smask + (t - ntypes) * W;
      int a = t - ntypes, b = -1;
      if (pair_t) untri(t, a, b);
      const int y = pair_t ? (a | (1 << 8) | (b << 16)) : a;
      int i0 = -1;
      for (int w = 0; w < W; ++w) {
        unsigned v = mk[w];
        while (v) {
          const int i = w * 32 + __ffs(v) - 1;
          v &= v - 1;
          if (i0 < 0) {
            i0 = i;
          } else {
            tmp[pos++] = make_int2(i0 | ((i + 1) << 16), y);
            i0 = -1;
          }
        }
      }
      if (i0 >= 0) tmp[pos++] = make_int2(i0, y);  // single-head lists only (pair types are even)
    }
    __syncthreads();
  } else {
    const int npair = (H + 1) >> 1;
    int* pcount = scan;  // [npair] jobs per pair, then their offsets
    auto kind_of = [&](int p, int i) -> int {  // 0: both, 1: first only, 2: second only, -1
      const int h1 = 2 * p;
      const unsigned m = (unsigned)(pv.hmask[i] >> h1) & (h1 + 1 < H ? 3u : 1u);
      return m == 3u ? 0 : m == 1u ? 1 : m == 2u ? 2 : -1;
    };
    if (tid < npair) {
      int n[3] = {0, 0, 0};
      for (int i = 0; i < rows; ++i) {
        const int k = kind_of(tid, i);
        if (k >= 0) ++n[k];
      }
      pcount[tid] = (n[0] + 1) / 2 + (n[1] + 1) / 2 + (n[2] + 1) / 2;
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int q = 0; q < npair; ++q) {
        const int c = pcount[q];
        pcount[q] = run;
        run += c;
      }
      pv.counts[7] = run;
    }
    __syncthreads();
    if (tid < npair) {
      const int h1 = 2 * tid;
      int pos = pcount[tid];
      int pending[3] = {-1, -1, -1};
      auto emit = [&](int i0, int i1, int k) {
        const int y = k == 0 ? (h1 | (1 << 8) | ((h1 + 1) << 16)) : (k == 1 ? h1 : h1 + 1);
        tmp[pos++] = make_int2(i0 | ((i1 + 1) << 16), y);
      };
      for (int i = 0; i < rows; ++i) {
        const int k = kind_of(tid, i);
        if (k < 0) continue;
        if (pending[k] < 0) {
          pending[k] = i;
        } else {
          emit(pending[k], i, k);
          pending[k] = -1;
        }
      }
      for (int k = 0; k < 3; ++k)
        if (pending[k] >= 0) emit(pending[k], -1, k);
    }
    __syncthreads();
  }
  {
    const int n2 = pv.counts[7];
    // counting sort by (cost class, first block): N = 256 two-block jobs, then
    // N = 128 two-block jobs, then single-block jobs, each by first block (jobs
    // in flight share x tiles in L2; the kernel deals the classes out snaking)
    const int ncls = 3 * rows <= avail ? 3 : 1;
    auto key = [&](int2 code) {
      const int i0 = code.x & 0xFFFF;
      if (ncls == 1) return i0;
      const int cls = (code.x >> 16) == 0 ? 2 : (((code.y >> 8) & 1) ? 0 : 1);
      return cls * rows + i0;
    };
    int* bcnt = plan_smem;  // [ncls * rows] (free after pass 2)
    for (int i = tid; i < ncls * rows; i += nt) bcnt[i] = 0;
    __syncthreads();
    for (int e = tid; e < n2; e += nt) atomicAdd(&bcnt[key(tmp[e])], 1);
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int i = 0; i < ncls * rows; ++i) {
        const int c = bcnt[i];
        bcnt[i] = run;
        run += c;
      }
    }
    __syncthreads();
    for (int e = tid; e < n2; e += nt) {
      const int2 code = tmp[e];
      pv.gq_jobs[atomicAdd(&bcnt[key(code)], 1)] = code;
    }
  }
}

// ---------------------------------------------------------------------------
// stale-symbol check for GEMM-O dispatch (gemm.py:201-209): decoded active
// heads of the dispatch symbols must equal those the bias was built under.
// ---------------------------------------------------------------------------
__global__ void compare_active_kernel(const uint8_t* __restrict__ s_c_a, const uint8_t* __restrict__ s_c_b,
                                      int H, int rows, int pool_n, uint32_t* status) {
  const int sc_len = ceil_div_d(ceil_div_d(rows, pool_n), 8);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < H * rows; idx += gridDim.x * blockDim.x) {
    int h = idx / rows, i = idx % rows;
    if (decode_spatial(s_c_a + (size_t)h * sc_len, i, pool_n) !=
        decode_spatial(s_c_b + (size_t)h * sc_len, i, pool_n))
      raise_status(status, ST_STATE);
  }
}

}  // namespace fo
