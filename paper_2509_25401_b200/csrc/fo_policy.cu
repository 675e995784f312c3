// Update-step mask policy on the GPU (reference policy.py:44-234).
//
// Turns fresh q/k into the next window's cache and skip masks without a host
// round trip. The reference computes in float32 / float64 numpy; to reproduce
// its decisions bit for bit the kernels follow numpy's reduction orders:
//   mean_pool_blocks   fp64 sequential block sums / lengths -> fp32 (tensor.py:112-126)
//   scores             fp64 dot products / sqrt(d) -> fp32 (policy.py:44-55)
//   row_softmax        fp64 exp, numpy pairwise row sum, / sum -> fp32 (tensor.py:42-47)
//   contribution       fp32 sequential column sums over text rows (policy.py:58-65)
//   guidance           row_softmax of the transposed vision x text block, fp32
//                      sequential column sums (policy.py:68-77)
//   prefix selection   stable ascending order (ties -> lower index), fp64
//                      sequential cumsum, csum <= budget (* total) (policy.py:80-121)
// Four small launches: pool (q and k, thread per (head, block, dim pair)),
// scores (CTA per (head, 16 compressed rows)), cache selection (CTA per head),
// skip selection (warp per (head, compressed row)). The compressed map of a
// 33K-token layer is 258 x 258 per head.
#include "fo_internal.cuh"

namespace fo {

namespace {

constexpr int kPolWarps = 4;  // warps per CTA in the per-row kernels

// thread per (tensor, block, head, dim pair): q and k in one launch, bf16x2
// loads (a warp reads 128 contiguous bytes of a row), fp64 sums in row order.
__global__ void pool_kernel(const __nv_bfloat16* __restrict__ xq, const __nv_bfloat16* __restrict__ xk,
                            int S, int H, int block, int rows_c, float* __restrict__ oq,
                            float* __restrict__ ok) {  // [H, rows_c, 128] each
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= H * rows_c * (kTile / 2)) return;
  const __nv_bfloat16* x = blockIdx.y ? xk : xq;
  float* out = blockIdx.y ? ok : oq;
  // heads vary fastest after the dims: consecutive warps read one token row
  const int d = 2 * (idx % (kTile / 2)), h = (idx / (kTile / 2)) % H,
            r = idx / ((kTile / 2) * H);
  const int s0 = r * block, s1 = min(S, s0 + block);
  const uint32_t* p =
      reinterpret_cast<const uint32_t*>(x + (size_t)s0 * H * kTile + (size_t)h * kTile + d);
  const size_t stride = (size_t)H * kTile / 2;
  double a0 = 0.0, a1 = 0.0;  // np.add.reduceat: sequential from the first element
#pragma unroll 8
  for (int s = s0; s < s1; ++s, p += stride) {
    const uint32_t v = __ldg(p);
    a0 += (double)__uint_as_float(v << 16);
    a1 += (double)__uint_as_float(v & 0xFFFF0000u);
  }
  const double n = (double)(s1 - s0);
  *reinterpret_cast<float2*>(out + (size_t)(h * rows_c + r) * kTile + d) =
      make_float2((float)(a0 / n), (float)(a1 / n));
}

__device__ double pairwise_leaf(const double* p, int n) {
  if (n < 8) {
    double res = 0.;
    for (int i = 0; i < n; ++i) res += p[i];
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = p[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += p[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += p[i];
  return res;
}

// numpy's pairwise_sum (umath loops_utils.h): blocks of <= 128 with eight
// accumulators, larger runs split at n/2 rounded down to a multiple of 8.
template <int DEPTH>
__device__ double pairwise_sum(const double* a, int n) {
  if (n <= 128) return pairwise_leaf(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum<DEPTH - 1>(a, n2) + pairwise_sum<DEPTH - 1>(a + n2, n - n2);
}
template <>
__device__ double pairwise_sum<0>(const double* a, int n) {
  return pairwise_leaf(a, n);  // unreachable for n <= kPolicyMaxBlocks
}

// Scores + row softmax. CTA per (head, 16 compressed rows), 4 warps of 4
// rows. The head's pooled k is staged through shared memory as fp64,
// transposed ([d][column], 64 columns per chunk) so a lane's column reads are
// conflict-free and every element is converted once; each lane keeps 4 rows x
// 2 columns of fp64 accumulators, summed over d in order (the same arithmetic
// as a per-column loop). The softmax exponentials run across the warp; lane 0
// does numpy's pairwise sum.
constexpr int kScWarps = 4, kScRows = 4, kScChunk = 64;

size_t scores_smem_bytes(int cols) {
  return (size_t)kTile * kScChunk * 8 + (size_t)kScWarps * kScRows * kTile * 8 +
         (size_t)kScWarps * cols * 8 + (size_t)kScWarps * kScRows * cols * 4;
}

__global__ void __launch_bounds__(kScWarps * 32, 2)
scores_kernel(const float* __restrict__ pq, const float* __restrict__ pk, int rows_c,
              float* __restrict__ p_tilde) {
  extern __shared__ __align__(16) unsigned char sc_smem[];
  const int cols = rows_c;
  double* pkT = reinterpret_cast<double*>(sc_smem);                 // [128][kScChunk]
  double* qs = pkT + kTile * kScChunk;                              // [warp][row][128]
  double* e = qs + kScWarps * kScRows * kTile;                      // [warp][cols]
  float* srow = reinterpret_cast<float*>(e + kScWarps * cols);      // [warp][row][cols]
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31, h = blockIdx.y;
  const int r0 = (blockIdx.x * kScWarps + wib) * kScRows;
  double* qw = qs + wib * kScRows * kTile;
  float* sw = srow + (size_t)wib * kScRows * cols;
  double* ew = e + (size_t)wib * cols;
  {
    float qv[kScRows][kTile / 32];  // loads first: one L2 round trip, not sixteen
#pragma unroll
    for (int i = 0; i < kScRows; ++i)
#pragma unroll
      for (int u = 0; u < kTile / 32; ++u)
        qv[i][u] = r0 + i < rows_c ? __ldg(&pq[((size_t)h * rows_c + r0 + i) * kTile + lane + 32 * u]) : 0.f;
#pragma unroll
    for (int i = 0; i < kScRows; ++i)
#pragma unroll
      for (int u = 0; u < kTile / 32; ++u) qw[i * kTile + lane + 32 * u] = (double)qv[i][u];
  }
  const double rs = sqrt((double)kTile);
  const float4* pk4 = reinterpret_cast<const float4*>(pk + (size_t)h * cols * kTile);
  const int nchunk = (cols + kScChunk - 1) / kScChunk;
  const int csz = ((cols + nchunk - 1) / nchunk + 31) & ~31;  // balanced, multiple of 32
  const int jn = csz >> 5;
  // the next chunk's loads are in flight while this chunk computes
  constexpr int kLd = kScChunk * (kTile / 4) / (kScWarps * 32);
  float4 v[kLd];
  auto load_chunk = [&](int c0) {
    const int cn = min(csz, cols - c0);
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int idx = threadIdx.x + u * kScWarps * 32, c = idx % kScChunk, d4 = idx / kScChunk;
      v[u] = c < cn ? __ldg(&pk4[(size_t)(c0 + c) * (kTile / 4) + d4]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  load_chunk(0);
  for (int c0 = 0; c0 < cols; c0 += csz) {
    const int cn = min(csz, cols - c0);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int idx = threadIdx.x + u * kScWarps * 32, c = idx % kScChunk, d4 = idx / kScChunk;
      pkT[(4 * d4 + 0) * kScChunk + c] = (double)v[u].x;
      pkT[(4 * d4 + 1) * kScChunk + c] = (double)v[u].y;
      pkT[(4 * d4 + 2) * kScChunk + c] = (double)v[u].z;
      pkT[(4 * d4 + 3) * kScChunk + c] = (double)v[u].w;
    }
    if (c0 + csz < cols) load_chunk(c0 + csz);
    __syncthreads();
    if (r0 >= rows_c) continue;
    double acc[kScRows][2] = {};
#pragma unroll 2
    for (int d = 0; d < kTile; ++d) {
      const double k0 = pkT[d * kScChunk + lane];
      const double k1 = jn > 1 ? pkT[d * kScChunk + lane + 32] : 0.0;
#pragma unroll
      for (int i = 0; i < kScRows; ++i) {
        const double qd = qw[i * kTile + d];
        acc[i][0] += qd * k0;
        acc[i][1] += qd * k1;
      }
    }
#pragma unroll
    for (int i = 0; i < kScRows; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = lane + 32 * j;
        if (r0 + i < rows_c && c < cn) sw[i * cols + c0 + c] = (float)(acc[i][j] / rs);
      }
  }
  __syncwarp();
  for (int i = 0; i < kScRows; ++i) {
    if (r0 + i >= rows_c) break;
    const float* s = sw + i * cols;
    float mx = -INFINITY;  // max is order independent for finite scores
    for (int c = lane; c < cols; c += 32) mx = fmaxf(mx, s[c]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int c = lane; c < cols; c += 32) ew[c] = exp((double)s[c] - (double)mx);
    __syncwarp();
    double sum = 0.0;
    if (lane == 0) sum = pairwise_sum<5>(ew, cols);
    sum = __shfl_sync(0xffffffffu, sum, 0);
    float* out = p_tilde + ((size_t)h * rows_c + r0 + i) * cols;
    for (int c = lane; c < cols; c += 32) out[c] = (float)(ew[c] / sum);
    __syncwarp();
  }
}

// Stable ascending budget prefix over v[0, n) (fp64 copies of fp32 values).
// Ranks by (value, index) in parallel; one lane scans the fp64 cumsum in rank
// order. Returns cut: elements with rank < cut are taken.
template <bool CTA>
__device__ int budget_prefix(const double* v, float* vf, int n, double budget, bool relative,
                             int* rank, double* sorted, int tid, int nt) {
  // ranks compare fp32 copies (v holds fp32 values, so the order is the same)
  // with up to eight elements per thread in registers against one broadcast read
  for (int i = tid; i < n; i += nt) vf[i] = (float)v[i];
  if (CTA) __syncthreads(); else __syncwarp();
  constexpr int kU = CTA ? 1 : 8;  // elements per thread (a CTA has 256 threads for <= 1024)
  for (int i0 = tid; i0 < n; i0 += kU * nt) {
    float vi[kU];
    int rk[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * nt;
      vi[u] = i < n ? vf[i] : INFINITY;
      rk[u] = 0;
    }
    for (int j = 0; j < n; ++j) {
      const float vj = vf[j];
#pragma unroll
      for (int u = 0; u < kU; ++u) rk[u] += (vj < vi[u]) | ((vj == vi[u]) & (j < i0 + u * nt));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * nt;
      if (i < n) {
        rank[i] = rk[u];
        sorted[rk[u]] = v[i];
      }
    }
  }
  if (CTA) __syncthreads(); else __syncwarp();
  int cut = 0;
  if (tid == 0) {
    // the relative total is csum[-1] of the same sequential cumsum
    double lim = budget;
    if (relative) {
      double t = 0.0;
      for (int k = 0; k < n; ++k) t += sorted[k];
      lim = budget * t;
    }
    double c = 0.0;
    for (; cut < n; ++cut) {
      c += sorted[cut];
      if (!(c <= lim)) break;
    }
  }
  if (CTA) {
    __shared__ int s_cut;
    if (tid == 0) s_cut = cut;
    __syncthreads();
    cut = s_cut;
    __syncthreads();
  } else {
    cut = __shfl_sync(0xffffffffu, cut, 0);
  }
  return cut;
}

// CTA per head: contribution / guidance -> compressed compute bits + degrade.
__global__ void __launch_bounds__(256)
cache_select_kernel(const float* __restrict__ p_tilde, int rows_c, int n_t, double tau_q,
                    double s_q, uint8_t* __restrict__ comp_cache) {  // [H, rows_c]
  extern __shared__ double cs_smem[];
  const int h = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int cols = rows_c, V = rows_c - n_t;
  const float* P = p_tilde + (size_t)h * rows_c * cols;
  double* contrib = cs_smem;                                   // [V]
  double* guid = contrib + rows_c;                             // [V]
  double* sorted = guid + rows_c;                              // [V]
  int* rank = reinterpret_cast<int*>(sorted + rows_c);         // [V]
  uint8_t* cut_c = reinterpret_cast<uint8_t*>(rank + rows_c);  // [V]
  uint8_t* cc = cut_c + rows_c;                                // [rows_c]
  double* e = reinterpret_cast<double*>(                        // [V] guidance scratch
      (reinterpret_cast<uintptr_t>(cc + rows_c) + 7) & ~uintptr_t(7));
  float* tmp = reinterpret_cast<float*>(e + rows_c);           // [V]
  float* acc = tmp + rows_c;                                   // [V]
  float* vf = acc + rows_c;                                    // [V] rank keys
  // vision_to_text_contribution: p[:n_t, n_t:].sum(axis=0), fp32 row by row
  for (int c = tid; c < V; c += nt) {
    float a = 0.f;
    for (int r = 0; r < n_t; ++r) {
      const float x = P[(size_t)r * cols + n_t + c];
      a = r ? a + x : x;
    }
    contrib[c] = (double)a;
  }
  // text_to_vision_guidance: text column j re-softmaxed over the vision rows,
  // then fp32 sums over j in order (exponentials across the CTA, numpy's
  // pairwise sum on one thread)
  __shared__ float red[32];
  __shared__ double s_sum;
  for (int j = 0; j < n_t; ++j) {
    float mx = -INFINITY;
    for (int c = tid; c < V; c += nt) {
      tmp[c] = P[(size_t)(n_t + c) * cols + j];
      mx = fmaxf(mx, tmp[c]);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < nt / 32; ++w) mx = fmaxf(mx, red[w]);
    for (int c = tid; c < V; c += nt) e[c] = exp((double)tmp[c] - (double)mx);
    __syncthreads();
    if (tid == 0) s_sum = pairwise_sum<5>(e, V);
    __syncthreads();
    const double sum = s_sum;
    for (int c = tid; c < V; c += nt) {
      const float beta = (float)(e[c] / sum);
      acc[c] = j ? acc[c] + beta : beta;
    }
    __syncthreads();
  }
  for (int c = tid; c < V; c += nt) guid[c] = n_t > 0 ? (double)acc[c] : 0.0;
  __syncthreads();
  // select_cached_blocks: both ascending prefixes within tau_q of their totals
  int cut = budget_prefix<true>(contrib, vf, V, tau_q, true, rank, sorted, tid, nt);
  for (int i = tid; i < V; i += nt) cut_c[i] = rank[i] < cut;
  __syncthreads();
  cut = budget_prefix<true>(guid, vf, V, tau_q, true, rank, sorted, tid, nt);
  for (int r = tid; r < rows_c; r += nt)
    cc[r] = (r < n_t) ? 1 : !(cut_c[r - n_t] && rank[r - n_t] < cut);
  __syncthreads();
  // degrade_to_full_cache: computed vision fraction below s_q -> cache all vision
  __shared__ int n_comp;
  if (tid == 0) {
    int c = 0;
    for (int r = n_t; r < rows_c; ++r) c += cc[r];
    n_comp = c;
  }
  __syncthreads();
  const bool degrade = V > 0 && (double)n_comp / (double)V < s_q;
  for (int r = tid; r < rows_c; r += nt)
    comp_cache[(size_t)h * rows_c + r] = (degrade && r >= n_t) ? 0 : cc[r];
}

// warp per (head, compressed row): select_skip_blocks for computed rows, then
// expand_blocks into block-granularity bits (policy.py:124-159, 190-193).
__global__ void skip_select_kernel(const float* __restrict__ p_tilde,
                                   const uint8_t* __restrict__ comp_cache, int H, int rows_c,
                                   int n_t, double tau_kv, int guard, int pool_n, int t_q,
                                   uint8_t* __restrict__ cache_bits,
                                   uint8_t* __restrict__ skip_bits) {
  extern __shared__ double sk_smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kPolWarps + wib;
  if (gw >= H * rows_c) return;
  const int cols = rows_c, t_kv = t_q;
  const int h = gw / rows_c, r = gw % rows_c;
  double* v = sk_smem + (size_t)wib * cols * 4;  // candidate scores
  double* sorted = v + cols;
  int* rank = reinterpret_cast<int*>(sorted + cols);
  float* vf = reinterpret_cast<float*>(rank + cols);
  uint8_t* keep = reinterpret_cast<uint8_t*>(vf + cols);
  const bool active = comp_cache[(size_t)h * rows_c + r] != 0;
  const float* P = p_tilde + ((size_t)h * rows_c + r) * cols;
  // guarded: text columns and the diagonal are protected (square map: r < cols)
  const bool any_prot = guard != 0;
  auto prot = [&](int c) { return guard && (c < n_t || c == r); };
  // candidate k -> column: the unprotected columns in increasing order
  auto cand_col = [&](int k) {
    if (!guard) return k;
    int c = n_t + k;
    if (r >= n_t && c >= r) ++c;
    return c;
  };
  const int nc = guard ? cols - n_t - (r >= n_t ? 1 : 0) : cols;
  for (int c = lane; c < cols; c += 32) keep[c] = active && prot(c);
  if (active && nc > 0) {
    for (int k = lane; k < nc; k += 32) v[k] = (double)P[cand_col(k)];
    __syncwarp();
    const int cut = budget_prefix<false>(v, vf, nc, tau_kv, false, rank, sorted, lane, 32);
    int spare = -1;
    if (!any_prot && cut == nc) {  // all skipped: spare argmax (first occurrence)
      if (lane == 0) {
        spare = 0;
        for (int k = 1; k < nc; ++k)
          if (v[k] > v[spare]) spare = k;
      }
      spare = __shfl_sync(0xffffffffu, spare, 0);
    }
    for (int k = lane; k < nc; k += 32)
      if (rank[k] >= cut || k == spare) keep[cand_col(k)] = 1;
  }
  __syncwarp();
  for (int rr = r * pool_n; rr < min((r + 1) * pool_n, t_q); ++rr) {
    uint8_t* out = skip_bits + ((size_t)h * t_q + rr) * t_kv;
    for (int j = lane; j < t_kv; j += 32) out[j] = keep[j / pool_n];
    if (lane == 0) cache_bits[(size_t)h * t_q + rr] = active;
  }
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t policy_workspace_bytes(int H, int rows_c) {
  // pooled q, k [H, rows_c, 128] fp32 | p_tilde [H, rows_c, rows_c] fp32 |
  // compressed compute bits [H, rows_c]
  return 2 * al256((size_t)H * rows_c * kTile * 4) + al256((size_t)H * rows_c * rows_c * 4) +
         al256((size_t)H * rows_c);
}

cudaError_t launch_generate_masks(const __nv_bfloat16* q, const __nv_bfloat16* k, int S, int H,
                                  int n_t, int pool_n, double tau_q, double tau_kv, double s_q,
                                  int guard, uint8_t* cache_bits, uint8_t* skip_bits, void* ws,
                                  cudaStream_t stream) {
  const int block = pool_n * kTile;
  const int rows_c = (S + block - 1) / block;
  const int t_q = (S + kTile - 1) / kTile;
  char* w = static_cast<char*>(ws);
  float* pq = reinterpret_cast<float*>(w);
  w += al256((size_t)H * rows_c * kTile * 4);
  float* pk = reinterpret_cast<float*>(w);
  w += al256((size_t)H * rows_c * kTile * 4);
  float* pt = reinterpret_cast<float*>(w);
  w += al256((size_t)H * rows_c * rows_c * 4);
  uint8_t* cc = reinterpret_cast<uint8_t*>(w);

  const int n_pool = H * rows_c * (kTile / 2);
  note_launch();
  pool_kernel<<<dim3((n_pool + 255) / 256, 2), 256, 0, stream>>>(q, k, S, H, block, rows_c, pq, pk);
  const size_t sm_sc = scores_smem_bytes(rows_c);
  cudaFuncSetAttribute(scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc);
  const int rows_cta = kScWarps * kScRows;
  note_launch();
  scores_kernel<<<dim3((rows_c + rows_cta - 1) / rows_cta, H), kScWarps * 32, sm_sc, stream>>>(
      pq, pk, rows_c, pt);
  const int grid_rows = (H * rows_c + kPolWarps - 1) / kPolWarps;
  const size_t sm_rows = (size_t)kPolWarps * rows_c * 4 * sizeof(double);
  const size_t sm_cache =
      (size_t)rows_c * (3 * sizeof(double) + sizeof(int) + 2) + 8 + (size_t)rows_c * (8 + 4 + 4 + 4);
  cudaFuncSetAttribute(cache_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm_cache);
  note_launch();
  cache_select_kernel<<<H, 256, sm_cache, stream>>>(pt, rows_c, n_t, tau_q, s_q, cc);
  cudaFuncSetAttribute(skip_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_rows);
  note_launch();
  skip_select_kernel<<<grid_rows, kPolWarps * 32, sm_rows, stream>>>(
      pt, cc, H, rows_c, n_t, tau_kv, guard, pool_n, t_q, cache_bits, skip_bits);
  return cudaGetLastError();
}

}  // namespace fo
