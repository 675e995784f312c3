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
#include "fo_numpy.cuh"

namespace fo {

namespace {

constexpr int kPolWarps = 4;  // warps per CTA in the per-row kernels

// thread per (tensor, block, head, dim pair): q and k in one launch (each
// with its own pool length), paired loads (a warp reads one 128-wide head
// row), fp64 sums in row order. TIn = bf16 (the engine's activations) or float
// (the reference's float32 matrices).
__device__ __forceinline__ float2 ld_pair(const __nv_bfloat16* p) {
  const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(p));
  return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
}
__device__ __forceinline__ float2 ld_pair(const float* p) {
  return __ldg(reinterpret_cast<const float2*>(p));
}

template <typename TIn>
__global__ void pool_kernel(const TIn* __restrict__ xq, const TIn* __restrict__ xk, int S_q,
                            int S_k, int H, int block_q, int rows_q, int block_k, int rows_k,
                            float* __restrict__ oq, float* __restrict__ ok) {  // [H, rows, 128]
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int S = blockIdx.y ? S_k : S_q;
  const int block = blockIdx.y ? block_k : block_q, rows_c = blockIdx.y ? rows_k : rows_q;
  if (idx >= H * rows_c * (kTile / 2)) return;
  const TIn* x = blockIdx.y ? xk : xq;
  float* out = blockIdx.y ? ok : oq;
  // heads vary fastest after the dims: consecutive warps read one token row
  const int d = 2 * (idx % (kTile / 2)), h = (idx / (kTile / 2)) % H,
            r = idx / ((kTile / 2) * H);
  const int s0 = r * block, s1 = min(S, s0 + block);
  const TIn* p = x + (size_t)s0 * H * kTile + (size_t)h * kTile + d;
  const size_t stride = (size_t)H * kTile;
  double a0 = 0.0, a1 = 0.0;  // np.add.reduceat: sequential from the first element
#pragma unroll 8
  for (int s = s0; s < s1; ++s, p += stride) {
    const float2 v = ld_pair(p);
    a0 += (double)v.x;
    a1 += (double)v.y;
  }
  const double n = (double)(s1 - s0);
  *reinterpret_cast<float2*>(out + (size_t)(h * rows_c + r) * kTile + d) =
      make_float2((float)(a0 / n), (float)(a1 / n));
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
scores_kernel(const float* __restrict__ pq, const float* __restrict__ pk, int rows_c, int cols,
              double rs, float* __restrict__ p_tilde) {  // rs = sqrt(d) of the unpadded head dim
  extern __shared__ __align__(16) unsigned char sc_smem[];
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
    if (lane == 0) sum = pairwise_sum<5, double>(ew, cols);
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

// CTA per head. Stages (each optional, so the reference's building blocks can
// run one at a time; the engine's policy runs them all in one launch):
//   scores  p_tilde != null: contribution [cols - n_t] and guidance [rows - n_t]
//           from the map (written to contrib_out / guid_out when given);
//           otherwise they are read from contrib_in / guid_in [H, V]
//   select  cached != null: both ascending prefixes within tau_q of their
//           totals -> cached [H, V] (1 = cached), select_cached_blocks
//   fused   comp_cache != null: compressed compute bits [H, rows] (text rows
//           always computed) after degrade_to_full_cache with s_q
// n is the smem array length (>= rows, cols, V).
__global__ void __launch_bounds__(256)
cache_select_kernel(const float* __restrict__ p_tilde, int rows, int cols, int n_t,
                    const double* __restrict__ contrib_in, const double* __restrict__ guid_in,
                    int V_in, double* __restrict__ contrib_out, double* __restrict__ guid_out,
                    double tau_q, double s_q, int n, uint8_t* __restrict__ cached,
                    uint8_t* __restrict__ comp_cache) {
  extern __shared__ double cs_smem[];
  const int h = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  double* contrib = cs_smem;                              // [n]
  double* guid = contrib + n;                             // [n]
  double* sorted = guid + n;                              // [n]
  int* rank = reinterpret_cast<int*>(sorted + n);         // [n]
  uint8_t* cut_c = reinterpret_cast<uint8_t*>(rank + n);  // [n]
  uint8_t* cc = cut_c + n;                                // [n]
  double* e = reinterpret_cast<double*>(                  // [n] guidance scratch
      (reinterpret_cast<uintptr_t>(cc + n) + 7) & ~uintptr_t(7));
  float* tmp = reinterpret_cast<float*>(e + n);           // [n]
  float* acc = tmp + n;                                   // [n]
  float* vf = acc + n;                                    // [n] rank keys
  int V = V_in;
  if (p_tilde) {
    const float* P = p_tilde + (size_t)h * rows * cols;
    const int Vc = cols - n_t, Vg = rows - n_t;
    V = Vc;
    // vision_to_text_contribution: p[:n_t, n_t:].sum(axis=0), fp32 row by row
    for (int c = tid; c < Vc; c += nt) {
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
      for (int c = tid; c < Vg; c += nt) {
        tmp[c] = P[(size_t)(n_t + c) * cols + j];
        mx = fmaxf(mx, tmp[c]);
      }
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((tid & 31) == 0) red[tid >> 5] = mx;
      __syncthreads();
      mx = red[0];
      for (int w = 1; w < nt / 32; ++w) mx = fmaxf(mx, red[w]);
      for (int c = tid; c < Vg; c += nt) e[c] = exp((double)tmp[c] - (double)mx);
      __syncthreads();
      if (tid == 0) s_sum = pairwise_sum<5, double>(e, Vg);
      __syncthreads();
      const double sum = s_sum;
      for (int c = tid; c < Vg; c += nt) {
        const float beta = (float)(e[c] / sum);
        acc[c] = j ? acc[c] + beta : beta;
      }
      __syncthreads();
    }
    for (int c = tid; c < Vg; c += nt) guid[c] = n_t > 0 ? (double)acc[c] : 0.0;
    if (contrib_out)
      for (int c = tid; c < Vc; c += nt) contrib_out[(size_t)h * Vc + c] = contrib[c];
    if (guid_out)
      for (int c = tid; c < Vg; c += nt) guid_out[(size_t)h * Vg + c] = guid[c];
  } else {
    for (int c = tid; c < V; c += nt) {
      contrib[c] = contrib_in[(size_t)h * V + c];
      guid[c] = guid_in[(size_t)h * V + c];
    }
  }
  __syncthreads();
  if (!cached && !comp_cache) return;
  // select_cached_blocks: both ascending prefixes within tau_q of their totals
  int cut = budget_prefix<true>(contrib, vf, V, tau_q, true, rank, sorted, tid, nt);
  for (int i = tid; i < V; i += nt) cut_c[i] = rank[i] < cut;
  __syncthreads();
  cut = budget_prefix<true>(guid, vf, V, tau_q, true, rank, sorted, tid, nt);
  if (cached)
    for (int i = tid; i < V; i += nt) cached[(size_t)h * V + i] = cut_c[i] && rank[i] < cut;
  if (!comp_cache) return;
  for (int r = tid; r < rows; r += nt)
    cc[r] = (r < n_t) ? 1 : !(cut_c[r - n_t] && rank[r - n_t] < cut);
  __syncthreads();
  // degrade_to_full_cache: computed vision fraction below s_q -> cache all vision
  __shared__ int n_comp;
  if (tid == 0) {
    int c = 0;
    for (int r = n_t; r < rows; ++r) c += cc[r];
    n_comp = c;
  }
  __syncthreads();
  const bool degrade = V > 0 && (double)n_comp / (double)V < s_q;
  for (int r = tid; r < rows; r += nt)
    comp_cache[(size_t)h * rows + r] = (degrade && r >= n_t) ? 0 : cc[r];
}

size_t cache_select_smem(int n) {
  return (size_t)n * (3 * sizeof(double) + sizeof(int) + 2) + 8 + (size_t)n * (8 + 4 + 4 + 4);
}

// warp per (head, compressed row): select_skip_blocks for computed rows, then
// expand_blocks into block-granularity bits (policy.py:124-159, 190-193).
// The map is rows x cols; with pool_n = 1 and t_q = rows, t_kv = cols the
// output is the compressed keep mask itself.
__global__ void skip_select_kernel(const float* __restrict__ p_tilde,
                                   const uint8_t* __restrict__ comp_cache, int H, int rows_c,
                                   int cols, int n_t, double tau_kv, int guard, int pool_n,
                                   int t_q, int t_kv, uint8_t* __restrict__ cache_bits,
                                   uint8_t* __restrict__ skip_bits) {
  extern __shared__ double sk_smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kPolWarps + wib;
  if (gw >= H * rows_c) return;
  const int h = gw / rows_c, r = gw % rows_c;
  double* v = sk_smem + (size_t)wib * cols * 4;  // candidate scores
  double* sorted = v + cols;
  int* rank = reinterpret_cast<int*>(sorted + cols);
  float* vf = reinterpret_cast<float*>(rank + cols);
  uint8_t* keep = reinterpret_cast<uint8_t*>(vf + cols);
  const bool active = comp_cache[(size_t)h * rows_c + r] != 0;
  const float* P = p_tilde + ((size_t)h * rows_c + r) * cols;
  // guarded: text columns and the diagonal block (when r < cols) are protected
  const bool diag = r < cols;
  const bool any_prot = guard != 0 && (n_t > 0 || diag);
  auto prot = [&](int c) { return guard && (c < n_t || c == r); };
  const bool diag_extra = guard && diag && r >= n_t;  // the diagonal sits among the candidates
  // candidate k -> column: the unprotected columns in increasing order
  auto cand_col = [&](int k) {
    if (!guard) return k;
    int c = n_t + k;
    if (diag_extra && c >= r) ++c;
    return c;
  };
  const int nc = guard ? cols - n_t - (diag_extra ? 1 : 0) : cols;
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
    if (cache_bits && lane == 0) cache_bits[(size_t)h * t_q + rr] = active;
  }
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

template <typename TIn>
void launch_map(const TIn* q, const TIn* k, int S_q, int S_k, int H, int block_q, int rows_q,
                int block_k, int rows_k, double rs, float* pq, float* pk, float* pt,
                cudaStream_t stream) {
  const int n_pool = H * max(rows_q, rows_k) * (kTile / 2);
  note_launch();
  pool_kernel<TIn><<<dim3((n_pool + 255) / 256, 2), 256, 0, stream>>>(
      q, k, S_q, S_k, H, block_q, rows_q, block_k, rows_k, pq, pk);
  const size_t sm_sc = scores_smem_bytes(rows_k);
  cudaFuncSetAttribute(scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc);
  const int rows_cta = kScWarps * kScRows;
  note_launch();
  scores_kernel<<<dim3((rows_q + rows_cta - 1) / rows_cta, H), kScWarps * 32, sm_sc, stream>>>(
      pq, pk, rows_q, rows_k, rs, pt);
}

void launch_cache_select(const float* pt, int H, int rows, int cols, int n_t, const double* c_in,
                         const double* g_in, int V_in, double* c_out, double* g_out, double tau_q,
                         double s_q, uint8_t* cached, uint8_t* comp_cache, cudaStream_t stream) {
  const int n = max(max(rows, cols), max(V_in, 1));
  const size_t sm = cache_select_smem(n);
  cudaFuncSetAttribute(cache_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  note_launch();
  cache_select_kernel<<<H, 256, sm, stream>>>(pt, rows, cols, n_t, c_in, g_in, V_in, c_out, g_out,
                                              tau_q, s_q, n, cached, comp_cache);
}

void launch_skip_select(const float* pt, const uint8_t* cc, int H, int rows, int cols, int n_t,
                        double tau_kv, int guard, int pool_n, int t_q, int t_kv,
                        uint8_t* cache_bits, uint8_t* skip_bits, cudaStream_t stream) {
  const int grid_rows = (H * rows + kPolWarps - 1) / kPolWarps;
  const size_t sm_rows = (size_t)kPolWarps * cols * 4 * sizeof(double);
  cudaFuncSetAttribute(skip_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_rows);
  note_launch();
  skip_select_kernel<<<grid_rows, kPolWarps * 32, sm_rows, stream>>>(
      pt, cc, H, rows, cols, n_t, tau_kv, guard, pool_n, t_q, t_kv, cache_bits, skip_bits);
}

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
  launch_map(q, k, S, S, H, block, rows_c, block, rows_c, sqrt((double)kTile), pq, pk, pt, stream);
  launch_cache_select(pt, H, rows_c, rows_c, n_t, nullptr, nullptr, 0, nullptr, nullptr, tau_q,
                      s_q, nullptr, cc, stream);
  launch_skip_select(pt, cc, H, rows_c, rows_c, n_t, tau_kv, guard, pool_n, t_q, t_q, cache_bits,
                     skip_bits, stream);
  return cudaGetLastError();
}

// ---- the reference's policy building blocks one stage at a time (policy.py:21-178)
size_t policy_map_workspace_bytes(int H, int rows_q, int rows_k) {
  return al256((size_t)H * rows_q * kTile * 4) + al256((size_t)H * rows_k * kTile * 4);
}

cudaError_t launch_policy_map(const void* q, const void* k, int is_f32, int S_q, int S_k, int H,
                              int d, int pool_q, int pool_k, float* p_tilde, void* ws,
                              cudaStream_t stream) {
  const int rows_q = (S_q + pool_q - 1) / pool_q, rows_k = (S_k + pool_k - 1) / pool_k;
  float* pq = static_cast<float*>(ws);
  float* pk = reinterpret_cast<float*>(static_cast<char*>(ws) +
                                       al256((size_t)H * rows_q * kTile * 4));
  const double rs = sqrt((double)d);
  if (is_f32)
    launch_map(static_cast<const float*>(q), static_cast<const float*>(k), S_q, S_k, H, pool_q,
               rows_q, pool_k, rows_k, rs, pq, pk, p_tilde, stream);
  else
    launch_map(static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), S_q, S_k,
               H, pool_q, rows_q, pool_k, rows_k, rs, pq, pk, p_tilde, stream);
  return cudaGetLastError();
}

cudaError_t launch_policy_scores(const float* p_tilde, int H, int rows, int cols, int n_t,
                                 double* contribution, double* guidance, cudaStream_t stream) {
  launch_cache_select(p_tilde, H, rows, cols, n_t, nullptr, nullptr, 0, contribution, guidance,
                      0.0, 0.0, nullptr, nullptr, stream);
  return cudaGetLastError();
}

cudaError_t launch_policy_select_cached(const double* contribution, const double* guidance, int H,
                                        int V, double tau_q, uint8_t* cached, cudaStream_t stream) {
  launch_cache_select(nullptr, H, 0, 0, 0, contribution, guidance, V, nullptr, nullptr, tau_q, 0.0,
                      cached, nullptr, stream);
  return cudaGetLastError();
}

cudaError_t launch_policy_select_skip(const float* p_tilde, const uint8_t* compute, int H, int rows,
                                      int cols, int n_t, double tau_kv, int guard, uint8_t* keep,
                                      cudaStream_t stream) {
  launch_skip_select(p_tilde, compute, H, rows, cols, n_t, tau_kv, guard, 1, rows, cols, nullptr,
                     keep, stream);
  return cudaGetLastError();
}

}  // namespace fo
