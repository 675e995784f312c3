// The reference's tile-level building blocks on the device: the online-softmax
// recurrence (attention.py:21-55), one cache entry's update / forecast
// (attention.py:71-113) and the dense numerics of tensor.py:33-126 that the
// policy and the tests build on. These are the operator API's small pieces,
// not the layer hot path (that is the batched kernels of fo_attention_cs.cu,
// fo_gemm.cu, fo_policy.cu); they follow numpy's float32 / float64 arithmetic
// so results match the reference bit for bit where numpy's order is fixed
// (sequential / pairwise sums, single-rounded products: __fmul_rn / __fadd_rn
// keep nvcc from contracting into FMAs), and within float32 rounding where it
// is BLAS- or libm-defined (p @ v, exp).
#include "fo_internal.cuh"
#include "fo_numpy.cuh"

namespace fo {

namespace {

constexpr int kRowThreads = 128;

__device__ float block_max(float v, float* red) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float m = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  return m;
}

// numpy maximum: NaN propagates
__device__ __forceinline__ float np_maximum(float a, float b) {
  return (a != a || b != b) ? __int_as_float(0x7fc00000) : fmaxf(a, b);
}

// CTA per query row (attention.py:39-49):
//   m' = max(m, rowmax(S)); corr = exp(m - m'); p = exp(S - m')
//   l' = l*corr + sum(p); acc' = acc*corr + p @ V
__global__ void __launch_bounds__(kRowThreads)
online_softmax_update_kernel(const float* __restrict__ m, const float* __restrict__ l,
                             const float* __restrict__ acc, const float* __restrict__ scores,
                             const float* __restrict__ v, int cols, int d, float* __restrict__ m_out,
                             float* __restrict__ l_out, float* __restrict__ acc_out) {
  extern __shared__ float p_s[];  // [cols]
  __shared__ float red[kRowThreads / 32];
  __shared__ float s_corr, s_m;
  const int r = blockIdx.x, tid = threadIdx.x;
  const float* srow = scores + (size_t)r * cols;
  float mx = -INFINITY;
  bool nan = false;
  for (int c = tid; c < cols; c += blockDim.x) {
    const float x = srow[c];
    nan |= x != x;
    mx = fmaxf(mx, x);
  }
  mx = block_max(mx, red);
  nan = __syncthreads_or(nan);
  if (tid == 0) {
    const float m_new = np_maximum(m[r], nan ? __int_as_float(0x7fc00000) : mx);
    s_m = m_new;
    s_corr = expf(__fsub_rn(m[r], m_new));
  }
  __syncthreads();
  const float m_new = s_m, corr = s_corr;
  for (int c = tid; c < cols; c += blockDim.x) p_s[c] = expf(__fsub_rn(srow[c], m_new));
  __syncthreads();
  if (tid == 0) {
    m_out[r] = m_new;
    l_out[r] = __fadd_rn(__fmul_rn(l[r], corr), pairwise_sum<8, float>(p_s, cols));
  }
  for (int j = tid; j < d; j += blockDim.x) {
    float pv = 0.f;
    for (int c = 0; c < cols; ++c) pv = fmaf(p_s[c], v[(size_t)c * d + j], pv);
    acc_out[(size_t)r * d + j] = __fadd_rn(__fmul_rn(acc[(size_t)r * d + j], corr), pv);
  }
}

// diag(l)^-1 acc (attention.py:52-55); an empty row (l <= 0) is a
// ConsistencyError, latched in the status word
__global__ void online_softmax_finalize_kernel(const float* __restrict__ acc,
                                               const float* __restrict__ l, int rows, int d,
                                               float* __restrict__ out, uint32_t* status) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)rows * d) return;
  const float li = l[i / d];
  if (li <= 0.f && i % d == 0) raise_status(status, ST_CONSISTENCY);
  out[i] = __fdiv_rn(acc[i], li);
}

// update_entry (attention.py:71-85): stack[0] = o; stack[k] = stack[k-1] - old[k-1]
// for k < valid; deeper levels zero. One thread per tile element.
__global__ void update_entry_kernel(const float* __restrict__ old, const float* __restrict__ o,
                                    size_t tile, int order, int valid, float* __restrict__ stack) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tile) return;
  float prev = o[i];
  stack[i] = prev;
  for (int k = 1; k <= order; ++k) {
    prev = k < valid ? __fsub_rn(prev, old[(size_t)(k - 1) * tile + i]) : 0.f;
    stack[(size_t)k * tile + i] = prev;
  }
}

struct Coef {
  float c[8];
};

// forecast (attention.py:96-113): out = c0*stack[0]; out += c_d*stack[d]
__global__ void forecast_entry_kernel(const float* __restrict__ stack, size_t tile, int n_orders,
                                      Coef coef, float* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tile) return;
  float acc = __fmul_rn(coef.c[0], stack[i]);
  for (int k = 1; k < n_orders; ++k)
    acc = __fadd_rn(acc, __fmul_rn(coef.c[k], stack[(size_t)k * tile + i]));
  out[i] = acc;
}

// mean_pool_blocks (tensor.py:112-126): np.add.reduceat in float64 from the
// block's first row, / actual length, -> float32. Thread per (block, column).
__global__ void mean_pool_kernel(const float* __restrict__ x, int n, int d, int pool, int blocks,
                                 float* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)blocks * d) return;
  const int c = (int)(i % d), b = (int)(i / d);
  const int s0 = b * pool, s1 = min(n, s0 + pool);
  double a = 0.0;
  for (int s = s0; s < s1; ++s) a += (double)x[(size_t)s * d + c];
  out[i] = (float)(a / (double)(s1 - s0));
}

// rms_norm (tensor.py:68-80): ms = pairwise fp64 mean of x^2; y = fp32(x*w) * (1/sqrt(ms+eps))
// in fp64, -> fp32. CTA per row.
__global__ void __launch_bounds__(kRowThreads)
rms_norm_kernel(const float* __restrict__ x, const float* __restrict__ w, int d, double eps,
                float* __restrict__ out) {
  extern __shared__ double sq[];  // [d]
  __shared__ double s_inv;
  const float* xr = x + (size_t)blockIdx.x * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const double v = (double)xr[c];
    sq[c] = v * v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double ms = pairwise_sum<10, double>(sq, d) / (double)d;
    s_inv = 1.0 / sqrt(ms + eps);
  }
  __syncthreads();
  const double inv = s_inv;
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    out[(size_t)blockIdx.x * d + c] = (float)((double)__fmul_rn(xr[c], w[c]) * inv);
}

// rope (tensor.py:83-109), interleaved pairs, cos/sin tables fp32 [n, d/2]
// (float64 angles cast once, as the reference computes them)
__global__ void rope_kernel(const float* __restrict__ x, const float* __restrict__ cs,
                            const float* __restrict__ sn, int n, int d, float* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int half = d / 2;
  if (i >= (size_t)n * half) return;
  const size_t r = i / half;
  const int j = (int)(i % half);
  const float e = x[r * d + 2 * j], o = x[r * d + 2 * j + 1];
  const float c = cs[i], s = sn[i];
  out[r * d + 2 * j] = __fsub_rn(__fmul_rn(e, c), __fmul_rn(o, s));
  out[r * d + 2 * j + 1] = __fadd_rn(__fmul_rn(e, s), __fmul_rn(o, c));
}

// row_softmax (tensor.py:42-47): fp64 exp(s - rowmax), pairwise fp64 row sum,
// e / sum -> fp32. CTA per row.
__global__ void __launch_bounds__(kRowThreads)
row_softmax_kernel(const float* __restrict__ s, int d, float* __restrict__ out) {
  extern __shared__ double e_s[];  // [d]
  __shared__ float red[kRowThreads / 32];
  __shared__ double s_sum;
  const float* sr = s + (size_t)blockIdx.x * d;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < d; c += blockDim.x) mx = fmaxf(mx, sr[c]);
  mx = block_max(mx, red);
  for (int c = threadIdx.x; c < d; c += blockDim.x) e_s[c] = exp((double)sr[c] - (double)mx);
  __syncthreads();
  if (threadIdx.x == 0) s_sum = pairwise_sum<10, double>(e_s, d);
  __syncthreads();
  const double sum = s_sum;
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    out[(size_t)blockIdx.x * d + c] = (float)(e_s[c] / sum);
}

int grid_of(size_t n) { return (int)((n + 255) / 256); }


// The reference tile kernel at any block size and head dim, in fp32
// (pyref.py:14-48 / _core.pyx:14-101): for every active query block i and
// every key block j with pair_bits[i][j] set, per row
//   m' = max(m, rowmax(S_ij)); corr = exp(m - m'); p = exp(S_ij - m')
//   l' = l*corr + sum(p); acc' = acc*corr + p V_j;   out_i = acc / l.
// One CTA per query block, one thread per row (128 rows per pass). K / V rows
// are staged in shared memory in chunks of KC rows padded to DP columns; S is
// recomputed in a second pass instead of stored. This is the drop-in's general
// path for shapes the tcgen05 kernel does not tile (b != 128, the reference's
// own small-d tests); it matches the reference's float32 arithmetic to
// rounding (expf, fp32 accumulation).
constexpr int kMbaThreads = 128;
constexpr int kMbaChunkFloats = 4096;  // per staged operand: 16 KB

template <int DP>
__global__ void __launch_bounds__(kMbaThreads)
masked_block_attention_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                  const float* __restrict__ v, int n, int d,
                                  const uint8_t* __restrict__ active,
                                  const uint8_t* __restrict__ pair_bits, int t_kv, int b_q, int b_k,
                                  float scale, float* __restrict__ out,
                                  unsigned long long* __restrict__ pairs, uint32_t* status) {
  constexpr int KC = kMbaChunkFloats / DP;
  __shared__ float sk[KC * DP], sv[KC * DP];
  const int i = blockIdx.x;
  if (!active[i]) return;
  const uint8_t* prow = pair_bits + (size_t)i * t_kv;
  if (threadIdx.x == 0) {
    unsigned long long c = 0;
    for (int j = 0; j < t_kv; ++j) c += prow[j] != 0;
    if (c == 0) raise_status(status, ST_CONSISTENCY);  // l = 0: pyref.py:44-46
    else if (pairs) atomicAdd(pairs, c);
  }
  const int r0 = i * b_q, r1 = min(r0 + b_q, n);
  for (int rb = r0; rb < r1; rb += kMbaThreads) {
    const int r = rb + (int)threadIdx.x;
    const bool live = r < r1;
    float qr[DP], acc[DP];
#pragma unroll
    for (int c = 0; c < DP; ++c) {
      qr[c] = (live && c < d) ? q[(size_t)r * d + c] : 0.f;
      acc[c] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < t_kv; ++j) {
      if (!prow[j]) continue;
      const int c0 = j * b_k, c1 = min(c0 + b_k, n);
      auto stage = [&](int cb, int ce, bool with_v) {
        __syncthreads();  // the previous chunk is consumed
        for (int e = threadIdx.x; e < (ce - cb) * DP; e += kMbaThreads) {
          const int kr = e / DP, c = e - kr * DP;
          sk[e] = c < d ? k[(size_t)(cb + kr) * d + c] : 0.f;
          if (with_v) sv[e] = c < d ? v[(size_t)(cb + kr) * d + c] : 0.f;
        }
        __syncthreads();
      };
      auto dot = [&](int kr) {
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < DP; ++c) s = fmaf(qr[c], sk[kr * DP + c], s);
        return s * scale;
      };
      float mb = -INFINITY;  // pass 1: the block's row max
      for (int cb = c0; cb < c1; cb += KC) {
        const int ce = min(cb + KC, c1);
        stage(cb, ce, false);
        for (int kr = 0; kr < ce - cb; ++kr) mb = fmaxf(mb, dot(kr));
      }
      const float m_new = fmaxf(m, mb);
      const float corr = expf(m - m_new);  // m = -inf on the first block: 0
      l *= corr;
#pragma unroll
      for (int c = 0; c < DP; ++c) acc[c] *= corr;
      for (int cb = c0; cb < c1; cb += KC) {  // pass 2: p, l and p V
        const int ce = min(cb + KC, c1);
        stage(cb, ce, true);
        for (int kr = 0; kr < ce - cb; ++kr) {
          const float pr = expf(dot(kr) - m_new);
          l += pr;
#pragma unroll
          for (int c = 0; c < DP; ++c) acc[c] = fmaf(pr, sv[kr * DP + c], acc[c]);
        }
      }
      m = m_new;
    }
    if (live) {
#pragma unroll
      for (int c = 0; c < DP; ++c)  // static indices: acc stays in registers
        if (c < d) out[(size_t)r * d + c] = acc[c] / l;
    }
  }
}

// C (+)= A B in fp32, row-major A [m, k], B [k, n], C [m, n]: the product of
// the reference-signature GEMM paths at shapes the tcgen05 kernels do not tile
// (gemm.py:44-229 at b_q != 128 or head dims != 128, numpy's float32 matmul).
// 64 x 64 output tiles, 16 x 16 threads with 4 x 4 outputs each, k in order.
constexpr int kMmTile = 64, kMmK = 16;
__global__ void __launch_bounds__(256)
matmul_f32_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ c,
                  int m, int n, int k, int accumulate) {
  __shared__ float as[kMmK][kMmTile + 4];  // A tile transposed: as[kk][row]
  __shared__ float bs[kMmK][kMmTile];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = blockIdx.y * kMmTile, c0 = blockIdx.x * kMmTile;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < k; k0 += kMmK) {
    for (int e = threadIdx.x; e < kMmTile * kMmK; e += 256) {
      const int rr = e / kMmK, kk = e % kMmK;  // A: 64 rows x 16 k
      const int gr = r0 + rr, gk = k0 + kk;
      as[kk][rr] = (gr < m && gk < k) ? a[(size_t)gr * k + gk] : 0.f;
      const int kb = e / kMmTile, cc = e % kMmTile;  // B: 16 k x 64 cols
      const int gk2 = k0 + kb, gc = c0 + cc;
      bs[kb][cc] = (gk2 < k && gc < n) ? b[(size_t)gk2 * n + gc] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kMmK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = as[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = r0 + ty * 4 + i;
    if (gr >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = c0 + tx * 4 + j;
      if (gc >= n) continue;
      float* cp = c + (size_t)gr * n + gc;
      *cp = accumulate ? __fadd_rn(*cp, acc[i][j]) : acc[i][j];
    }
  }
}
}  // namespace

// largest row width of the per-row kernels (shared-memory bound)
constexpr int kMaxRowWidth = 24576;

cudaError_t launch_online_softmax_update(const float* m, const float* l, const float* acc,
                                         const float* scores, const float* v, int rows, int cols,
                                         int d, float* m_out, float* l_out, float* acc_out,
                                         cudaStream_t st) {
  const size_t sm = (size_t)cols * 4;
  cudaFuncSetAttribute(online_softmax_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm);
  note_launch();
  online_softmax_update_kernel<<<rows, kRowThreads, sm, st>>>(m, l, acc, scores, v, cols, d, m_out,
                                                              l_out, acc_out);
  return cudaGetLastError();
}

cudaError_t launch_online_softmax_finalize(const float* acc, const float* l, int rows, int d,
                                           float* out, uint32_t* status, cudaStream_t st) {
  note_launch();
  online_softmax_finalize_kernel<<<grid_of((size_t)rows * d), 256, 0, st>>>(acc, l, rows, d, out,
                                                                            status);
  return cudaGetLastError();
}

cudaError_t launch_update_entry(const float* old, const float* o, size_t tile, int order, int valid,
                                float* stack, cudaStream_t st) {
  note_launch();
  update_entry_kernel<<<grid_of(tile), 256, 0, st>>>(old, o, tile, order, valid, stack);
  return cudaGetLastError();
}

cudaError_t launch_forecast_entry(const float* stack, size_t tile, int n_orders, const float* coef,
                                  float* out, cudaStream_t st) {
  Coef c{};
  for (int k = 0; k < n_orders && k < 8; ++k) c.c[k] = coef[k];
  note_launch();
  forecast_entry_kernel<<<grid_of(tile), 256, 0, st>>>(stack, tile, n_orders, c, out);
  return cudaGetLastError();
}

cudaError_t launch_mean_pool(const float* x, int n, int d, int pool, float* out, cudaStream_t st) {
  const int blocks = (n + pool - 1) / pool;
  note_launch();
  mean_pool_kernel<<<grid_of((size_t)blocks * d), 256, 0, st>>>(x, n, d, pool, blocks, out);
  return cudaGetLastError();
}

cudaError_t launch_rms_norm(const float* x, const float* w, int n, int d, double eps, float* out,
                            cudaStream_t st) {
  const size_t sm = (size_t)d * 8;
  cudaFuncSetAttribute(rms_norm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  note_launch();
  rms_norm_kernel<<<n, kRowThreads, sm, st>>>(x, w, d, eps, out);
  return cudaGetLastError();
}

cudaError_t launch_rope(const float* x, const float* cs, const float* sn, int n, int d, float* out,
                        cudaStream_t st) {
  note_launch();
  rope_kernel<<<grid_of((size_t)n * (d / 2)), 256, 0, st>>>(x, cs, sn, n, d, out);
  return cudaGetLastError();
}

cudaError_t launch_row_softmax(const float* s, int n, int d, float* out, cudaStream_t st) {
  const size_t sm = (size_t)d * 8;
  cudaFuncSetAttribute(row_softmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  note_launch();
  row_softmax_kernel<<<n, kRowThreads, sm, st>>>(s, d, out);
  return cudaGetLastError();
}

cudaError_t launch_masked_block_attention_f32(const float* q, const float* k, const float* v, int n,
                                              int d, const uint8_t* active,
                                              const uint8_t* pair_bits, int b_q, int b_k,
                                              float scale, float* out, unsigned long long* pairs,
                                              uint32_t* status, cudaStream_t st) {
  const int t_q = (n + b_q - 1) / b_q, t_kv = (n + b_k - 1) / b_k;
  note_launch();
#define FO_MBA(DP)                                                                        \
  masked_block_attention_f32_kernel<DP><<<t_q, kMbaThreads, 0, st>>>(                     \
      q, k, v, n, d, active, pair_bits, t_kv, b_q, b_k, scale, out, pairs, status)
  if (d <= 16) FO_MBA(16);
  else if (d <= 32) FO_MBA(32);
  else if (d <= 64) FO_MBA(64);
  else if (d <= 128) FO_MBA(128);
  else FO_MBA(256);
#undef FO_MBA
  return cudaGetLastError();
}

cudaError_t launch_matmul_f32(const float* a, const float* b, float* c, int m, int n, int k,
                              int accumulate, cudaStream_t st) {
  note_launch();
  const dim3 grid((n + kMmTile - 1) / kMmTile, (m + kMmTile - 1) / kMmTile);
  matmul_f32_kernel<<<grid, 256, 0, st>>>(a, b, c, m, n, k, accumulate);
  return cudaGetLastError();
}

int max_row_width() { return kMaxRowWidth; }

}  // namespace fo
