// Bandwidth-bound helpers around the tensor-core kernels.
//
// forecast_materialize: OP_reuse for mode="materialize" (reference
//   attention.py:96-113,212-216): cached query tiles are written as
//   sum_d c_d * diff_stack[d] into the attention output.
// cache_push: FeatureCache.update for an arbitrary set of (head, block) entries
//   (attention.py:71-85,128-131), the standalone form of the push the
//   update-mode attention epilogue performs.
// Both are HBM-bound; one CTA per (head, block) tile, 16-byte accesses.
#include "fo_internal.cuh"

namespace fo {

__global__ void forecast_materialize_kernel(const __nv_bfloat16* __restrict__ cache, int S, int H,
                                            int t_q, int order_d,
                                            const unsigned long long* __restrict__ hmask,
                                            const int32_t* __restrict__ valid, float c0, float c1,
                                            float c2, float c3, __nv_bfloat16* __restrict__ out) {
  const int tile = blockIdx.x;
  const int h = tile / t_q, i = tile % t_q;
  if ((hmask[i] >> h) & 1ull) return;  // computed tile, not forecast
  const int n = min(order_d + 1, valid[(size_t)h * t_q + i]);
  const float cf[4] = {c0, c1, c2, c3};
  const size_t HD = (size_t)H * kTile;
  const size_t SS = (size_t)S * HD;
  const int rows = min(kTile, S - i * kTile);
  for (int e = threadIdx.x; e < rows * 16; e += blockDim.x) {
    const int rr = e >> 4, v = e & 15;
    const size_t off = (size_t)(i * kTile + rr) * HD + (size_t)h * kTile + v * 8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int d = 0; d < n; ++d) {
      const uint4 w = *reinterpret_cast<const uint4*>(cache + d * SS + off);
      const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[2 * q] = fmaf(cf[d], bf16lo(w4[q]), acc[2 * q]);
        acc[2 * q + 1] = fmaf(cf[d], bf16hi(w4[q]), acc[2 * q + 1]);
      }
    }
    uint4 pk;
    pk.x = pack_bf16x2(acc[0], acc[1]);
    pk.y = pack_bf16x2(acc[2], acc[3]);
    pk.z = pack_bf16x2(acc[4], acc[5]);
    pk.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(out + off) = pk;
  }
}

__global__ void cache_push_kernel(const __nv_bfloat16* __restrict__ o, __nv_bfloat16* __restrict__ cache,
                                  int32_t* __restrict__ valid, int S, int H, int t_q, int order_d,
                                  const uint8_t* __restrict__ sel, int one_tile) {
  // one_tile >= 0: a single (head, block) entry h * t_q + i whose fresh output
  // `o` is that tile alone, [rows, 128] (FeatureCache.update, attention.py:128-131)
  const int tile = one_tile >= 0 ? one_tile : blockIdx.x;
  const int h = tile / t_q, i = tile % t_q;
  if (sel && !sel[(size_t)h * t_q + i]) return;
  const int valid_old = valid[(size_t)h * t_q + i];
  const int vn = min(valid_old + 1, order_d + 1);
  const size_t HD = (size_t)H * kTile;
  const size_t SS = (size_t)S * HD;
  const int rows = min(kTile, S - i * kTile);
  for (int e = threadIdx.x; e < rows * 16; e += blockDim.x) {
    const int rr = e >> 4, v = e & 15;
    const size_t off = (size_t)(i * kTile + rr) * HD + (size_t)h * kTile + v * 8;
    const size_t o_off = one_tile >= 0 ? (size_t)rr * kTile + v * 8 : off;
    const uint4 ov = *reinterpret_cast<const uint4*>(o + o_off);
    float cur[8] = {bf16lo(ov.x), bf16hi(ov.x), bf16lo(ov.y), bf16hi(ov.y),
                    bf16lo(ov.z), bf16hi(ov.z), bf16lo(ov.w), bf16hi(ov.w)};
    for (int d = 0; d <= order_d; ++d) {
      uint4* slot = reinterpret_cast<uint4*>(cache + d * SS + off);
      float nxt[8];
      const bool live_next = d + 1 < vn;
      if (live_next) {
        const uint4 w = *slot;
        const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          nxt[2 * q] = cur[2 * q] - bf16lo(w4[q]);
          nxt[2 * q + 1] = cur[2 * q + 1] - bf16hi(w4[q]);
        }
      }
      uint4 pk = make_uint4(0, 0, 0, 0);
      if (d < vn) {
        pk.x = pack_bf16x2(cur[0], cur[1]);
        pk.y = pack_bf16x2(cur[2], cur[3]);
        pk.z = pack_bf16x2(cur[4], cur[5]);
        pk.w = pack_bf16x2(cur[6], cur[7]);
      }
      *slot = pk;
      if (live_next) {
#pragma unroll
        for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) valid[(size_t)h * t_q + i] = vn;
}

// SyntheticWorkload.x(t) (reference pipeline.py:160-171) in one pass: the
// float32 products and float64 sums in numpy's order, rounded to float32 then
// bf16. __fmul_rn / __fadd_rn keep nvcc from contracting into FMAs, which
// numpy does not do. kind 0 drift, 1 poly1, 2 poly2.
__global__ void synthetic_x_kernel(const float* __restrict__ x0, const float* __restrict__ a,
                                   const float* __restrict__ b, size_t n, int kind, float c1,
                                   float c2, float s, __nv_bfloat16* __restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    double x = (double)x0[e];
    if (kind == 0) {  // base + s * (t * a + (t*t/steps) * b)
      const float inner = __fadd_rn(__fmul_rn(c1, a[e]), __fmul_rn(c2, b[e]));
      x = x + (double)__fmul_rn(s, inner);
    } else if (kind == 1) {  // base + (s*t) * a
      x = x + (double)__fmul_rn(c1, a[e]);
    } else {  // base + (s*t) * a + (s*t)**2 * b
      x = x + (double)__fmul_rn(c1, a[e]);
      x = x + (double)__fmul_rn(c2, b[e]);
    }
    out[e] = __float2bfloat16_rn((float)x);
  }
}

// Input validation (reference tensor.py:19-30 as_matrix, attention.py:176-196):
// any NaN / Inf among the bf16 values sets ST_PARAM. With `hmask`, element
// (row, col) is checked only when head col/128 is active for block row/128
// (cached q rows are unwritten placeholders the kernels never read). A bf16 is
// non-finite iff its exponent bits are all ones. HBM-bound: 16-byte loads.
__global__ void check_finite_kernel(const uint4* __restrict__ data, long long rows, int cols,
                                    const unsigned long long* __restrict__ hmask,
                                    uint32_t* status) {
  const int cpr = cols / 8;  // 16-byte chunks per row
  const long long total = rows * cpr;
  uint32_t bad = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    if (hmask) {
      const long long r = e / cpr;
      const int h = (int)(e - r * cpr) * 8 / kTile;
      if (!((hmask[r / kTile] >> h) & 1ull)) continue;
    }
    const uint4 v = __ldcs(data + e);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      bad |= ((w[q] & 0x7F80u) == 0x7F80u) | ((w[q] & 0x7F800000u) == 0x7F800000u);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_status(status, ST_PARAM);
}

void launch_check_finite(const void* data, long long rows, int cols,
                         const unsigned long long* hmask, uint32_t* status, cudaStream_t stream) {
  note_launch();
  check_finite_kernel<<<148 * 8, 256, 0, stream>>>(static_cast<const uint4*>(data), rows, cols,
                                                   hmask, status);
}

void launch_synthetic_x(const float* x0, const float* a, const float* b, size_t n, int kind,
                        float c1, float c2, float s, __nv_bfloat16* out, cudaStream_t stream) {
  note_launch();
  synthetic_x_kernel<<<148 * 8, 256, 0, stream>>>(x0, a, b, n, kind, c1, c2, s, out);
}

void launch_forecast_materialize(const __nv_bfloat16* cache, int S, int H, int t_q, int order_d,
                                 const unsigned long long* hmask, const int32_t* valid,
                                 const float* coef, __nv_bfloat16* out, cudaStream_t stream) {
  note_launch();
  forecast_materialize_kernel<<<H * t_q, 256, 0, stream>>>(cache, S, H, t_q, order_d, hmask, valid,
                                                           coef[0], coef[1], coef[2], coef[3], out);
}

void launch_cache_push(const __nv_bfloat16* o, __nv_bfloat16* cache, int32_t* valid, int S, int H,
                       int t_q, int order_d, const uint8_t* sel, int one_tile, cudaStream_t stream) {
  note_launch();
  cache_push_kernel<<<one_tile >= 0 ? 1 : H * t_q, 256, 0, stream>>>(o, cache, valid, S, H, t_q,
                                                                     order_d, sel, one_tile);
}

}  // namespace fo
