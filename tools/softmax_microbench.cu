// Microbenchmark: throughput of the attention tile softmax on one SMSP (sm_100a).
// Not part of the product. Each warp repeatedly runs the per-row softmax of a
// 128-column S tile exactly as the attention kernels do (TMEM load of S, row max,
// exp2 split MUFU / FMA polynomial, bf16 pack, TMEM store of P), with 1 or 2
// warps per SMSP, to find which part bounds it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/smx tools/softmax_microbench.cu
#include <cstdio>

#include "../paper_2509_25401_b200/csrc/fo_common.cuh"
using namespace fo;

template <int N>
__device__ __forceinline__ void rfence(uint32_t (&r)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) asm volatile("" : "+r"(r[k]));
}

// V: 0 full (max, split exp 2/8 poly, row sum, pack), 1 no row sum, 2 MUFU only,
//    3 poly only, 4 max only (no exp), 5 exp only (no max), 6 ld/st only
// PF: poly pairs of every 8 (V 0/1/5); IPACK: integer round-to-nearest bf16 pack
// (IADD + PRMT on the ALU) instead of F2FP
__device__ __forceinline__ uint32_t ipack(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
  return __byte_perm(a, b, 0x7632);
}
template <int V, int PF = 2, bool IPACK = false>
__global__ void __launch_bounds__(256, 1) smx(long long* out, float* sink, int iters, float scale) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t sa = tbase_s + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 256;
  // seed S with something finite
  {
    uint32_t r[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(0.01f * (k + threadIdx.x % 7));
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st32(sa + c * 32, r);
    tmem_st_wait();
  }
  const float2 sc2 = make_float2(scale, scale);
  float2 l2 = make_float2(0.f, 0.f);
  float m_run = 0.f;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t u[4][32];
    tmem_ld32(sa + 0, u[0]);
    tmem_ld32(sa + 32, u[1]);
    tmem_ld32(sa + 64, u[2]);
    tmem_ld32(sa + 96, u[3]);
    tmem_ld_wait();
    rfence(u[0]);
    rfence(u[1]);
    rfence(u[2]);
    rfence(u[3]);
    float sv[128];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int k = 0; k < 32; ++k) sv[c * 32 + k] = __uint_as_float(u[c][k]);
    float m_new = m_run;
    if (V != 5 && V != 6) {
      float mc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float a = fmax3f(sv[16 * c], sv[16 * c + 1], sv[16 * c + 2]);
#pragma unroll
        for (int k = 3; k < 15; k += 2) a = fmax3f(a, sv[16 * c + k], sv[16 * c + k + 1]);
        mc[c] = fmaxf(a, sv[16 * c + 15]);
      }
      const float mx = fmax3f(fmax3f(mc[0], mc[1], mc[2]), fmax3f(mc[3], mc[4], mc[5]),
                              fmaxf(mc[6], mc[7]));
      m_new = fmaxf(m_run, mx * scale);
    }
    m_run = m_new;
    const float2 nm2 = make_float2(-m_new, -m_new);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e0 = c * 32 + 2 * q;
        float2 e;
        if (V == 4 || V == 6) {
          e = make_float2(sv[e0], sv[e0 + 1]);
        } else {
          const float2 x = ffma2(make_float2(sv[e0], sv[e0 + 1]), sc2, nm2);
          const bool poly = (V == 3) || ((V == 0 || V == 1 || V == 5) && ((c * 16 + q) & 7) < PF);
          if (poly) {
            e = exp2_poly2(x);
          } else {
            e.x = fast_exp2(x.x);
            e.y = fast_exp2(x.y);
          }
        }
        if (V == 0) l2 = fadd2(l2, e);
        pk[q] = IPACK ? ipack(e.x, e.y) : pack_bf16x2(e.x, e.y);
      }
      tmem_st16(sa + 128 + c * 16, pk);  // P into the other half (keeps S intact)
    }
    tmem_st_wait();
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = l2.x + l2.y + m_run;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase_s);
  }
}

template <int V, int PF = 2, bool IPACK = false>
void run(const char* name, int threads, int iters) {
  long long* d;
  float* s;
  cudaMalloc(&d, 148 * 8 * sizeof(long long));
  cudaMalloc(&s, 148 * 256 * sizeof(float));
  smx<V, PF, IPACK><<<148, threads>>>(d, s, 10, 0.1f);
  smx<V, PF, IPACK><<<148, threads>>>(d, s, iters, 0.1f);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  int nw = threads / 32;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < nw; ++w) avg += h[b * 8 + w];
  avg /= 148.0 * nw * iters;
  printf("%-28s warps/SMSP=%d  cycles/tile/warp=%7.1f  per-SMSP cycles/tile=%7.1f  %s\n", name,
         nw / 4, avg, avg / (nw / 4), e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(s);
}

int main() {
  const int it = 2000;
  for (int t : {128, 256}) {
    run<1, 2, false>("no row sum, poly2, F2FP", t, it);
    run<1, 2, true>("no row sum, poly2, ipack", t, it);
    run<1, 3, false>("no row sum, poly3, F2FP", t, it);
    run<1, 3, true>("no row sum, poly3, ipack", t, it);
    run<1, 4, true>("no row sum, poly4, ipack", t, it);
    run<0, 2, true>("row sum, poly2, ipack", t, it);
    run<0, 3, true>("row sum, poly3, ipack", t, it);
    run<6, 2, false>("ld/st + F2FP pack", t, it);
    run<6, 2, true>("ld/st + ipack", t, it);
    run<2, 0, true>("MUFU-only, ipack", t, it);
  }
  return 0;
}
