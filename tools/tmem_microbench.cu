// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM (sm_100a). Not part of the product.
#include <cstdio>
#include "../paper_2509_25401_b200/csrc/fo_common.cuh"
using namespace fo;

template <int MODE>  // 0: ld x32 + wait each, 1: ld 4 x32 then wait, 2: st x32, 3: ld x32 with 2 warps/SMSP
__global__ void tm_bench(long long* out, float* sink, int iters) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[4][32];
    if (MODE == 0 || MODE == 3) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tb + c * 32 + (warp >> 2) * 128, r[c]);
        tmem_ld_wait();
        acc += __uint_as_float(r[c][c]);
      }
    } else if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tb + c * 32, r[c]);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += __uint_as_float(r[c][3 * c]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int k = 0; k < 32; ++k) r[c][k] = it + k;
        tmem_st32(tb + c * 32, r[c]);
      }
      tmem_st_wait();
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase_s);
  }
}

template <int MODE>
void run(const char* name, int threads, int iters) {
  long long* d;
  float* s;
  cudaMalloc(&d, 148 * 16 * sizeof(long long));
  cudaMalloc(&s, 148 * 1024 * sizeof(float));
  tm_bench<MODE><<<148, threads>>>(d, s, 10);
  tm_bench<MODE><<<148, threads>>>(d, s, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes_per_iter_warp = 4 * 32 * 32 * 4.0;  // 16 KB per warp per iter
  double cyc = h[0] / (double)iters;
  printf("%-34s %s  %.1f cycles/iter/warp  -> %.1f B/clk per warp, %.1f B/clk per SM\n", name,
         cudaGetErrorString(e), cyc, bytes_per_iter_warp / cyc, bytes_per_iter_warp / cyc * threads / 32);
  cudaFree(d);
  cudaFree(s);
}

int main() {
  run<0>("ld x32+wait, 4 warps", 128, 2000);
  run<1>("ld 4x32 then wait, 4 warps", 128, 2000);
  run<3>("ld x32+wait, 8 warps", 256, 2000);
  run<2>("st x32, 4 warps", 128, 2000);
  return 0;
}
