// MUFU ex2 throughput per SM: f32 vs packed f16x2 / bf16x2 (8 independent chains per thread)
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
template <int MODE>
__global__ void k(unsigned* out, long long* cyc, int iters) {
  unsigned v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x * 8 + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        float f = __uint_as_float(v[i]);
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f));
        v[i] = __float_as_uint(f) & 0x807fffffu | 0x3e000000u;
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
        v[i] = (v[i] & 0x83ff83ffu) | 0x38003800u;
      } else {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
        v[i] = (v[i] & 0x807f807fu) | 0x3e003e00u;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int threads : {256, 512, 1024}) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, threads>>>(out, cyc, iters);
        if (mode == 1) k<1><<<148, threads>>>(out, cyc, iters);
        if (mode == 2) k<2><<<148, threads>>>(out, cyc, iters);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      double ops = (double)threads * iters * 8 * (mode ? 2 : 1);  // exps per SM
      printf("mode %d (%s) threads %d: %.2f exps/clk/SM (%s)\n", mode,
             mode == 0 ? "f32" : mode == 1 ? "f16x2" : "bf16x2", threads, ops / h,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
