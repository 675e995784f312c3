// DFMA throughput / latency and fp32->fp64 conversion rate on one B200
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/fp64_rate tools/fp64_rate.cu)
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dfma(double* out, double a, double b, int iters) {
  double acc[CH];
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  double s = 0; for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}
__global__ void dadd_cvt(double* out, const float* x, int iters) {
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  float f = x[threadIdx.x];
  for (int it = 0; it < iters; ++it) { a0 += (double)f; a1 += (double)(f+1.f); a2 += (double)(f+2.f); a3 += (double)(f+3.f); f += 0.5f; }
  if (a0 + a1 + a2 + a3 == 12345.0) out[0] = a0;
}
int main() {
  double* o; cudaMalloc(&o, 8); float* x; cudaMalloc(&x, 4096); cudaMemset(x, 0, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; float ms;
  for (int rep = 0; rep < 2; ++rep) {
  cudaEventRecord(e0); dfma<8><<<148 * 8, 256>>>(o, 1.0000001, 1e-9, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA 8 chains: %.1f DFMA/clk/SM at 1.9GHz (%.3f ms, %.2f TFLOP/s)\n", 148.0*8*256*8*iters/(ms*1e-3)/148/1.9e9, ms, 2.0*148*8*256*8*iters/(ms*1e-3)/1e12);
  cudaEventRecord(e0); dfma<1><<<148 * 8, 256>>>(o, 1.0000001, 1e-9, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA 1 chain, 64 warps/SM: %.2f DFMA/clk/SM (%.3f ms)\n", 148.0*8*256*iters/(ms*1e-3)/148/1.9e9, ms);
  cudaEventRecord(e0); dfma<1><<<148, 32>>>(o, 1.0000001, 1e-9, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA latency: %.1f cycles\n", ms*1e-3*1.9e9/iters);
  cudaEventRecord(e0); dadd_cvt<<<148 * 8, 256>>>(o, x, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cvt+DADD: %.1f (cvt+add)/clk/SM\n", 148.0*8*256*4*iters/(ms*1e-3)/148/1.9e9);
  }
}
