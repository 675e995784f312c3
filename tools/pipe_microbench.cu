// Which pipe does the bf16x2 pack (F2FP) share? Throughput per SM of MUFU.EX2,
// cvt.rn.bf16x2.f32, PRMT, and MUFU + F2FP mixed (8 independent chains / thread).
#include <cstdio>
template <int MODE>
__global__ void k(unsigned* out, long long* cyc, int iters) {
  float f[8];
  unsigned u[8];
  for (int i = 0; i < 8; ++i) { f[i] = 0.5f + threadIdx.x * 1e-3f + i; u[i] = threadIdx.x + i; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // MUFU only
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      } else if (MODE == 1) {  // F2FP only
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(f[i]), "f"(__uint_as_float(u[i])));
      } else if (MODE == 2) {  // MUFU + F2FP (one each)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(f[i]), "f"(__uint_as_float(u[i])));
      } else {  // PRMT pack (truncation)
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(u[i]) : "r"(__float_as_uint(f[i])), "r"(u[i]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= u[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2", "F2FP.BF16 pack", "MUFU+F2FP", "PRMT pack"};
  int iters = 4096;
  for (int mode = 0; mode < 4; ++mode) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 512>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, 512>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, 512>>>(out, cyc, iters);
      if (mode == 3) k<3><<<148, 512>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    double warp_instr = 512.0 / 32 * iters * 8 * (mode == 2 ? 2 : 1);
    printf("%-16s %.3f warp-instr/clk/SM  (%.1f lanes/clk)\n", names[mode], warp_instr / h,
           warp_instr * 32 / h);
  }
  return 0;
}
