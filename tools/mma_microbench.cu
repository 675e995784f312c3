// Microbenchmark: tcgen05.mma throughput per operand source / shape on sm_100a.
// Not part of the product; used to choose tile shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_microbench.cu
#include <cstdio>

#include "../paper_2509_25401_b200/csrc/fo_common.cuh"

using namespace fo;

template <int MODE>  // 0: SS N128, 1: SS N256, 2: TS N128, 3: TS N256, 4: SS N128 + TMA-free smem writes
__global__ void __launch_bounds__(128, 1) mma_bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  constexpr int N = (MODE == 1 || MODE == 3) ? 256 : 128;
  const uint32_t idesc = make_idesc_bf16(128, N, false, false);
  const uint32_t a = smem_u32(smem), b = a + 32768;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = make_sdesc_sw128(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        if (MODE <= 1 || MODE == 4) {
          const uint64_t ad = make_sdesc_sw128(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          mma_bf16_ss(tbase + 256, ad, bd, idesc, 1);
        } else {
          mma_bf16_ts(tbase + 256, tbase + k * 8, bd, idesc, 1);
        }
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (MODE == 4 && threadIdx.x >= 32) {
    // competing generic smem writes (~TMA-like traffic) into a separate region
    uint4* p = reinterpret_cast<uint4*>(smem + 98304);
    for (int it = 0; it < iters * 64; ++it) p[(threadIdx.x + it * 96) & 4095] = make_uint4(it, it, it, it);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int MODE>
void run(const char* name, int iters) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(mma_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  mma_bench<MODE><<<148, 128, 180 * 1024>>>(d, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_bench<MODE><<<148, 128, 180 * 1024>>>(d, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const int N = (MODE == 1 || MODE == 3) ? 256 : 128;
  const double mmas = 8.0 * iters;
  const double flops = 2.0 * 128 * N * 16 * mmas * 148;
  printf("%-28s %s cycles/MMA %.1f  (ideal %d)  %.0f TFLOP/s\n", name, cudaGetErrorString(err),
         avg / mmas, N / 2, flops / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  const int iters = 20000;
  run<0>("SS M128 N128 K16", iters);
  run<1>("SS M128 N256 K16", iters);
  run<2>("TS M128 N128 K16", iters);
  run<3>("TS M128 N256 K16", iters);
  run<4>("SS M128 N128 + st.shared", iters / 4);
  return 0;
}
