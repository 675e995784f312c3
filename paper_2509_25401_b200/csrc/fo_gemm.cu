// K3 GEMM-Q and K4/K5 GEMM-O on sm_100a (tcgen05 + TMEM + TMA, persistent).
//
// GEMM-Q (reference gemm.py:44-93 + tensor.py:68-109): output tile = (query
// block i, head h), 128 x 128, so RMSNorm over the head dim and the
// interleaved-pair RoPE are tile-local and run in the epilogue. Tiles whose
// cache symbol is 0 are never scheduled (the plan lists only active tiles).
//
// GEMM-O (gemm.py:110-229): output tile = (block i, 128 columns of d_model);
// the K loop walks heads, 128 K-columns each.
//   dispatch: only heads active for block i are multiplied; the epilogue adds
//             sum_d c_d * B_c[d] (the forecast of the cached-head bias).
//   update:   job (i, n, d). d=0 accumulates cached heads (their cache stack 0)
//             into accumulator B and active heads (o) into accumulator A in one
//             K pass; B -> B_c[0],
//             A + B -> out. d>=1 projects the cached heads' d-th difference
//             stacks into B_c[d]. Every head is projected exactly once.
// Warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4..7 epilogue
// (one accumulator row per thread). TMEM accumulators are double-buffered so
// the epilogue of tile t overlaps the mainloop of tile t+1.
#include <algorithm>

#include "fo_internal.cuh"

// GEMM-O dispatch: the bias stream and the output are touched once, so they go
// through L2 as evict-first and leave W and o (re-read by every row block) in L2
#ifndef FO_GO_EVICT_FIRST
#define FO_GO_EVICT_FIRST 1
#endif
#ifndef FO_GO_EF_LOAD
#define FO_GO_EF_LOAD 0  // dispatch bias loads evict-first (measured slower without the L2 prefetch)
#endif
#ifndef FO_GO_EF_STORE
#define FO_GO_EF_STORE FO_GO_EVICT_FIRST  // dispatch out stores evict-first
#endif
#ifndef FO_GU_EL_W
#define FO_GU_EL_W 0  // update: W loads evict-last
#endif
#ifndef FO_GU_EF_STORE
#define FO_GU_EF_STORE 1  // update: out / B_c stores evict-first
#endif
#ifndef FO_GO_EL_OPS
#define FO_GO_EL_OPS 1  // dispatch o / W operand loads evict-last
#endif

#ifndef FO_GO_PF
#define FO_GO_PF 0  // GEMM-O dispatch: bias L2 prefetch distance in jobs (0: none; 1 re-read 13-17% of the bias from DRAM)
#endif

namespace fo {
namespace gemm {
constexpr int BM = 128, BN = 128, BK = 64;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STAGES = 6;
constexpr int NTHREADS = 256;

// GEMM-O dispatch: 128 x 256 output tiles (N=256 halves the W/A feed per MMA
// cycle relative to N=128 for A), 3 stages of 48 KB, and a ring of bias /
// output chunks (128 rows x 32 columns, orders 0 and 1, SW64) between the
// bias-loader warp, the epilogue and the TMA store
constexpr int D_BN = 256;
constexpr int D_STAGE_BYTES = A_BYTES + 2 * B_BYTES;  // 48 KB
#ifndef FO_GO_DST
#define FO_GO_DST 3
#endif
#ifndef FO_GO_RING
#define FO_GO_RING 4  // bias ring in 16 KB units
#endif
#ifndef FO_GO_OST
#define FO_GO_OST 2  // output staging buffers
#endif
constexpr int D_STAGES = FO_GO_DST;
constexpr int BIAS_SLOTS = 2 * FO_GO_RING;  // max slots (8 KB each at order 0, 16 KB at orders >= 1)
constexpr int OST = FO_GO_OST;
constexpr int BIAS_ORDER_BYTES = BM * 32 * 2;  // 8 KB
constexpr int BIAS_SLOT_BYTES = 2 * BIAS_ORDER_BYTES;

struct Bars {
  uint64_t full[STAGES], empty[STAGES];
  uint64_t tfull[2], tempty[2];
  uint64_t bfull[BIAS_SLOTS], bempty[BIAS_SLOTS];
  uint32_t tmem_base;
};
// output chunks are staged separately (double-buffered) so a bias slot is free
// as soon as the epilogue has read it, not when the chunk's store has read it
constexpr int OUT_STAGE_BYTES = BM * 32 * 2;  // 8 KB, SW64 like the bias chunks
constexpr int BIAS_RING_BYTES = FO_GO_RING * BIAS_SLOT_BYTES;  // 64 KB
constexpr int SMEM_BYTES_D = D_STAGES * D_STAGE_BYTES + BIAS_RING_BYTES +
                             OST * OUT_STAGE_BYTES + 1024 + (int)sizeof(Bars);
static_assert(SMEM_BYTES_D <= 232448, "dispatch shared memory over the sm_100 limit");

// empty_count: consumers that release a stage (2 when the A tile is multicast
// across a CTA pair: both MMA warps must be done before either producer refills)
__device__ __forceinline__ void init_bars(Bars* b, uint32_t empty_count = 1,
                                          uint32_t bias_consumers = 1) {
  for (int s = 0; s < STAGES; ++s) {
    mbar_init(&b->full[s], 1);
    mbar_init(&b->empty[s], empty_count);
  }
  for (int a = 0; a < 2; ++a) {
    mbar_init(&b->tfull[a], 1);
    mbar_init(&b->tempty[a], 128);
  }
  for (int a = 0; a < BIAS_SLOTS; ++a) {
    mbar_init(&b->bfull[a], 1);
    mbar_init(&b->bempty[a], bias_consumers);
  }
  fence_barrier_init();
}

// ring-buffer cursor
template <int NS = STAGES>
struct Ring {
  int s = 0, ph = 0;
  __device__ __forceinline__ void next() {
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
};

// ring cursor over a runtime slot count
struct DynRing {
  int s = 0, ph = 0, n;
  __device__ explicit DynRing(int n_) : n(n_) {}
  __device__ __forceinline__ void next() {
    if (++s == n) {
      s = 0;
      ph ^= 1;
    }
  }
};

// issue one BK=64 k-block: 4 x (128x128x16) MMAs from warp-uniform descriptors
// (K-chunk k of a SW128 K-major tile starts 32 B = 2 descriptor units further)
__device__ __forceinline__ void mma_kblock(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, bool acc_in) {
#pragma unroll
  for (int k = 0; k < BK / 16; ++k)
    mma_bf16_ss(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (acc_in || k > 0) ? 1u : 0u);
}

template <int N>
__device__ __forceinline__ void reg_fence(uint32_t (&r)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) asm volatile("" : "+r"(r[k]));
}

// 32 bf16 of one row (64 B, 32-B aligned) as two 256-bit stores
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4 pk[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    pk[q].x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
    pk[q].y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
    pk[q].z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
    pk[q].w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
  }
  st_global_256(dst, pk[0], pk[1]);
  st_global_256(dst + 16, pk[2], pk[3]);
}
}  // namespace gemm

// launch a persistent kernel as 2-CTA clusters, as many as can be co-resident
template <typename Kernel, typename... Args>
static void launch_pair_clusters_max(Kernel kernel, int smem, int* grid_cache, int max_ctas,
                                     cudaStream_t stream, Args... args);
template <typename Kernel, typename... Args>
static void launch_pair_clusters(Kernel kernel, int smem, int* grid_cache, cudaStream_t stream,
                                 Args... args) {
  launch_pair_clusters_max(kernel, smem, grid_cache, 1 << 30, stream, args...);
}
// max_ctas < the co-resident grid leaves SMs free for a concurrent kernel (the
// all-reduce of the previous row chunk)
template <typename Kernel, typename... Args>
static void launch_pair_clusters_max(Kernel kernel, int smem, int* grid_cache, int max_ctas,
                                     cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // FO_PDL (fo_common.cuh)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(gemm::NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (*grid_cache == 0) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 0, clusters = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3(sms & ~1);
    if (cudaOccupancyMaxActiveClusters(&clusters, kernel, &cfg) != cudaSuccess || clusters < 1)
      clusters = sms / 2;
    *grid_cache = 2 * std::min(clusters, sms / 2);
  }
  cfg.gridDim = dim3(std::max(2, std::min(*grid_cache, max_ctas & ~1)));
  cfg.numAttrs = FO_PDL ? 2 : 1;
  note_launch();
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// =============================================================================
// GEMM-Q: output tile = (query block i, head h), 128 x 128, so RMSNorm over the
// head dim and RoPE are tile-local; each head's 128 accumulator columns get
// them in the epilogue. The kernel (gemm_q2_kernel below) runs on CTA pairs.
// =============================================================================
namespace gemm {
constexpr int Q_BN = 256;
constexpr int Q_NW_BYTES = 64 * 128 * 4;  // RMSNorm weights of up to 64 heads
}  // namespace gemm

namespace gemm {
// GEMM-Q epilogue of one job for accumulator row r (one thread per row):
// pass 1 reads both heads' rows from TMEM for the RMS sums; pass 2 walks
// 32-column chunks, loading the row's rotary chunk once for both heads
// (prefetched a chunk ahead) and the norm weights from shared memory.
// release() hands the accumulator back to the MMA warp after its last read.
// Per projection (segment): out is its [S, H*128] output, norm / rope its
// epilogue (Q, K: RMSNorm + RoPE; V: plain), nw_u32 its norm weights' smem.
template <typename Release>
__device__ __forceinline__ void q_epilogue_job(const GemmQParams& p, uint32_t ta0, int r, int i,
                                               int h1, int h2, uint32_t nw_u32,
                                               __nv_bfloat16* out, bool norm, bool rope,
                                               Release release) {
  const size_t HD = (size_t)p.H * 128;
  const int row = i * BM + r;
  const bool row_ok = row < p.S;
  const int nh = h2 >= 0 ? 2 : 1;
  float inv[2] = {1.f, 1.f};
  if (norm) {
    // RMSNorm (tensor.py:68-80): y * w / sqrt(mean(y^2) + eps)
    for (int sl = 0; sl < nh; ++sl) {
      float ss = 0.f;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t u[32];
        tmem_ld32(ta0 + sl * BN + cc * 32, u);
        tmem_ld_wait();
        gemm::reg_fence(u);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float v = __uint_as_float(u[k]);
          ss = fmaf(v, v, ss);
        }
      }
      inv[sl] = rsqrtf(ss * (1.f / 128.f) + p.eps);
    }
  }
  const float4* cs4 = rope ? reinterpret_cast<const float4*>(p.rope_cos + (size_t)row * 64)
                           : nullptr;
  const float4* sn4 = rope ? reinterpret_cast<const float4*>(p.rope_sin + (size_t)row * 64)
                           : nullptr;
  float4 cn[4], sx[4];  // rotary chunk in flight (16 cos + 16 sin)
  if (rope && row_ok) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cn[q] = __ldg(cs4 + q);
      sx[q] = __ldg(sn4 + q);
    }
  }
#pragma unroll 1
  for (int cc = 0; cc < 4; ++cc) {
    float cvv[16], svv[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cvv[4 * q] = cn[q].x; cvv[4 * q + 1] = cn[q].y; cvv[4 * q + 2] = cn[q].z; cvv[4 * q + 3] = cn[q].w;
      svv[4 * q] = sx[q].x; svv[4 * q + 1] = sx[q].y; svv[4 * q + 2] = sx[q].z; svv[4 * q + 3] = sx[q].w;
    }
    if (rope && row_ok && cc < 3) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cn[q] = __ldg(cs4 + (cc + 1) * 4 + q);
        sx[q] = __ldg(sn4 + (cc + 1) * 4 + q);
      }
    }
    for (int sl = 0; sl < nh; ++sl) {
      const int h = sl ? h2 : h1;
      uint32_t u[32];
      tmem_ld32(ta0 + sl * BN + cc * 32, u);
      tmem_ld_wait();
      gemm::reg_fence(u);
      if (cc == 3 && sl == nh - 1) release();  // accumulator drained
      if (!row_ok) continue;
      float o[32];
      if (!norm) {
        // plain projection (V): no normalisation, no rotary encoding
#pragma unroll
        for (int k = 0; k < 32; ++k) o[k] = __uint_as_float(u[k]);
      } else {
        float wv[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // broadcast reads: every thread, same address
          const uint4 w4 = lds128(nw_u32 + (uint32_t)((h * 128 + cc * 32 + 4 * q) * 4));
          wv[4 * q] = __uint_as_float(w4.x); wv[4 * q + 1] = __uint_as_float(w4.y);
          wv[4 * q + 2] = __uint_as_float(w4.z); wv[4 * q + 3] = __uint_as_float(w4.w);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          // interleaved-pair RoPE (tensor.py:83-109)
          const float e = __uint_as_float(u[2 * k]) * wv[2 * k] * inv[sl];
          const float od = __uint_as_float(u[2 * k + 1]) * wv[2 * k + 1] * inv[sl];
          if (rope) {
            const float cv = cvv[k], sv = svv[k];
            o[2 * k] = e * cv - od * sv;
            o[2 * k + 1] = e * sv + od * cv;
          } else {
            o[2 * k] = e;
            o[2 * k + 1] = od;
          }
        }
      }
      gemm::store_bf16x32(out + (size_t)row * HD + (size_t)h * 128 + cc * 32, o);
    }
  }
}
}  // namespace gemm

// =============================================================================
// GEMM-Q on CTA pairs (cta_group::2), every tile of both phases in one
// persistent launch. A cluster job is two query blocks (i0 on CTA 0, i1 on
// CTA 1) x one N-tile of heads, one M=256 tcgen05 tile over both SMs:
//   N=256: heads (h, h+1) active in both blocks; each CTA loads its 128 x rows
//          and its own head's 128 W rows per k-block (B is split by CTA);
//   N=128: head h alone; each CTA loads its 128 x rows and 64 of h's W rows.
// The even CTA issues the MMAs, which read both CTAs' shared memory and write
// each CTA's 128 accumulator rows to its own TMEM. Per SM the operand feed is
// 64 B per MMA cycle (N=256) or 96 B (N=128), against 128 B for a 1-CTA
// 128 x 128 tile. The dense phase walks (block pair, head pair) jobs in place
// (plus an N=128 job per block pair for an odd last head); the sparse phase
// walks the plan's job list (PlanView::gq_jobs), which is ordered by first
// block so jobs in flight share x tiles in L2. A job with one block loads
// zero rows past the end on CTA 1 (TMA fills them) and skips its epilogue.
// =============================================================================
namespace gemm {
constexpr int Q2_STAGE_BYTES = A_BYTES + B_BYTES;  // 32 KB per CTA
constexpr int Q2_STAGES = 6;
constexpr int Q2_SMEM_BYTES = Q2_STAGES * Q2_STAGE_BYTES + 1024 + 1024 + Q_NW_BYTES;
static_assert(Q2_SMEM_BYTES <= 232448, "2-CTA GEMM-Q shared memory over the sm_100 limit");
}  // namespace gemm

__global__ void __launch_bounds__(gemm::NTHREADS, 1)
    gemm_q2_kernel(const __grid_constant__ CUtensorMap xm,    // x, box 64 K x 128 rows
                   const __grid_constant__ CUtensorMap wm,    // W_q, box 64 K x 128 rows
                   const __grid_constant__ CUtensorMap wm64,  // W_q, box 64 K x 64 rows
                   const GemmQParams p) {
  using namespace gemm;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + Q2_STAGES * Q2_STAGE_BYTES);
  float* nw_smem = reinterpret_cast<float*>(smem + Q2_STAGES * Q2_STAGE_BYTES + 1024);
  const int warp = warp_id(), lane = lane_id();
  const int rank = (int)cluster_ctarank();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bars->full[s], 1);   // the even CTA's producer arrives (tx from both CTAs)
      mbar_init(&bars->empty[s], 1);  // the pair's MMA commit reaches both CTAs
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bars->tfull[a], 1);
      mbar_init(&bars->tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
    tma_prefetch_desc(&xm);
    tma_prefetch_desc(&wm);
    tma_prefetch_desc(&wm64);
  }
  if (warp == 2) tmem_alloc_2sm<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  pdl_release_and_wait();
  if (p.norm_w || (p.qkv && p.k_norm)) {
    // Q's norm weights at heads [0, H), K's (fused launch) at [H, 2H)
    for (int e = threadIdx.x; e < p.H * 32; e += blockDim.x) {
      if (p.norm_w)
        reinterpret_cast<float4*>(nw_smem)[e] = __ldg(reinterpret_cast<const float4*>(p.norm_w) + e);
      if (p.qkv && p.k_norm)
        reinterpret_cast<float4*>(nw_smem)[p.H * 32 + e] =
            __ldg(reinterpret_cast<const float4*>(p.k_norm) + e);
    }
    __syncthreads();
  }
  const uint32_t tbase = bars->tmem_base;
  const int nph = p.H >> 1;            // full head pairs
  const int npj = nph + (p.H & 1);     // dense jobs per block pair (odd last head: N=128)
  const int nbp = (p.t_q + 1) >> 1;    // block pairs
  // fused launch: the dense K and V jobs (block-pair-major, K then V head pairs
  // of each block pair) come first, then Q's (dense or the plan's sparse list)
  const int n_kv = p.qkv ? 2 * nbp * npj : 0;
  const int n_cjobs = n_kv + (p.dense ? nbp * npj : *p.n_jobs);
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // round rr of cluster cid takes job rr*ncl + cid, snaking (reversed on odd
  // rounds): the plan lists the sparse jobs by cost class (N = 256, then
  // N = 128 pairs, then single-block jobs), so clusters that drew a heavy job
  // in one round draw a light one in the next
  auto job_of = [&](int rr) { return rr * ncl + ((rr & 1) ? ncl - 1 - cid : cid); };
  const int nkb = p.dm / BK;
  // job -> this CTA's block i, head h and width (n256: heads h, h2 as one N=256
  // tile); false: no block for this CTA (it loads zero rows past the end and
  // skips its epilogue). seg: 0 Q, 1 K, 2 V (rows seg*H*128.. of the fused weight)
  auto job = [&](int c, int& i, int& h, int& h2, bool& n256, int& seg) -> bool {
    int i0, i1;
    seg = 0;
    if (c < n_kv) {  // fused K / V: block-pair-major, then K / V, then head pair
      const int bp = c / (2 * npj), r2 = c - bp * 2 * npj, r = r2 % npj;
      seg = 1 + r2 / npj;
      i0 = 2 * bp;
      i1 = 2 * bp + 1 < p.t_q ? 2 * bp + 1 : -1;
      h = 2 * r;
      n256 = r < nph;
      h2 = h + 1;
    } else if (p.dense) {  // block-pair-major
      c -= n_kv;
      const int bp = c / npj, r = c - bp * npj;
      i0 = 2 * bp;
      i1 = 2 * bp + 1 < p.t_q ? 2 * bp + 1 : -1;
      h = 2 * r;
      n256 = r < nph;
      h2 = h + 1;
    } else {
      const int2 code = p.jobs[c - n_kv];
      i0 = code.x & 0xFFFF;
      i1 = (code.x >> 16) - 1;
      h = code.y & 0xFF;
      n256 = (code.y >> 8) & 1;
      h2 = (code.y >> 16) & 0xFF;  // any head (heads paired per block by the plan)
    }
    i = rank ? (i1 >= 0 ? i1 : p.t_q) : i0;
    return rank == 0 || i1 >= 0;
  };

  if (warp == 0) {
    // both CTAs load their own x rows and their half of B; the bytes of both
    // land on the even CTA's full barrier
    Ring<Q2_STAGES> rg;
    for (int rr = 0; rr * ncl < n_cjobs; ++rr) {
      const int c = job_of(rr);
      if (c >= n_cjobs) continue;
      int i, h, h2, seg;
      bool n256;
      job(c, i, h, h2, n256, seg);  // a missing block loads zero rows (coordinates past the end)
      const uint32_t b_bytes = n256 ? B_BYTES : B_BYTES / 2;
      h += seg * p.H;  // the projection's rows of the (fused) weight
      h2 += seg * p.H;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&bars->empty[rg.s], rg.ph ^ 1);
        if (elect_one()) {
          uint8_t* st = smem + rg.s * Q2_STAGE_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&bars->full[rg.s], 2 * (A_BYTES + b_bytes));
          tma_load_2d_2sm(st, &xm, &bars->full[rg.s], kb * BK, i * BM);
          if (n256)
            tma_load_2d_2sm(st + A_BYTES, &wm, &bars->full[rg.s], kb * BK, (rank ? h2 : h) * BN);
          else
            tma_load_2d_2sm(st + A_BYTES, &wm64, &bars->full[rg.s], kb * BK, h * BN + rank * 64);
        }
        __syncwarp();
        rg.next();
      }
    }
  } else if (warp == 1 && rank == 0) {
    // MMA issuer of the pair
    const uint32_t idesc256 = make_idesc_bf16(2 * BM, Q_BN, false, false);
    const uint32_t idesc128 = make_idesc_bf16(2 * BM, BN, false, false);
    const uint64_t desc0 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
    Ring<Q2_STAGES> rg;
    int t = 0;
    for (int rr = 0; rr * ncl < n_cjobs; ++rr) {
      const int c = job_of(rr);
      if (c >= n_cjobs) continue;
      int i, h, h2, seg;
      bool n256;
      job(c, i, h, h2, n256, seg);
      const uint32_t idesc = n256 ? idesc256 : idesc128;
      const int acc = t & 1;
      mbar_wait(&bars->tempty[acc], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tbase + acc * Q_BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&bars->full[rg.s], rg.ph);
        tc_fence_after();
        const uint64_t a = desc0 + (uint64_t)((rg.s * Q2_STAGE_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss_2sm(d, a + 2 * k, a + (A_BYTES >> 4) + 2 * k, idesc,
                            (kb > 0 || k > 0) ? 1u : 0u);
          tc_commit_2sm_mc(&bars->empty[rg.s], 0x3);
        }
        __syncwarp();
        rg.next();
      }
      if (elect_one()) tc_commit_2sm_mc(&bars->tfull[acc], 0x3);
      __syncwarp();
      ++t;
    }
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t nw_u32 = smem_u32(nw_smem);
    int t = 0;
    for (int rr = 0; rr * ncl < n_cjobs; ++rr) {
      const int c = job_of(rr);
      if (c >= n_cjobs) continue;
      int i, h, h2, seg;
      bool n256;
      const bool mine = job(c, i, h, h2, n256, seg);
      const int acc = t & 1;
      mbar_wait(&bars->tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&bars->tempty[acc], 0);
      };
      if (mine) {
        __nv_bfloat16* out = seg == 0 ? p.q : (seg == 1 ? p.k_out : p.v_out);
        const bool norm = seg == 0 ? p.norm_w != nullptr : (seg == 1 && p.k_norm != nullptr);
        const bool rope = seg < 2 && p.rope_cos != nullptr;
        gemm::q_epilogue_job(p, tbase + lane_off + acc * Q_BN, r, i, h, n256 ? h2 : -1,
                             nw_u32 + (seg == 1 ? p.H * 128 * 4 : 0), out, norm, rope, release);
      }
      else
        release();
      ++t;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tbase);
  }
}

void launch_gemm_q2(const CUtensorMap& xm, const CUtensorMap& wm, const CUtensorMap& wm64,
                    const GemmQParams& p, cudaStream_t stream) {
  static int grid = 0;
  launch_pair_clusters(gemm_q2_kernel, gemm::Q2_SMEM_BYTES, &grid, stream, xm, wm, wm64, p);
}

// =============================================================================
// GEMM-O (update: UPDATE=true, dispatch: UPDATE=false)
// =============================================================================
// Dispatch epilogue data path: the forecast bias is HBM traffic the size of the
// output per order, so it moves as TMA tiles, not per-thread row loads (a warp
// of row-per-thread 16-B loads touches 32 rows = 32 L1 wavefronts). Warp 3
// streams 128 x 32 bias chunks (orders 0/1, SW64) into a 4-slot ring and pulls
// the next job's tiles into L2; each epilogue thread reads its row's chunk
// conflict-free from the swizzled slot, adds the accumulator, writes bf16 back
// in place and one elected thread TMA-stores the chunk to `out`.
template <bool UPDATE>
__global__ void __launch_bounds__(gemm::NTHREADS, 1)
    gemm_o_kernel(const __grid_constant__ CUtensorMap am,  // o   [S, H*128]
                  const __grid_constant__ CUtensorMap cm,  // update: diff stacks [(D+1)*S, H*128]
                                                           // dispatch: bias [(D+1)*S, dm], 32x128 SW64
                  const __grid_constant__ CUtensorMap wm,  // W_out^T [dm, H*128]
                  const __grid_constant__ CUtensorMap om,  // dispatch: out [S, dm], 32x128 SW64
                  const GemmOParams p) {
  using namespace gemm;
  constexpr int ST = UPDATE ? STAGES : D_STAGES;
  constexpr int SB = UPDATE ? STAGE_BYTES : D_STAGE_BYTES;  // bytes per stage
  constexpr int TBN = UPDATE ? BN : D_BN;                     // output tile columns
  constexpr int ACC_COLS = UPDATE ? 2 * BN : D_BN;  // update: accumulator A (active) + B (cached)
  constexpr int TM_COLS = 512;
  // dispatch runs as 2-CTA clusters: both CTAs take the same block i (hence the
  // same K sequence of active heads) and neighbouring 256-column n-tiles; each
  // loads half of the o tile and multicasts it to both
  constexpr bool MC = !UPDATE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* ring = smem + ST * SB;  // dispatch bias / output chunks
  uint8_t* ostage = ring + (UPDATE ? 0 : BIAS_RING_BYTES);  // dispatch out chunks
  Bars* bars = reinterpret_cast<Bars*>(ostage + (UPDATE ? 0 : OST * OUT_STAGE_BYTES));
  const int warp = warp_id(), lane = lane_id();
  const int rank = MC ? (int)cluster_ctarank() : 0;
  if (warp == 0 && lane == 0) {
    init_bars(bars, MC ? 2 : 1, 4);  // bias slots: released by each epilogue warp
    tma_prefetch_desc(&am);
    tma_prefetch_desc(&cm);
    tma_prefetch_desc(&wm);
    if (!UPDATE) tma_prefetch_desc(&om);
  }
  if (warp == 2) tmem_alloc<TM_COLS>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync();  // both CTAs' barriers exist before any multicast lands
  tc_fence_after();
  pdl_release_and_wait();
  const uint32_t tbase = bars->tmem_base;
  const int nbn = (p.dm + TBN - 1) / TBN;
  // columns of n-tile nb (dispatch: the last tile is 128 wide when dm % 256 != 0)
  auto tile_cols = [&](int nb) { return min(TBN, p.dm - nb * TBN); };
  const int nord = UPDATE ? p.order_d + 1 : 1;
  const int ncb = (nbn + 1) >> 1;  // dispatch: n-tile pairs per block (one per cluster job)
  const int n_jobs = MC ? (p.i_end - p.i_begin) * ncb : p.t_q * nbn * nord;
  const int jstart = MC ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int jstep = MC ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const unsigned long long all_heads = (p.H >= 64) ? ~0ull : ((1ull << p.H) - 1);
  // job decode, order-major (all d = 0 tiles first): the static round-robin over
  // CTAs then stays balanced when the d >= 1 jobs of blocks without cached heads
  // are skipped. Returns false for update jobs with no work (d >= orders[i]).
  // Dispatch: cluster job w = (block i, n-tile pair); false when this CTA's
  // n-tile is past the end (it still loads its half of the shared o tile).
  auto job = [&](int w, int& i, int& nb, int& d) -> bool {
    if (MC) {
      const int ib = w / ncb;
      i = p.i_begin + ib;
      nb = 2 * (w - ib * ncb) + rank;
      d = 0;
      return nb < nbn;
    }
    const int per = p.t_q * nbn;
    d = w / per;
    const int rest = w - d * per;
    nb = rest % nbn;
    i = rest / nbn;
    return !(UPDATE && d > 0 && d >= p.orders[i]);
  };
  // dispatch: bias orders staged through the ring for block i (orders >= 2 are
  // rare and read directly)
  auto staged_orders = [&](int i) { return min(min(p.order_d + 1, p.orders[i]), 2); };
  // the 64 KB bias ring holds 8 KB per staged order and chunk: 8 slots when
  // only order 0 is staged (twice the bytes in flight of a fixed 4-slot ring)
  const int bias_slot_bytes = min(p.order_d + 1, 2) * BIAS_ORDER_BYTES;
  const int bias_slots = BIAS_RING_BYTES / bias_slot_bytes;

  if (warp == 0) {
    {
      Ring<ST> rg;
      for (int w = jstart; w < n_jobs; w += jstep) {
        int i, nb, d;
        const bool mine = job(w, i, nb, d);
        if (!MC && !mine) continue;
        const unsigned long long act = p.hmask[i];
        const unsigned long long cached = all_heads & ~act;
        // K order: [cached heads (update only)] then [active heads (d == 0 only)]
        for (int pass = 0; pass < 2; ++pass) {
          unsigned long long m;
          if (pass == 0) m = UPDATE ? cached : 0ull;
          else m = (d == 0) ? act : 0ull;
          // cached heads read the cache's difference stack d, order 0 included
          // (gemm.py:155-161 projects entry.diff_stack[dd] for every dd)
          const CUtensorMap* src = (UPDATE && pass == 0) ? &cm : &am;
          const int row0 = (UPDATE && pass == 0) ? d * p.S + i * BM : i * BM;
          while (m) {
            const int h = __ffsll(m) - 1;
            m &= m - 1;
            const bool two = mine && tile_cols(nb) > BN;
            for (int kk = 0; kk < 2; ++kk) {
              mbar_wait(&bars->empty[rg.s], rg.ph ^ 1);
              if (elect_one()) {
                uint8_t* st = smem + rg.s * SB;
                mbar_arrive_expect_tx(&bars->full[rg.s],
                                      A_BYTES + (mine ? (two ? 2 : 1) * B_BYTES : 0));
#if FO_GO_EL_OPS
                const uint64_t pol = l2_evict_last_policy();
                if (MC)
                  tma_load_2d_mc_hint(st + rank * (A_BYTES / 2), src, &bars->full[rg.s],
                                      h * 128 + kk * BK, row0 + rank * (BM / 2), 0x3, pol);
                else
                  tma_load_2d_hint(st, src, &bars->full[rg.s], h * 128 + kk * BK, row0, pol);
                if (mine)
                  tma_load_2d_hint(st + A_BYTES, &wm, &bars->full[rg.s], h * 128 + kk * BK,
                                   nb * TBN, pol);
                if (two)
                  tma_load_2d_hint(st + A_BYTES + B_BYTES, &wm, &bars->full[rg.s],
                                   h * 128 + kk * BK, nb * TBN + BN, pol);
#else
                if (MC)
                  tma_load_2d_mc(st + rank * (A_BYTES / 2), src, &bars->full[rg.s],
                                 h * 128 + kk * BK, row0 + rank * (BM / 2), 0x3);
                else
                  tma_load_2d(st, src, &bars->full[rg.s], h * 128 + kk * BK, row0);
                if (mine)
                  tma_load_2d(st + A_BYTES, &wm, &bars->full[rg.s], h * 128 + kk * BK, nb * TBN);
                if (two)
                  tma_load_2d(st + A_BYTES + B_BYTES, &wm, &bars->full[rg.s], h * 128 + kk * BK,
                              nb * TBN + BN);
#endif
              }
              __syncwarp();
              rg.next();
            }
          }
        }
      }
      if (MC)  // drain: both CTAs' MMA warps have released every stage
        for (int k = 0; k < ST; ++k) {
          mbar_wait(&bars->empty[rg.s], rg.ph ^ 1);
          rg.next();
        }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      const uint32_t idesc1 = make_idesc_bf16(BM, BN, false, false);
      const uint32_t idesc2 = make_idesc_bf16(BM, 2 * BN, false, false);
      const uint64_t desc0 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
      Ring<ST> rg;
      int t = 0;
      for (int w = jstart; w < n_jobs; w += jstep) {
        int i, nb, d;
        const bool mine = job(w, i, nb, d);
        if (!MC && !mine) continue;
        const uint32_t idesc = (mine && tile_cols(nb) > BN) ? idesc2 : idesc1;
        const int acc = t & 1;
        if (mine) {
          mbar_wait(&bars->tempty[acc], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const unsigned long long act = p.hmask[i];
        const unsigned long long cached = all_heads & ~act;
        const uint32_t dA = tbase + acc * ACC_COLS;
        const uint32_t dB = dA + (UPDATE ? BN : 0);
        for (int pass = 0; pass < 2; ++pass) {
          int nk;
          if (pass == 0) nk = UPDATE ? 2 * __popcll(cached) : 0;
          else nk = (d == 0) ? 2 * __popcll(act) : 0;
          const uint32_t dst = (pass == 0) ? dB : dA;
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&bars->full[rg.s], rg.ph);
            tc_fence_after();
            const uint64_t a = desc0 + (uint64_t)((rg.s * SB) >> 4);
            if (elect_one()) {
              if (mine) mma_kblock(dst, a, a + (A_BYTES >> 4), idesc, kb > 0);
              if (MC)
                tc_commit_mc(&bars->empty[rg.s], 0x3);  // free in both CTAs' view
              else
                tc_commit(&bars->empty[rg.s]);
            }
            __syncwarp();
            rg.next();
          }
        }
        if (!mine) continue;
        if (elect_one()) tc_commit(&bars->tfull[acc]);
        __syncwarp();
        ++t;
      }
    }
    __syncwarp();
  } else if (!UPDATE && warp == 3) {
    // bias loader: 4 chunks per job through the slot ring, next job prefetched into L2
    DynRing rb(bias_slots);
    for (int w = jstart; w < n_jobs; w += jstep) {
      int i, nb, d;
      if (!job(w, i, nb, d)) continue;
      const int ns = staged_orders(i);
      const int nch = tile_cols(nb) / 32;
      // L2 prefetch FO_GO_PF jobs ahead: DRAM requests in flight beyond the ring
      auto prefetch = [&](int wn) {
        int i2, nb2, d2;
        if (wn < n_jobs && job(wn, i2, nb2, d2) && elect_one()) {
          const int ns2 = staged_orders(i2);
          for (int dd = 0; dd < ns2; ++dd)
            for (int c = 0; c < tile_cols(nb2) / 32; ++c)
              tma_prefetch_l2_2d(&cm, nb2 * TBN + c * 32, dd * p.S + i2 * BM);
        }
      };
      if (FO_GO_PF > 0) {
        if (w == jstart)
          for (int k = 1; k < FO_GO_PF; ++k) prefetch(w + k * jstep);
        prefetch(w + FO_GO_PF * jstep);
      }
      __syncwarp();
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&bars->bempty[rb.s], rb.ph ^ 1);
        if (elect_one()) {
          uint8_t* slot = ring + rb.s * bias_slot_bytes;
          mbar_arrive_expect_tx(&bars->bfull[rb.s], ns * BIAS_ORDER_BYTES);
          for (int dd = 0; dd < ns; ++dd)
#if FO_GO_EF_LOAD
            tma_load_2d_hint(slot + dd * BIAS_ORDER_BYTES, &cm, &bars->bfull[rb.s],
                             nb * TBN + c * 32, dd * p.S + i * BM, l2_evict_first_policy());
#else
            tma_load_2d(slot + dd * BIAS_ORDER_BYTES, &cm, &bars->bfull[rb.s], nb * TBN + c * 32,
                        dd * p.S + i * BM);
#endif
        }
        __syncwarp();
        rb.next();
      }
    }
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const size_t SD = (size_t)p.S * p.dm;
    if constexpr (UPDATE) {
      int t = 0;
      for (int w = blockIdx.x; w < n_jobs; w += gridDim.x) {
        int i, nb, d;
        if (!job(w, i, nb, d)) continue;
        const int acc = t & 1;
        const unsigned long long act = p.hmask[i];
        const unsigned long long cached = all_heads & ~act;
        const bool hasA = (d == 0) && act != 0ull;
        const bool hasB = cached != 0ull;
        const int row = i * BM + r;
        const bool row_ok = row < p.S;
        const size_t obase = (size_t)row * p.dm + (size_t)nb * BN;
        mbar_wait(&bars->tfull[acc], (t >> 1) & 1);
        tc_fence_after();
        const uint32_t tA = tbase + lane_off + acc * ACC_COLS;
        const uint32_t tB = tA + BN;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t ua[32], ub[32];
          if (hasA) tmem_ld32(tA + c * 32, ua);
          if (hasB) tmem_ld32(tB + c * 32, ub);
          tmem_ld_wait();
          gemm::reg_fence(ua);
          gemm::reg_fence(ub);
          if (!row_ok) continue;
          float o[32], b[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            o[k] = hasA ? __uint_as_float(ua[k]) : 0.f;
            b[k] = hasB ? __uint_as_float(ub[k]) : 0.f;
          }
          if (d == 0) {
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] += b[k];
            gemm::store_bf16x32(p.out + obase + c * 32, o);
          }
          if (hasB && p.orders[i] > d) gemm::store_bf16x32(p.bias + d * SD + obase + c * 32, b);
        }
        tc_fence_before();
        mbar_arrive(&bars->tempty[acc]);
        ++t;
      }
    } else {
      const float c0 = p.coef[0], c1 = p.coef[1], c2 = p.coef[2], c3 = p.coef[3];
      const uint32_t ring_u32 = smem_u32(ring);
      const uint32_t ostage_u32 = smem_u32(ostage);
      const int sw = (r >> 1) & 3;  // SW64: 16-B chunk q of row r sits at q ^ ((r >> 1) & 3)
      DynRing rb(bias_slots);
      int ob = 0;  // output staging buffer of this chunk
      int t = 0;
      for (int w = jstart; w < n_jobs; w += jstep) {
        int i, nb, d;
        if (!job(w, i, nb, d)) continue;
        const int nch = tile_cols(nb) / 32;
        const int acc = t & 1;
        const bool hasA = p.hmask[i] != 0ull;
        const int no = min(p.order_d + 1, p.orders[i]);
        const int ns = min(no, 2);
        const int row = i * BM + r;
        const bool row_ok = row < p.S;
        mbar_wait(&bars->tfull[acc], (t >> 1) & 1);
        tc_fence_after();
        const uint32_t tA = tbase + lane_off + acc * ACC_COLS;
        for (int c = 0; c < nch; ++c) {
          uint32_t ua[32];
          if (hasA) {
            tmem_ld32(tA + c * 32, ua);
            tmem_ld_wait();
            gemm::reg_fence(ua);
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) ua[k] = 0u;
          }
          if (c == nch - 1) {  // accumulator drained: release it to the MMA warp
            tc_fence_before();
            mbar_arrive(&bars->tempty[acc]);
          }
          mbar_wait(&bars->bfull[rb.s], rb.ph);
          const uint32_t rowa = ring_u32 + rb.s * bias_slot_bytes + r * 64;
          // every shared-memory load of the chunk first, then packed FMAs
          uint4 b0[4], b1[4];
          if (ns > 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) b0[q] = lds128(rowa + ((q ^ sw) << 4));
          }
          if (ns > 1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) b1[q] = lds128(rowa + BIAS_ORDER_BYTES + ((q ^ sw) << 4));
          }
          float2 o2[16];
#pragma unroll
          for (int k = 0; k < 16; ++k)
            o2[k] = make_float2(__uint_as_float(ua[2 * k]), __uint_as_float(ua[2 * k + 1]));
          auto fma_bias = [&](const uint4 (&bb)[4], float cf) {
            const float2 c2v = make_float2(cf, cf);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t w4[4] = {bb[q].x, bb[q].y, bb[q].z, bb[q].w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                o2[q * 4 + e] = ffma2(c2v, make_float2(bf16lo(w4[e]), bf16hi(w4[e])), o2[q * 4 + e]);
            }
          };
          if (ns > 0) fma_bias(b0, c0);
          if (ns > 1) fma_bias(b1, c1);
          if (no > 2 && row_ok) {  // orders 2..3 (rare): direct loads
            for (int dd = 2; dd < no; ++dd) {
              uint4 bb[4];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                bb[q] = __ldg(reinterpret_cast<const uint4*>(
                    p.bias + dd * SD + (size_t)row * p.dm + (size_t)nb * TBN + c * 32 + q * 8));
              fma_bias(bb, dd == 2 ? c2 : c3);
            }
          }
          uint4 res[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            res[q] = make_uint4(pack_bf16x2(o2[4 * q].x, o2[4 * q].y),
                                pack_bf16x2(o2[4 * q + 1].x, o2[4 * q + 1].y),
                                pack_bf16x2(o2[4 * q + 2].x, o2[4 * q + 2].y),
                                pack_bf16x2(o2[4 * q + 3].x, o2[4 * q + 3].y));
          __syncwarp();  // this warp's rows of the bias slot are read: release it
          if (lane == 0) mbar_arrive(&bars->bempty[rb.s]);
          rb.next();
          // each warp stores its own 32 rows (a 32 x 32 TMA box) from its quarter
          // of staging buffer ob, so the four epilogue warps never wait for each
          // other; the store that last read this quarter (two chunks ago) is done
          // reading (lane 0 waited for it right after issuing the next one)
          const uint32_t orow = ostage_u32 + ob * OUT_STAGE_BYTES + r * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q) sts128(orow + ((q ^ sw) << 4), res[q]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            uint8_t* src = ostage + ob * OUT_STAGE_BYTES + q4 * (OUT_STAGE_BYTES / 4);
#if FO_GO_EF_STORE
            tma_store_2d_hint(&om, src, nb * TBN + c * 32, i * BM + q4 * 32,
                              l2_evict_first_policy());
#else
            tma_store_2d(&om, src, nb * TBN + c * 32, i * BM + q4 * 32);
#endif
            bulk_commit();
            bulk_wait_read<OST - 1>();  // this warp's quarter of the other buffer is free
          }
          __syncwarp();
          ob = ob + 1 == OST ? 0 : ob + 1;
        }
        ++t;
      }
      if (lane == 0) bulk_wait<0>();
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TM_COLS>(tbase);
  }
}

// =============================================================================
// GEMM-O update (gemm.py:110-175), 2-CTA clusters like dispatch: both CTAs take
// the same block i (same K sequences) and neighbouring 256-column n-tiles, and
// each loads half of every A tile (o or a cache stack) and multicasts it.
//
// A d = 0 job (i, n-tile) runs two passes into ONE TMEM accumulator slot:
//   C pass: the heads cached under the next symbols, A = cache stack 0
//           -> the slot holds B_c[0]; the epilogue stores it (E1) and hands
//              the slot back;
//   A pass: the active heads, A = o, accumulated on top -> the slot holds
//           B_c[0] + sum_active o W = out; the epilogue stores it (E2).
// A d >= 1 job (d < orders[i]) is a C pass over cache stack d -> B_c[d].
// Every head is projected exactly once per order, as in the reference.
// Two slots (2 x 256 TMEM columns) and jobs taken in pairs (j, j'), issued
// C(j) C(j') A(j) A(j') on the tensor core while the epilogue runs
// E1(j) E1(j') E2(j) E2(j'): every epilogue step overlaps the next pass on the
// other slot, so the tensor core only waits when a store step is longer than
// a whole pass. The cache and bias are addressed through 3-D maps
// [order+1][S][cols], so a ragged last block never reads or writes across the
// slab of the next order.
// =============================================================================
namespace gemm {
constexpr int U_STAGES = 4;
constexpr int SMEM_BYTES_U = U_STAGES * D_STAGE_BYTES + 2 * OUT_STAGE_BYTES + 1024 + (int)sizeof(Bars);
static_assert(SMEM_BYTES_U <= 232448, "update shared memory over the sm_100 limit");
}  // namespace gemm

__global__ void __launch_bounds__(gemm::NTHREADS, 1)
    gemm_o_update_kernel(const __grid_constant__ CUtensorMap am,  // o [S, H*128], box 64 x 64
                         const __grid_constant__ CUtensorMap cm,  // cache [D+1][S][H*128], 64 x 64 x 1
                         const __grid_constant__ CUtensorMap wm,  // W_out^T [dm, H*128], 64 x 128
                         const __grid_constant__ CUtensorMap om,  // out [S, dm], 32 x 32 SW64
                         const __grid_constant__ CUtensorMap bm,  // B_c [D+1][S][dm], 32 x 32 x 1 SW64
                         const GemmOParams p) {
  using namespace gemm;
  constexpr int ST = U_STAGES, SB = D_STAGE_BYTES, TBN = D_BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* ostage = smem + ST * SB;
  Bars* bars = reinterpret_cast<Bars*>(ostage + 2 * OUT_STAGE_BYTES);
  const int warp = warp_id(), lane = lane_id();
  const int rank = (int)cluster_ctarank();
  if (warp == 0 && lane == 0) {
    init_bars(bars, 2, 4);  // a stage is free once both CTAs' MMA warps are done with it
    tma_prefetch_desc(&am);
    tma_prefetch_desc(&cm);
    tma_prefetch_desc(&wm);
    tma_prefetch_desc(&om);
    tma_prefetch_desc(&bm);
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  pdl_release_and_wait();
  const uint32_t tbase = bars->tmem_base;
  const int nbn = (p.dm + TBN - 1) / TBN;
  auto tile_cols = [&](int nb) { return min(TBN, p.dm - nb * TBN); };
  const int ncb = (nbn + 1) >> 1;  // n-tile pairs per block: one cluster job each
  const int per_d = p.t_q * ncb;
  const int n_jobs = (p.order_d + 1) * per_d;
  const int jstart = (int)(blockIdx.x >> 1), jstep = (int)(gridDim.x >> 1);
  const unsigned long long all_heads = (p.H >= 64) ? ~0ull : ((1ull << p.H) - 1);
  // order-major jobs; d >= 1 jobs exist only for blocks with that many orders
  // (the same test in both CTAs, so the pair walks identical job lists)
  auto valid = [&](int w) {
    const int d = w / per_d;
    return d == 0 || d < p.orders[(w - d * per_d) / ncb];
  };
  auto next_valid = [&](int w) {
    while (w < n_jobs && !valid(w)) w += jstep;
    return w;
  };
  struct Job {
    int i, nb, d;
    bool mine;
    unsigned long long cached, act;
  };
  auto decode = [&](int w) {
    Job j;
    j.d = w / per_d;
    const int rest = w - j.d * per_d;
    j.i = rest / ncb;
    j.nb = 2 * (rest - j.i * ncb) + rank;
    j.mine = j.nb < nbn;
    j.act = p.hmask[j.i];
    j.cached = all_heads & ~j.act;
    return j;
  };
  // heads of pass ph (0: C, 1: A) of a job
  auto pass_mask = [&](const Job& j, int ph) {
    return ph == 0 ? j.cached : (j.d == 0 ? j.act : 0ull);
  };

  if (warp == 0) {
    Ring<ST> rg;
    for (int w0 = next_valid(jstart); w0 < n_jobs;) {
      const int w1 = next_valid(w0 + jstep);
      const int ws[2] = {w0, w1};
      for (int ph = 0; ph < 2; ++ph)
        for (int k = 0; k < 2; ++k) {
          if (ws[k] >= n_jobs) continue;
          const Job j = decode(ws[k]);
          unsigned long long m = pass_mask(j, ph);
          const bool two = j.mine && tile_cols(j.nb) > BN;
          while (m) {
            const int h = __ffsll(m) - 1;
            m &= m - 1;
            for (int kk = 0; kk < 2; ++kk) {
              mbar_wait(&bars->empty[rg.s], rg.ph ^ 1);
              if (elect_one()) {
                uint8_t* st = smem + rg.s * SB;
                mbar_arrive_expect_tx(&bars->full[rg.s],
                                      A_BYTES + (j.mine ? (two ? 2 : 1) * B_BYTES : 0));
                if (ph == 0)
                  tma_load_3d_mc(st + rank * (A_BYTES / 2), &cm, &bars->full[rg.s],
                                 h * 128 + kk * BK, j.i * BM + rank * (BM / 2), j.d, 0x3);
                else
                  tma_load_2d_mc(st + rank * (A_BYTES / 2), &am, &bars->full[rg.s],
                                 h * 128 + kk * BK, j.i * BM + rank * (BM / 2), 0x3);
#if FO_GU_EL_W
                const uint64_t wpol = l2_evict_last_policy();
                if (j.mine)
                  tma_load_2d_hint(st + A_BYTES, &wm, &bars->full[rg.s], h * 128 + kk * BK,
                                   j.nb * TBN, wpol);
                if (two)
                  tma_load_2d_hint(st + A_BYTES + B_BYTES, &wm, &bars->full[rg.s],
                                   h * 128 + kk * BK, j.nb * TBN + BN, wpol);
#else
                if (j.mine)
                  tma_load_2d(st + A_BYTES, &wm, &bars->full[rg.s], h * 128 + kk * BK, j.nb * TBN);
                if (two)
                  tma_load_2d(st + A_BYTES + B_BYTES, &wm, &bars->full[rg.s], h * 128 + kk * BK,
                              j.nb * TBN + BN);
#endif
              }
              __syncwarp();
              rg.next();
            }
          }
        }
      w0 = w1 < n_jobs ? next_valid(w1 + jstep) : n_jobs;
    }
    // drain: both CTAs' MMA warps have released every stage
    for (int k = 0; k < ST; ++k) {
      mbar_wait(&bars->empty[rg.s], rg.ph ^ 1);
      rg.next();
    }
  } else if (warp == 1) {
    const uint32_t idesc1 = make_idesc_bf16(BM, BN, false, false);
    const uint32_t idesc2 = make_idesc_bf16(BM, 2 * BN, false, false);
    const uint64_t desc0 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
    Ring<ST> rg;
    int uses[2] = {0, 0};  // passes issued into each slot
    for (int w0 = next_valid(jstart); w0 < n_jobs;) {
      const int w1 = next_valid(w0 + jstep);
      const int ws[2] = {w0, w1};
      for (int ph = 0; ph < 2; ++ph)
        for (int k = 0; k < 2; ++k) {
          if (ws[k] >= n_jobs) continue;
          const Job j = decode(ws[k]);
          const uint32_t idesc = (j.mine && tile_cols(j.nb) > BN) ? idesc2 : idesc1;
          // the slot is free once the epilogue step of its previous pass is done
          if (uses[k] > 0) {
            mbar_wait(&bars->tempty[k], (uses[k] - 1) & 1);
            tc_fence_after();
          }
          const int nk = 2 * __popcll(pass_mask(j, ph));
          // the A pass accumulates onto the C pass's B_c[0]
          const bool acc0 = ph == 1 && j.cached != 0ull;
          const uint32_t dslot = tbase + k * D_BN;
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&bars->full[rg.s], rg.ph);
            tc_fence_after();
            const uint64_t a = desc0 + (uint64_t)((rg.s * SB) >> 4);
            if (elect_one()) {
              if (j.mine) mma_kblock(dslot, a, a + (A_BYTES >> 4), idesc, acc0 || kb > 0);
              tc_commit_mc(&bars->empty[rg.s], 0x3);
            }
            __syncwarp();
            rg.next();
          }
          if (elect_one()) tc_commit(&bars->tfull[k]);
          __syncwarp();
          ++uses[k];
        }
      w0 = w1 < n_jobs ? next_valid(w1 + jstep) : n_jobs;
    }
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t ostage_u32 = smem_u32(ostage);
    const int sw = (r >> 1) & 3;  // SW64: 16-B chunk q of row r sits at q ^ ((r >> 1) & 3)
#if FO_GU_EF_STORE
    const uint64_t pol = l2_evict_first_policy();
#else
    const uint64_t pol = l2_evict_normal_policy();
#endif
    int uses[2] = {0, 0};
    int ob = 0;
    for (int w0 = next_valid(jstart); w0 < n_jobs;) {
      const int w1 = next_valid(w0 + jstep);
      const int ws[2] = {w0, w1};
      for (int ph = 0; ph < 2; ++ph)
        for (int k = 0; k < 2; ++k) {
          if (ws[k] >= n_jobs) continue;
          const Job j = decode(ws[k]);
          mbar_wait(&bars->tfull[k], uses[k] & 1);
          tc_fence_after();
          ++uses[k];
          // E1 (after the C pass): B_c[d]; E2 (after the A pass of a d = 0 job): out
          const bool store = j.mine && (ph == 0 ? (j.cached != 0ull && j.d < p.orders[j.i])
                                                : j.d == 0);
          if (!store) {
            tc_fence_before();
            mbar_arrive(&bars->tempty[k]);
            continue;
          }
          const int nch = tile_cols(j.nb) / 32;
          const uint32_t ts = tbase + lane_off + k * D_BN;
          for (int c = 0; c < nch; ++c) {
            uint32_t u[32];
            tmem_ld32(ts + c * 32, u);
            tmem_ld_wait();
            if (c == nch - 1) {  // slot drained: the tensor core may take it
              tc_fence_before();
              mbar_arrive(&bars->tempty[k]);
            }
            uint4 res[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              res[q] = make_uint4(
                  pack_bf16x2(__uint_as_float(u[8 * q + 0]), __uint_as_float(u[8 * q + 1])),
                  pack_bf16x2(__uint_as_float(u[8 * q + 2]), __uint_as_float(u[8 * q + 3])),
                  pack_bf16x2(__uint_as_float(u[8 * q + 4]), __uint_as_float(u[8 * q + 5])),
                  pack_bf16x2(__uint_as_float(u[8 * q + 6]), __uint_as_float(u[8 * q + 7])));
            // this warp's 32 rows -> its quarter of staging buffer ob -> one TMA
            // store; the store that last read the quarter (two chunks ago) is done
            const uint32_t orow = ostage_u32 + ob * OUT_STAGE_BYTES + r * 64;
#pragma unroll
            for (int q = 0; q < 4; ++q) sts128(orow + ((q ^ sw) << 4), res[q]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              uint8_t* src = ostage + ob * OUT_STAGE_BYTES + q4 * (OUT_STAGE_BYTES / 4);
              if (ph == 0)
                tma_store_3d_hint(&bm, src, j.nb * TBN + c * 32, j.i * BM + q4 * 32, j.d, pol);
              else
                tma_store_2d_hint(&om, src, j.nb * TBN + c * 32, j.i * BM + q4 * 32, pol);
              bulk_commit();
              bulk_wait_read<1>();
            }
            __syncwarp();
            ob ^= 1;
          }
        }
      w0 = w1 < n_jobs ? next_valid(w1 + jstep) : n_jobs;
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

void launch_gemm_o(const CUtensorMap& am, const CUtensorMap& cm, const CUtensorMap& wm,
                   const CUtensorMap& om, const GemmOParams& p, int max_ctas, cudaStream_t stream) {
  static int grid_d = 0;
  launch_pair_clusters_max(gemm_o_kernel<false>, gemm::SMEM_BYTES_D, &grid_d, max_ctas, stream, am,
                           cm, wm, om, p);
}

void launch_gemm_o_update(const CUtensorMap& am, const CUtensorMap& cm, const CUtensorMap& wm,
                          const CUtensorMap& om, const CUtensorMap& bm, const GemmOParams& p,
                          cudaStream_t stream) {
  static int grid_u = 0;
  launch_pair_clusters(gemm_o_update_kernel, gemm::SMEM_BYTES_U, &grid_u, stream, am, cm, wm, om, bm,
                       p);
}

}  // namespace fo
