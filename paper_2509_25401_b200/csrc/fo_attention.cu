// K2 / K2u: symbol-guided sparse attention on sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces reference attention.py:150-221 (sparse_attention) together with its
// tile kernel pyref.py:14-48 / _core.pyx:14-101 (masked_block_attention): for
// every query block i of head h whose cache symbol is 1 (compute), run the
// online-softmax over exactly the key blocks j whose skip symbol is 1; cached
// query blocks are never scheduled (their rows are left untouched, the
// reference's mode="bias"). In update mode (dense=1) every pair is computed
// and the epilogue pushes the fresh tile into the feature cache's backward
// difference stacks in place (attention.py:71-85, pipeline.py:274-278).
//
// One persistent CTA per SM walks a schedule of (head, q-block) items sorted
// by KV-block count (longest first). Warp roles:
//   warp 0      TMA producer: decodes the item's s_s row with a warp ballot
//               (the "register run cache" of PAPER.md:248) and streams Q and the
//               surviving K/V tiles into a 3-deep K ring / 2-deep V ring.
//   warp 1      tcgen05.mma issuer: S_j = Q K_j^T (SS) into one of two TMEM S
//               buffers, O += P_j V_j and L += P_j 1 (TS, P read straight from
//               TMEM; L is the softmax row sum, computed on the tensor core).
//   warps 4..7  softmax: one thread per query row; S from TMEM, lazy rescale
//               (threshold 2^8) of the TMEM O accumulator, P written back as bf16
//               over the S columns; epilogue O/l -> bf16 -> HBM (+ cache push).
// TMEM: O cols [0,128), L [128,144), S0 [256,384), S1 [384,512).
#include "fo_internal.cuh"

// pairs (out of every 8) whose exp2 runs as an FMA-pipe polynomial instead of
// on the MUFU
#ifndef FO_POLY_OF_8
#define FO_POLY_OF_8 2
#endif

#ifdef FO_ATTN_TIMING
#define TSTAMP(k)                     \
  if (tim) {                          \
    const long long _t = clock64();   \
    tacc[k] += _t - tlast;            \
    tlast = _t;                       \
  }
#else
#define TSTAMP(k)
#endif

namespace fo {
namespace attn {
constexpr int KST = 3, VST = 2;
constexpr int TILE_BYTES = kTile * kTile * 2;  // 32 KB bf16 tile
constexpr int HALF_BYTES = TILE_BYTES / 2;     // 128 rows x 64 cols, 128B-swizzled
constexpr int SMEM_TILES = 1 + KST + VST;
constexpr int NTHREADS = 256;
constexpr uint32_t TM_O = 0, TM_L = 128, TM_S0 = 256;
constexpr int ONES_BYTES = 2048;  // 16 rows x 128 B of bf16 1.0 (the B operand of the row-sum MMA)

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[KST], k_empty[KST];
  uint64_t v_full[VST], v_empty[VST];
  uint64_t s_full[2];
  uint64_t p_full, o_done, o_last, o_free;
  uint32_t tmem_base;
  int fc_tile;  // fused forecast: the tile the softmax warps take next
};
constexpr int SMEM_BYTES = SMEM_TILES * TILE_BYTES + ONES_BYTES + 1024 + (int)sizeof(Bars);
}  // namespace attn

// keep the compiler from hoisting uses of tcgen05.ld results above the wait
template <int N>
__device__ __forceinline__ void reg_fence(uint32_t (&r)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) asm volatile("" : "+r"(r[k]));
}

__global__ void __launch_bounds__(attn::NTHREADS, 1)
    sparse_attention_kernel(const __grid_constant__ CUtensorMap qm,
                            const __grid_constant__ CUtensorMap km,
                            const __grid_constant__ CUtensorMap vm, const AttnParams p) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;
  uint8_t* sV = smem + TILE_BYTES * (1 + KST);
  uint8_t* sOnes = smem + TILE_BYTES * SMEM_TILES;  // 1024-aligned
  Bars* bars = reinterpret_cast<Bars*>(sOnes + ONES_BYTES);
  for (int e = threadIdx.x; e < ONES_BYTES / 4; e += blockDim.x)
    reinterpret_cast<uint32_t*>(sOnes)[e] = 0x3F803F80u;  // bf16 1.0 pairs
  fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    mbar_init(&bars->s_full[0], 1);
    mbar_init(&bars->s_full[1], 1);
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->o_done, 1);
    mbar_init(&bars->o_last, 1);
    mbar_init(&bars->o_free, 128);
    fence_barrier_init();
    tma_prefetch_desc(&qm);
    tma_prefetch_desc(&km);
    tma_prefetch_desc(&vm);
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars->tmem_base;
  const int n_items = *p.n_items;
  const size_t head_sym = (size_t)p.comp_rows * p.row_stride;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    int kst = 0, kph = 0, vst = 0, vph = 0, qi = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++qi) {
      const int2 it = p.items[w];
      const int h = it.x >> 20, i = it.x & 0xFFFFF;
      mbar_wait(&bars->q_empty, (qi & 1) ^ 1, p.status);
      if (elect_one()) {
        mbar_arrive_expect_tx(&bars->q_full, TILE_BYTES);
        tma_load_2d(sQ, &qm, &bars->q_full, h * kTile, i * kTile);
        tma_load_2d(sQ + HALF_BYTES, &qm, &bars->q_full, h * kTile + 64, i * kTile);
      }
      __syncwarp();
      const uint8_t* sym = p.s_s + h * head_sym;
      for (int base = 0; base < p.t_kv; base += 32) {
        const int j = base + lane;
        const uint32_t bit =
            (j < p.t_kv) && (p.dense || decode_reduction(sym, p.row_stride, i, j, p.pool_n));
        uint32_t m = __ballot_sync(0xffffffffu, bit);  // warp-uniform
        while (m) {
          const int jj = base + __ffs(m) - 1;
          m &= m - 1;
          mbar_wait(&bars->k_empty[kst], kph ^ 1, p.status);
          if (elect_one()) {
            mbar_arrive_expect_tx(&bars->k_full[kst], TILE_BYTES);
            uint8_t* dk = sK + kst * TILE_BYTES;
            tma_load_2d(dk, &km, &bars->k_full[kst], h * kTile, jj * kTile);
            tma_load_2d(dk + HALF_BYTES, &km, &bars->k_full[kst], h * kTile + 64, jj * kTile);
          }
          __syncwarp();
          if (++kst == KST) {
            kst = 0;
            kph ^= 1;
          }
          mbar_wait(&bars->v_empty[vst], vph ^ 1, p.status);
          if (elect_one()) {
            mbar_arrive_expect_tx(&bars->v_full[vst], TILE_BYTES);
            uint8_t* dv = sV + vst * TILE_BYTES;
            tma_load_2d(dv, &vm, &bars->v_full[vst], h * kTile, jj * kTile);
            tma_load_2d(dv + HALF_BYTES, &vm, &bars->v_full[vst], h * kTile + 64, jj * kTile);
          }
          __syncwarp();
          if (++vst == VST) {
            vst = 0;
            vph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the schedule (every value stays warp-uniform, so the
    // descriptors live in uniform registers); one elected lane issues the MMAs
    // and the commits that track them.
    {
      const uint32_t idesc_qk = make_idesc_bf16(128, 128, false, false);
      const uint32_t idesc_pv = make_idesc_bf16(128, 128, false, true);
      const uint32_t idesc_l = make_idesc_bf16(128, 16, false, false);
      const uint64_t ones_desc = make_sdesc_sw128(smem_u32(sOnes), 16, 1024);
      int kst = 0, kph = 0, vst = 0, vph = 0, qi = 0;
      uint32_t qk_cnt = 0, pv_cnt = 0;
      // descriptor of K-chunk k (16 elements) of a K-major SW128 tile: +32 B within a
      // 64-column half, +16 KB to the second half (start address is in 16 B units)
      const uint64_t qdesc = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t kdesc0 = make_sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t vdesc0 = make_sdesc_sw128(smem_u32(sV), HALF_BYTES, 1024);
#ifdef FO_ATTN_TIMING
      const bool tim = p.dbg != nullptr && lane == 0;
      long long tacc[16] = {0};
      long long tlast = clock64();
#endif
      auto issue_qk = [&]() {
        TSTAMP(11);
        mbar_wait(&bars->k_full[kst], kph, p.status);
        TSTAMP(10);
        tc_fence_after();
        const uint32_t sb = qk_cnt & 1;
        const uint32_t d = tbase + TM_S0 + sb * 128;
        const uint64_t kdesc = kdesc0 + (uint64_t)((kst * TILE_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t off = (uint64_t)((k >> 2) * (HALF_BYTES >> 4) + (k & 3) * 2);
            mma_bf16_ss(d, qdesc + off, kdesc + off, idesc_qk, k > 0);
          }
          tc_commit(&bars->k_empty[kst]);
          tc_commit(&bars->s_full[sb]);
        }
        __syncwarp();
        if (++kst == KST) {
          kst = 0;
          kph ^= 1;
        }
        ++qk_cnt;
      };
      auto commit_q_empty = [&]() {
        if (elect_one()) tc_commit(&bars->q_empty);
        __syncwarp();
      };
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++qi) {
        const int n = p.items[w].y;
        mbar_wait(&bars->q_full, qi & 1, p.status);
        tc_fence_after();
        issue_qk();
        if (n == 1) commit_q_empty();
        for (int j = 0; j < n; ++j) {
          if (j + 1 < n) {
            issue_qk();
            if (j + 2 == n) commit_q_empty();
          }
          TSTAMP(8);
          mbar_wait(&bars->p_full, pv_cnt & 1, p.status);
          TSTAMP(9);
          if (j == 0 && qi > 0) mbar_wait(&bars->o_free, (qi - 1) & 1, p.status);
          TSTAMP(12);
          mbar_wait(&bars->v_full[vst], vph, p.status);
          TSTAMP(13);
          tc_fence_after();
          const uint32_t a_t = tbase + TM_S0 + (pv_cnt & 1) * 128;
          const uint64_t vdesc = vdesc0 + (uint64_t)((vst * TILE_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              mma_bf16_ts(tbase + TM_O, a_t + k * 8, vdesc + (uint64_t)(k * (2048 >> 4)), idesc_pv,
                          (j > 0 || k > 0));
            // row sums on the tensor core: L += P . 1 (every B element is 1.0, so one
            // descriptor serves all K chunks); l is then exactly sum(bf16(P))
#pragma unroll
            for (int k = 0; k < 8; ++k)
              mma_bf16_ts(tbase + TM_L, a_t + k * 8, ones_desc, idesc_l, (j > 0 || k > 0));
            tc_commit(&bars->v_empty[vst]);
            tc_commit(&bars->o_done);
            if (j == n - 1) tc_commit(&bars->o_last);  // every PV of the item is done
          }
          __syncwarp();
          if (++vst == VST) {
            vst = 0;
            vph ^= 1;
          }
          ++pv_cnt;
        }
      }
#ifdef FO_ATTN_TIMING
      if (tim)
        for (int q = 8; q < 16; ++q) p.dbg[blockIdx.x * 32 + 16 + q] = tacc[q];
#endif
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const int last_valid = p.S - (p.t_kv - 1) * kTile;  // valid key columns of the last block
    const size_t HD = (size_t)p.H * kTile;
    const size_t stack_stride = (size_t)p.S * HD;
    uint32_t qk_seen = 0, o_base = 0;  // o_base: PVs of all earlier items
#ifdef FO_ATTN_TIMING
    const bool tim = (r == 0) && p.dbg;
    long long tacc[16] = {0};
    long long tlast = clock64();
#endif
    int qi = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++qi) {
      const int2 it = p.items[w];
      const int h = it.x >> 20, i = it.x & 0xFFFFF, n = it.y;
      const bool tail = (last_valid < kTile) &&
                        (p.dense || decode_reduction(p.s_s + h * head_sym, p.row_stride, i,
                                                     p.t_kv - 1, p.pool_n));
      const int valid_old = (p.cache && p.valid) ? p.valid[(size_t)h * p.t_q + i] : 0;
      float m_run = -INFINITY;
      for (int j = 0; j < n; ++j) {
        const uint32_t sb = qk_seen & 1;
        TSTAMP(7);
        mbar_wait(&bars->s_full[sb], (qk_seen >> 1) & 1, p.status);
        TSTAMP(0);
        tc_fence_after();
        ++qk_seen;
        const uint32_t sa = tbase + lane_off + TM_S0 + sb * 128;
        uint32_t u[4][32];
        tmem_ld32(sa + 0, u[0]);
        tmem_ld32(sa + 32, u[1]);
        tmem_ld32(sa + 64, u[2]);
        tmem_ld32(sa + 96, u[3]);
        tmem_ld_wait();
        TSTAMP(1);
        reg_fence(u[0]);
        reg_fence(u[1]);
        reg_fence(u[2]);
        reg_fence(u[3]);
        const bool mask_tail = tail && (j == n - 1);
        float sv[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int k = 0; k < 32; ++k) sv[c * 32 + k] = __uint_as_float(u[c][k]);
        if (mask_tail) {
          // key columns past the sequence end in the last (partial) block
#pragma unroll
          for (int k = 0; k < 128; ++k)
            if (k >= last_valid) sv[k] = -INFINITY;
        }
        // row max: eight independent FMNMX3 chains of 16 values, then a 3-level tree
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
        const float m_tile = mx * p.scale_log2;
        TSTAMP(2);
        bool need = false;
        float m_new;
        if (j == 0) {
          m_new = m_tile;
        } else if (m_tile > m_run + 8.f) {
          need = true;
          m_new = m_tile;
        } else {
          m_new = m_run;
        }
        const float corr = need ? fast_exp2(m_run - m_new) : 1.f;
        m_run = m_new;
        // P = 2^(s*scale - m): packed FFMA2; exp2 split between the MUFU and an
        // FMA-pipe polynomial (FO_POLY_OF_8 of every 8 pairs), which balances the
        // two pipes (packed fp32x2 ops cost 4 issue cycles per warp, MUFU 8)
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-m_new, -m_new);

        uint32_t pk[2][32];
        if (!mask_tail) {
#pragma unroll
          for (int q = 0; q < 64; ++q) {
            const float2 x = ffma2(make_float2(sv[2 * q], sv[2 * q + 1]), sc2, nm2);
            float2 e;
            if ((q & 7) < FO_POLY_OF_8) {
              e = exp2_poly2(x);
            } else {
              e.x = fast_exp2(x.x);
              e.y = fast_exp2(x.y);
            }
            pk[q >> 5][q & 31] = pack_bf16x2(e.x, e.y);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 64; ++q) {
            const float2 x = ffma2(make_float2(sv[2 * q], sv[2 * q + 1]), sc2, nm2);
            float2 e;
            e.x = fast_exp2(x.x);  // exact zeros for the masked (-inf) columns
            e.y = fast_exp2(x.y);
            pk[q >> 5][q & 31] = pack_bf16x2(e.x, e.y);
          }
        }
        tmem_st32(sa + 0, pk[0]);
        TSTAMP(3);
        tmem_st32(sa + 32, pk[1]);
        tmem_st_wait();
        TSTAMP(4);
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          // PV_{j-1} must be complete before O can be rescaled for P_j. Waits are
          // taken only when a lane rescales: S_j's commit already tracked every
          // PV before PV_{j-1}, so o_done has completed o_base+j-1 or o_base+j
          // phases and the parity of completion o_base+j is unambiguous.
          mbar_wait(&bars->o_done, (o_base + j - 1) & 1, p.status);
          tc_fence_after();
          {
            const uint32_t oa = tbase + lane_off + TM_O;
#pragma unroll
            for (int c = 0; c < 5; ++c) {  // O and the row-sum columns
              uint32_t o[32];
              tmem_ld32(oa + c * 32, o);
              tmem_ld_wait();
              reg_fence(o);
#pragma unroll
              for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * corr);
              tmem_st32(oa + c * 32, o);
            }
            tmem_st_wait();
          }
        }
        TSTAMP(5);
        tc_fence_before();
        mbar_arrive(&bars->p_full);
        TSTAMP(6);
      }
      // ---------------- epilogue: O / l -> bf16 -> HBM (+ feature-cache push)
      mbar_wait(&bars->o_last, qi & 1, p.status);  // one phase per item
      o_base += n;
      tc_fence_after();
      uint32_t lsum[16];
      tmem_ld16(tbase + lane_off + TM_L, lsum);
      tmem_ld_wait();
      reg_fence(lsum);
      const float inv_l = 1.f / __uint_as_float(lsum[0]);
      const int row = i * kTile + r;
      const bool row_ok = row < p.S;
      const int vn = min(valid_old + 1, p.order_d + 1);
      const uint32_t oa = tbase + lane_off + TM_O;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld32(oa + c * 32, o);
        tmem_ld_wait();
        reg_fence(o);
        float of[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) of[k] = __uint_as_float(o[k]) * inv_l;
        if (row_ok) {
          const size_t off = (size_t)row * HD + (size_t)h * kTile + c * 32;
          uint4* dst = reinterpret_cast<uint4*>(p.out + off);
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            uint4 pkv;
            pkv.x = pack_bf16x2(of[v4 * 8 + 0], of[v4 * 8 + 1]);
            pkv.y = pack_bf16x2(of[v4 * 8 + 2], of[v4 * 8 + 3]);
            pkv.z = pack_bf16x2(of[v4 * 8 + 4], of[v4 * 8 + 5]);
            pkv.w = pack_bf16x2(of[v4 * 8 + 6], of[v4 * 8 + 7]);
            dst[v4] = pkv;
          }
          if (p.cache) {
            // backward-difference push: new[0]=o, new[d]=new[d-1]-old[d-1] for d<vn, else 0
            float cur[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) cur[k] = of[k];
            for (int d = 0; d <= p.order_d; ++d) {
              uint4* cd = reinterpret_cast<uint4*>(p.cache + d * stack_stride + off);
              float nxt[32];
              const bool live_next = (d + 1 < vn);
              if (live_next) {
                // read old[d] before overwriting slot d
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                  uint4 ov = cd[v4];
                  const uint32_t w4[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    nxt[v4 * 8 + 2 * e] = cur[v4 * 8 + 2 * e] - bf16lo(w4[e]);
                    nxt[v4 * 8 + 2 * e + 1] = cur[v4 * 8 + 2 * e + 1] - bf16hi(w4[e]);
                  }
                }
              }
              const bool live = d < vn;
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4) {
                uint4 pkv;
                if (live) {
                  pkv.x = pack_bf16x2(cur[v4 * 8 + 0], cur[v4 * 8 + 1]);
                  pkv.y = pack_bf16x2(cur[v4 * 8 + 2], cur[v4 * 8 + 3]);
                  pkv.z = pack_bf16x2(cur[v4 * 8 + 4], cur[v4 * 8 + 5]);
                  pkv.w = pack_bf16x2(cur[v4 * 8 + 6], cur[v4 * 8 + 7]);
                } else {
                  pkv = make_uint4(0, 0, 0, 0);
                }
                cd[v4] = pkv;
              }
              if (live_next) {
#pragma unroll
                for (int k = 0; k < 32; ++k) cur[k] = nxt[k];
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->o_free);
      if (r == 0) {
        if (p.pairs) atomicAdd(reinterpret_cast<unsigned long long*>(&p.pairs[h]),
                               static_cast<unsigned long long>(n));
        if (p.cache && p.valid) p.valid[(size_t)h * p.t_q + i] = vn;
      }
    }
#ifdef FO_ATTN_TIMING
    if (tim)
      for (int q = 0; q < 16; ++q) p.dbg[blockIdx.x * 32 + q] = tacc[q];
#endif
    if (p.fc_cache) forecast_cached_tiles<128>(p, threadIdx.x - 128, 8, &bars->fc_tile);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

void launch_attention(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                      const AttnParams& p, int grid, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(sparse_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         attn::SMEM_BYTES);
    configured = true;
  }
  note_launch();
  sparse_attention_kernel<<<grid, attn::NTHREADS, attn::SMEM_BYTES, stream>>>(qm, km, vm, p);
}

}  // namespace fo
