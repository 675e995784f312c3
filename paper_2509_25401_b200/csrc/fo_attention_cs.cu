// K2 / K2u, column-split softmax (sm_100a): the default attention kernel.
//
// Same contract and pipeline as fo_attention.cu (reference attention.py:150-221
// with the tile kernel pyref.py:14-48): producer warp, MMA warp with a
// double-buffered S in TMEM and P read straight from TMEM by the PV MMA. The
// softmax differs: two warpgroups share every tile, warp w (4..7) taking key
// columns 0-63 and warp w+4 (8..11) columns 64-127 of the same 32 rows (the
// same TMEM lane quarter, hence the same SMSP).
//
// Why (tools/softmax_microbench.cu, ncu): the 128x128 tile softmax costs ~1340
// cycles per SMSP with one warp, which cannot cover its own dependency
// latencies, and ~1030 with two. Splitting columns puts two warps on every
// SMSP while keeping the S double buffer, so QK(j+1) still overlaps softmax(j).
// The two-stream ping-pong alternative serialises each stream's
// S -> P -> PV -> S chain and measured 20% slower. The partners exchange
// half-row maxima through shared memory behind a 64-thread named barrier, so
// both apply the same running max. Each writes its half of P (P columns 0-31 /
// 32-63, after both have read S) and rescales its half of O. Row sums are fp32
// in registers, combined once per item: the P x ones row-sum MMA of
// fo_attention.cu re-reads P from TMEM and costs ~512 tensor cycles per tile.
#include "fo_internal.cuh"

// pairs (of every 8) whose exp2 runs as the FMA-pipe polynomial; with two
// softmax warps per SMSP the MUFU is the tighter pipe, so more go to the FMA
// 1: the epilogue stages each warp's 32 x 32 bf16 O chunk in shared memory and
// TMA-stores it (4 L1 wavefronts per 16-B shared store instead of 32 per
// uncoalesced 256-bit global store; the softmax warps' next shared-memory ops
// no longer queue behind the stores)
#ifndef FO_CS_TMA_OUT
#define FO_CS_TMA_OUT 1
#endif
#ifndef FO_CS_VPROD
#define FO_CS_VPROD 0  // 1: V tiles loaded by their own producer warp (warp 3)
#endif
#ifndef FO_CS_ODONE_ALL
#define FO_CS_ODONE_ALL 0  // 1: await every o_done phase (synccheck-clean, ~2% slower)
#endif
#ifndef FO_CS_POLY_OF_8
#define FO_CS_POLY_OF_8 3
#endif
// finer split: pairs (of every 16) on the polynomial; default 2 * FO_CS_POLY_OF_8
#ifndef FO_CS_POLY_OF_16
#define FO_CS_POLY_OF_16 (2 * FO_CS_POLY_OF_8)
#endif
// 1: row sums by a P x ones MMA into TMEM (re-reads P from TMEM: ~512 tensor
// cycles per tile); 0: fp32 row sums in registers, halves combined per item
#ifndef FO_CS_TC_ROWSUM
#define FO_CS_TC_ROWSUM 0
#endif
// 1 (default): row sums come out of the PV MMA itself. Every V stage carries a
// third 64-column strip of bf16 ones after its two 64-column halves, and PV runs
// with N = 144, so TMEM columns 128..143 accumulate l = sum(bf16(P)) next to O.
// That costs 16/128 more PV tensor cycles (64 per tile) and removes the 32
// packed fp32 adds per warp per tile from the FMA pipe, which (with the exp2
// polynomial) is what bounds the softmax. The K ring drops to 2 stages to make
// room (measured neutral).
#ifndef FO_CS_ONESCOL
#define FO_CS_ONESCOL 1
#endif
#if FO_CS_ONESCOL
#undef FO_CS_TC_ROWSUM
#define FO_CS_TC_ROWSUM 1  // l lives in TMEM: rescaled with O, read by the epilogue
#ifndef FO_CS_KST
#define FO_CS_KST 2
#endif
#endif

namespace fo {
namespace attn_cs {
#ifndef FO_CS_KST
#define FO_CS_KST 3
#endif
constexpr int KST = FO_CS_KST, VST = 2;
constexpr int TILE_BYTES = kTile * kTile * 2;  // 32 KB bf16 tile
constexpr int HALF_BYTES = TILE_BYTES / 2;     // 128 rows x 64 cols, 128B-swizzled
constexpr int V_STAGE_BYTES = FO_CS_ONESCOL ? TILE_BYTES + HALF_BYTES : TILE_BYTES;
constexpr int SMEM_TILE_BYTES = TILE_BYTES * (1 + KST) + V_STAGE_BYTES * VST;
// softmax warps per lane quarter (each takes 128/SPLIT key columns of its rows)
#ifndef FO_CS_SPLIT
#define FO_CS_SPLIT 2
#endif
constexpr int SPLIT = FO_CS_SPLIT;
constexpr int NCOL = kTile / SPLIT;  // key columns per softmax warp
constexpr int NCH = NCOL / 32;       // 32-column TMEM chunks per softmax warp
static_assert(SPLIT == 2 || SPLIT == 4, "column split of 2 or 4 warps per lane quarter");
static_assert(SPLIT == 2 || FO_CS_TC_ROWSUM, "a 4-way split needs the row sums in TMEM");
constexpr int SOFTMAX_THREADS = 128 * SPLIT;
constexpr int NTHREADS = 128 + SOFTMAX_THREADS;
// S buffers in TMEM: QK(j + SBUF - 1) is issued while P(j) is produced. Two
// buffers leave one tile of slack between a softmax step and the S it needs
// next (S(j) waits on PV(j-2) + QK(j)); three need the row sums in registers
// (O 128 + 3 x 128 S columns = all 512)
#ifndef FO_CS_SBUF
#define FO_CS_SBUF 2
#endif
constexpr int SBUF = FO_CS_SBUF;
static_assert(SBUF == 2 || (SBUF == 3 && !FO_CS_TC_ROWSUM), "three S buffers need register row sums");
constexpr uint32_t TM_O = 0, TM_L = 128, TM_S0 = SBUF == 3 ? 128 : 256;
constexpr int ONES_BYTES = 2048;  // 16 rows x 128 B of bf16 1.0 (B operand of the row-sum MMA)

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[KST], k_empty[KST];
  uint64_t v_full[VST], v_empty[VST];
  uint64_t s_full[SBUF];
  // p_full[b]: P of the tiles using S buffer b stored (one phase per use). One
  // barrier per buffer: a softmax step may finish P(j + 1) before the MMA warp,
  // busy issuing QK(j + SBUF - 1), has observed P(j)
  uint64_t p_full[SBUF];
  uint64_t o_done, o_last, o_free;
  uint32_t tmem_base;
  float xmax[2][SPLIT][128];  // [tile parity][column group][row]: partial row maxima
  float xsum[2][128];     // [column half][row]: partial row sums at the epilogue
  int fc_tile;            // fused forecast: the tile the softmax warps take next
};
// O staging: one 32-row x 32-column SW64 box (2 KB) per softmax warp
constexpr int OSTAGE_BYTES = FO_CS_TMA_OUT ? SOFTMAX_THREADS / 32 * 2048 : 0;
constexpr int SMEM_BYTES =
    SMEM_TILE_BYTES + ONES_BYTES + OSTAGE_BYTES + 1024 + (int)sizeof(Bars);
static_assert(SMEM_BYTES <= 232448, "column-split attention exceeds shared memory");
}  // namespace attn_cs

namespace {
template <int N>
__device__ __forceinline__ void reg_fence_cs(uint32_t (&r)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) asm volatile("" : "+r"(r[k]));
}
}  // namespace

// This CTA's item sequence (plan schedule: the k-th item is sched[k * grid +
// blockIdx.x]), read ahead: the schedule entry two items ahead and the item
// record one item ahead are loaded while the current item runs. Read at the
// top of each item, the two dependent global loads stalled every role ~1 us
// per item (the MMA warp's first QK, the producer's Q load).
struct ItemCursor {
  const int* sched;
  const int2* items;
  int n_waves, w1, w2;
  int2 it1;
  int slot, nslots;  // schedule column (CTA, or cluster in the CTA-pair kernel) and width
  __device__ ItemCursor(const int* s, const int2* its, int nw, int sl, int ns)
      : sched(s), items(its), n_waves(nw), slot(sl), nslots(ns) {
    w1 = nw > 0 ? s[sl] : -1;
    it1 = w1 >= 0 ? its[w1] : make_int2(0, 0);
    w2 = nw > 1 ? s[ns + sl] : -1;
  }
  // item k (call with k = 0, 1, ...): false at the end of the schedule
  __device__ __forceinline__ bool next(int k, int& w, int2& it) {
    w = w1;
    it = it1;
    if (w < 0) return false;
    w1 = w2;
    it1 = w2 >= 0 ? items[w2] : make_int2(0, 0);
    w2 = k + 2 < n_waves ? sched[(k + 2) * nslots + slot] : -1;
    return true;
  }
  __device__ __forceinline__ int peek_w() const { return w1; }
  __device__ __forceinline__ int2 peek_item() const { return it1; }
};

#ifdef FO_CS_TIMING  // tools/cs_timing.py: per-CTA start/end (globaltimer), SM id, tiles
__device__ unsigned long long g_cs_timing[16 * 1024];
__device__ long long g_cs_ph[5 * 1024];
__device__ long long g_cs_ep[6 * 1024];  // epilogue sub-phases (cycles, summed over items)
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// PAIR: 2-CTA clusters for pooled symbols (pool_n even). Query blocks 2c and
// 2c+1 share one compressed skip row, so the CTAs of a cluster take them
// together (item (h, 2c); a missing 2c+1 is a zero-filled block past the end)
// and walk the same K/V sequence in lockstep: each CTA TMA-loads one 64-column
// half of every K and V tile and multicasts it to both, halving the K/V reads
// from L2. A stage is refilled once both CTAs' MMAs have released it.
template <bool PAIR>
__global__ void __launch_bounds__(attn_cs::NTHREADS, 1)
    sparse_attention_cs_kernel(const __grid_constant__ CUtensorMap qm,
                               const __grid_constant__ CUtensorMap km,
                               const __grid_constant__ CUtensorMap vm,
                               const __grid_constant__ CUtensorMap om,  // out, 32 x 32 SW64
                               const AttnParams p) {
  using namespace attn_cs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;
  uint8_t* sV = smem + TILE_BYTES * (1 + KST);
  uint8_t* sOnes = smem + SMEM_TILE_BYTES;  // 1024-aligned
  uint8_t* sOst = sOnes + ONES_BYTES;       // 1024-aligned (ONES_BYTES = 2 KB)
  Bars* bars = reinterpret_cast<Bars*>(sOst + OSTAGE_BYTES);
  for (int e = threadIdx.x; e < ONES_BYTES / 4; e += blockDim.x)
    reinterpret_cast<uint32_t*>(sOnes)[e] = 0x3F803F80u;  // bf16 1.0 pairs
  if (FO_CS_ONESCOL)  // the ones strip behind each V stage (every byte 1.0, so swizzle-free)
    for (int s = 0; s < VST; ++s)
      for (int e = threadIdx.x; e < HALF_BYTES / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(sV + s * V_STAGE_BYTES + TILE_BYTES)[e] =
            make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
  const int warp = warp_id(), lane = lane_id();
  const int rank = PAIR ? (int)cluster_ctarank() : 0;  // this CTA's block: item block + rank
  const int slot = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nslots = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  constexpr uint32_t kEmptyCount = PAIR ? 2 : 1;  // both CTAs' MMAs release a K/V stage
  // one K or V tile (two 64-column SW128 halves) into a stage; in a pair each
  // CTA loads its half and multicasts it (the full barrier of each CTA counts
  // the bytes of both halves)
  auto load_tile = [&](uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int h, int jj) {
    if (PAIR) {
      tma_load_2d_mc(dst + rank * HALF_BYTES, map, bar, h * kTile + rank * 64, jj * kTile, 0x3);
    } else {
      tma_load_2d(dst, map, bar, h * kTile, jj * kTile);
      tma_load_2d(dst + HALF_BYTES, map, bar, h * kTile + 64, jj * kTile);
    }
  };

  if (warp == 0 && lane == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], kEmptyCount);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], kEmptyCount);
    }
    for (int b = 0; b < SBUF; ++b) mbar_init(&bars->s_full[b], 1);
    for (int b = 0; b < SBUF; ++b)
      mbar_init(&bars->p_full[b], SOFTMAX_THREADS / 32);  // one arrival per softmax warp
    mbar_init(&bars->o_done, 1);
    mbar_init(&bars->o_last, 1);
    mbar_init(&bars->o_free, SOFTMAX_THREADS);
    fence_barrier_init();
    tma_prefetch_desc(&qm);
    tma_prefetch_desc(&km);
    tma_prefetch_desc(&vm);
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // both CTAs' barriers exist before any multicast lands
  tc_fence_after();
  const uint32_t tbase = bars->tmem_base;
#ifdef FO_CS_TIMING
  if (threadIdx.x == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_cs_timing[16 * blockIdx.x] = global_ns();
    g_cs_timing[16 * blockIdx.x + 2] = smid;
    g_cs_timing[16 * blockIdx.x + 3] = 0;
    g_cs_timing[16 * blockIdx.x + 8] = 0;
    g_cs_timing[16 * blockIdx.x + 9] = 0;
    g_cs_timing[16 * blockIdx.x + 10] = 0;
    g_cs_timing[16 * blockIdx.x + 11] = 0;
  }
#endif
  pdl_release_and_wait();
  const int n_items = *p.n_items;
  const int n_waves = *p.n_waves;  // plan schedule: CTA b's k-th item is sched[k * grid + b]
  (void)n_items;
  const size_t head_sym = (size_t)p.comp_rows * p.row_stride;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    int kst = 0, kph = 0, vst = 0, vph = 0, qi = 0;
    ItemCursor sched_cur(p.sched, p.items, n_waves, slot, nslots);
    for (int k = 0; k < n_waves; ++k, ++qi) {
      int w;
      int2 it;
      if (!sched_cur.next(k, w, it)) break;
      const int h = it.x >> 20, i = it.x & 0xFFFFF, ib = i + rank;
#ifdef FO_CS_TIMING
      const unsigned long long tq0 = global_ns();
#endif
      mbar_wait_small(&bars->q_empty, (qi & 1) ^ 1, p.status);
#ifdef FO_CS_TIMING
      if (lane == 0 && k > 0) g_cs_timing[16 * blockIdx.x + 8] += global_ns() - tq0;
#endif
      if (elect_one()) {
        mbar_arrive_expect_tx(&bars->q_full, TILE_BYTES);
        tma_load_2d(sQ, &qm, &bars->q_full, h * kTile, ib * kTile);
        tma_load_2d(sQ + HALF_BYTES, &qm, &bars->q_full, h * kTile + 64, ib * kTile);
        // the next item's Q into L2 now: its load is only issued once this
        // item's last QK is done, and from HBM it would stall the next item's
        // first QK by ~1 us
        if (sched_cur.peek_w() >= 0) {
          const int2 itn = sched_cur.peek_item();
          tma_prefetch_l2_2d(&qm, (itn.x >> 20) * kTile, ((itn.x & 0xFFFFF) + rank) * kTile);
          tma_prefetch_l2_2d(&qm, (itn.x >> 20) * kTile + 64, ((itn.x & 0xFFFFF) + rank) * kTile);
        }
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
          mbar_wait_small(&bars->k_empty[kst], kph ^ 1, p.status);
          if (elect_one()) {
            mbar_arrive_expect_tx(&bars->k_full[kst], TILE_BYTES);
            uint8_t* dk = sK + kst * TILE_BYTES;
            load_tile(dk, &km, &bars->k_full[kst], h, jj);
          }
          __syncwarp();
          if (++kst == KST) {
            kst = 0;
            kph ^= 1;
          }
          if (!FO_CS_VPROD) {
            mbar_wait_small(&bars->v_empty[vst], vph ^ 1, p.status);
            if (elect_one()) {
              mbar_arrive_expect_tx(&bars->v_full[vst], TILE_BYTES);
              uint8_t* dv = sV + vst * V_STAGE_BYTES;
              load_tile(dv, &vm, &bars->v_full[vst], h, jj);
            }
            __syncwarp();
            if (++vst == VST) {
              vst = 0;
              vph ^= 1;
            }
          }
        }
      }
    }
  } else if (FO_CS_VPROD && warp == 3) {
    // ------------------------------------------------------------ V producer: walks the
    // same item / key-block sequence as the K producer, so a K load never queues
    // behind a V load waiting for its stage (QK runs ahead of PV)
    int vst = 0, vph = 0;
    ItemCursor sched_cur(p.sched, p.items, n_waves, slot, nslots);
    for (int k = 0; k < n_waves; ++k) {
      int w;
      int2 it;
      if (!sched_cur.next(k, w, it)) break;
      const int h = it.x >> 20, i = it.x & 0xFFFFF;
      const uint8_t* sym = p.s_s + h * head_sym;
      for (int base = 0; base < p.t_kv; base += 32) {
        const int j = base + lane;
        const uint32_t bit =
            (j < p.t_kv) && (p.dense || decode_reduction(sym, p.row_stride, i, j, p.pool_n));
        uint32_t m = __ballot_sync(0xffffffffu, bit);
        while (m) {
          const int jj = base + __ffs(m) - 1;
          m &= m - 1;
          mbar_wait_small(&bars->v_empty[vst], vph ^ 1, p.status);
          if (elect_one()) {
            mbar_arrive_expect_tx(&bars->v_full[vst], TILE_BYTES);
            uint8_t* dv = sV + vst * V_STAGE_BYTES;
            load_tile(dv, &vm, &bars->v_full[vst], h, jj);
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
    {
      const uint32_t idesc_qk = make_idesc_bf16(128, 128, false, false);
      // ONESCOL: N = 144 = V's 128 columns + 16 of the ones strip (row sums at 128..143)
      const uint32_t idesc_pv = make_idesc_bf16(128, FO_CS_ONESCOL ? 144 : 128, false, true);
      const uint32_t idesc_l = make_idesc_bf16(128, 16, false, false);
      const uint64_t ones_desc = make_sdesc_sw128(smem_u32(sOnes), 16, 1024);
      (void)idesc_l;
      (void)ones_desc;
      int kst = 0, kph = 0, vst = 0, vph = 0, qi = 0;
      uint32_t qk_cnt = 0, pv_cnt = 0;
      const uint64_t qdesc = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t kdesc0 = make_sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t vdesc0 = make_sdesc_sw128(smem_u32(sV), HALF_BYTES, 1024);
      auto issue_qk = [&]() {
        mbar_wait_small(&bars->k_full[kst], kph, p.status);
        tc_fence_after();
        const uint32_t sb = qk_cnt % SBUF;
        const uint32_t d = tbase + TM_S0 + sb * 128;
        const uint64_t kdesc = kdesc0 + (uint64_t)((kst * TILE_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t off = (uint64_t)((k >> 2) * (HALF_BYTES >> 4) + (k & 3) * 2);
            mma_bf16_ss(d, qdesc + off, kdesc + off, idesc_qk, k > 0);
          }
          if (PAIR)
            tc_commit_mc(&bars->k_empty[kst], 0x3);  // released in both CTAs' view
          else
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
      ItemCursor sched_cur(p.sched, p.items, n_waves, slot, nslots);
#ifdef FO_CS_TIMING
      unsigned long long t_pvl = 0;
#endif
      for (int k = 0; k < n_waves; ++k, ++qi) {
        int w;
        int2 it;
        if (!sched_cur.next(k, w, it)) break;
        const int n = it.y;
        mbar_wait_small(&bars->q_full, qi & 1, p.status);
#ifdef FO_CS_TIMING
        if (lane == 0 && k > 0) g_cs_timing[16 * blockIdx.x + 9] += global_ns() - t_pvl;
#endif
        tc_fence_after();
        // QK runs SBUF - 1 tiles ahead of PV; Q is released after the item's last QK
        const int la = n < SBUF - 1 ? n : SBUF - 1;
        for (int a = 0; a < la; ++a) issue_qk();
#ifdef FO_CS_TIMING
        if (k > 0) {
          const unsigned long long t0 = global_ns();
          const uint32_t c = qk_cnt - la;
          while (!mbar_try_wait(&bars->s_full[c % SBUF], (c / SBUF) & 1)) {
          }
          if (lane == 0) g_cs_timing[16 * blockIdx.x + 11] += global_ns() - t0;
        }
#endif
        if (la == n) commit_q_empty();
        for (int j = 0; j < n; ++j) {
          if (j + la < n) {
            issue_qk();
            if (j + la + 1 == n) commit_q_empty();
          }
          mbar_wait_small(&bars->p_full[pv_cnt % SBUF], (pv_cnt / SBUF) & 1, p.status);
          if (j == 0 && qi > 0) mbar_wait_small(&bars->o_free, (qi - 1) & 1, p.status);
          mbar_wait_small(&bars->v_full[vst], vph, p.status);
          tc_fence_after();
          const uint32_t a_t = tbase + TM_S0 + (pv_cnt % SBUF) * 128;
          const uint64_t vdesc = vdesc0 + (uint64_t)((vst * V_STAGE_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              mma_bf16_ts(tbase + TM_O, a_t + k * 8, vdesc + (uint64_t)(k * (2048 >> 4)), idesc_pv,
                          (j > 0 || k > 0));
#if FO_CS_TC_ROWSUM && !FO_CS_ONESCOL
            // row sums on the tensor core: L += P . 1, so l is exactly sum(bf16(P))
#pragma unroll
            for (int k = 0; k < 8; ++k)
              mma_bf16_ts(tbase + TM_L, a_t + k * 8, ones_desc, idesc_l, (j > 0 || k > 0));
#endif
            if (PAIR)
              tc_commit_mc(&bars->v_empty[vst], 0x3);
            else
              tc_commit(&bars->v_empty[vst]);
            // o_done: PV_j complete, awaited by softmax step j + 1 of this item;
            // the item's last PV signals o_last (the epilogue) instead
            if (j + 1 < n) tc_commit(&bars->o_done);
            else tc_commit(&bars->o_last);
          }
          __syncwarp();
          if (++vst == VST) {
            vst = 0;
            vph ^= 1;
          }
          ++pv_cnt;
        }
#ifdef FO_CS_TIMING
        t_pvl = global_ns();
#endif
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------- softmax + epilogue (column groups)
    const int half = (warp - 4) >> 2;  // column group: key columns [NCOL*half, NCOL*half + NCOL)
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const int last_valid = p.S - (p.t_kv - 1) * kTile;  // valid key columns of the last block
    const int col0 = half * NCOL;
    const size_t HD = (size_t)p.H * kTile;
    const size_t stack_stride = (size_t)p.S * HD;
    const int pair_bar = 1 + q4;  // named barrier of the SPLIT warps of lane quarter q4
    const uint32_t xmax_u32 = smem_u32(&bars->xmax[0][0][0]);
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    uint32_t qk_seen = 0, o_base = 0;
    int qi = 0;
    ItemCursor sched_cur(p.sched, p.items, n_waves, slot, nslots);
    // the next item's record and cache counter are fetched before this item's
    // epilogue stores: a global load or atomic issued behind 8 uncoalesced
    // 16-B stores per thread waits for them to drain (~0.9 us per item)
    auto valid_of = [&](int2 itv) {
      return (p.cache && p.valid) ? p.valid[(size_t)(itv.x >> 20) * p.t_q + (itv.x & 0xFFFFF)] : 0;
    };
    int w_cur;
    int2 it_cur;
    bool have = sched_cur.next(0, w_cur, it_cur);
    int valid_cur = have ? valid_of(it_cur) : 0;
#ifdef FO_CS_TIMING
    const bool tmr = threadIdx.x == 128;
    unsigned long long t_mark = 0, g_a = 0, g_b = 0, g_c = 0, n_it = 0;
    long long g_sw = 0, g_sb = 0, g_st = 0;  // steady-state tiles: S wait, softmax busy (cycles)
    long long g_ph[5] = {0, 0, 0, 0, 0};      // softmax phases (cycles)
    long long g_ep[6] = {0, 0, 0, 0, 0, 0};   // epilogue sub-phases (cycles)
    long long te_prev = 0;
#endif
    for (int k = 0; have; ++k, ++qi) {
      const int2 it = it_cur;
      const int h = it.x >> 20, i = it.x & 0xFFFFF, n = it.y;
      const bool tail = (last_valid < kTile) &&
                        (p.dense || decode_reduction(p.s_s + h * head_sym, p.row_stride, i,
                                                     p.t_kv - 1, p.pool_n));
      const int valid_old = valid_cur;
      float m_run = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);
      for (int j = 0; j < n; ++j) {
        const uint32_t sb = qk_seen % SBUF;
#ifdef FO_CS_TIMING
        if (tmr && j == 0 && t_mark) g_cs_timing[16 * blockIdx.x + 10] += global_ns() - t_mark;
#endif
#ifdef FO_CS_TIMING
        const long long tw0 = clock64();
#endif
        mbar_wait_small(&bars->s_full[sb], (qk_seen / SBUF) & 1, p.status);
#ifdef FO_CS_TIMING
        const long long tw1 = clock64();
        if (tmr && j > 0) g_sw += tw1 - tw0;  // steady-state wait for S
        if (tmr && j == 0 && t_mark) {
          const unsigned long long t = global_ns();
          g_c += t - t_mark;  // epilogue end -> first S
        }
#endif
        tc_fence_after();
        const uint32_t sa = tbase + lane_off + TM_S0 + sb * 128;
        const bool mask_tail = tail && (j == n - 1);
        uint32_t u[NCH][32];
#pragma unroll
        for (int c = 0; c < NCH; ++c) tmem_ld32(sa + col0 + 32 * c, u[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < NCH; ++c) reg_fence_cs(u[c]);
#ifdef FO_CS_TIMING
        const long long tp1 = clock64();
#endif
        float sv[NCOL];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 32; ++k) sv[c * 32 + k] = __uint_as_float(u[c][k]);
        if (mask_tail) {
#pragma unroll
          for (int k = 0; k < NCOL; ++k)
            if (col0 + k >= last_valid) sv[k] = -INFINITY;
        }
        // partial row max: FMNMX3 chains of 16, then exchange with the partner warps
        float mc[NCOL / 16];
#pragma unroll
        for (int c = 0; c < NCOL / 16; ++c) {
          float a = fmax3f(sv[16 * c], sv[16 * c + 1], sv[16 * c + 2]);
#pragma unroll
          for (int k = 3; k < 15; k += 2) a = fmax3f(a, sv[16 * c + k], sv[16 * c + k + 1]);
          mc[c] = fmaxf(a, sv[16 * c + 15]);
        }
        float mh = mc[0];
#pragma unroll
        for (int c = 1; c < NCOL / 16; ++c) mh = fmaxf(mh, mc[c]);
        const uint32_t xa = xmax_u32 + (((qk_seen & 1) * SPLIT) * 128 + r) * 4;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(xa + half * 512), "f"(mh) : "memory");
        // all partners have read their S columns before any overwrites S with P
        named_bar_sync(pair_bar, 32 * SPLIT);
        float mo = -INFINITY;
#pragma unroll
        for (int g = 0; g < SPLIT; ++g) {
          if (g == half) continue;
          float v;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(xa + g * 512) : "memory");
          mo = fmaxf(mo, v);
        }
#ifdef FO_CS_TIMING
        asm volatile("" : "+f"(mo));
        const long long tp2 = clock64();
#endif
        ++qk_seen;
        const float m_tile = fmaxf(mh, mo) * p.scale_log2;
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
        l2.x *= corr;  // the running sum moves to the new max before this tile adds to it
        l2.y *= corr;
        const float2 nm2 = make_float2(-m_new, -m_new);
        uint32_t pk[NCOL / 2];
        // one copy of the exp loop (the softmax loop is sensitive to its code size;
        // a separate MUFU-only copy for the masked tail tile cost 1.7%): masked
        // tail columns are -inf, which the polynomial clamps to 2^-127 instead of 0
        (void)mask_tail;
#pragma unroll
        for (int q = 0; q < NCOL / 2; ++q) {
          const float2 x = ffma2(make_float2(sv[2 * q], sv[2 * q + 1]), sc2, nm2);
          float2 e;
#ifdef FO_CS_POLY_MASK  // which pairs of every 16 take the polynomial (interleave pattern)
          if ((FO_CS_POLY_MASK >> (q & 15)) & 1) {
#else
          if ((q & 15) < FO_CS_POLY_OF_16) {
#endif
            e = exp2_poly2(x);
          } else {
            e.x = fast_exp2(x.x);
            e.y = fast_exp2(x.y);
          }
          if (!FO_CS_TC_ROWSUM) l2 = fadd2(l2, e);
          pk[q] = pack_bf16x2(e.x, e.y);
        }
#ifdef FO_CS_TIMING
        reg_fence_cs(pk);
        const long long tp3 = clock64();
#endif
#if FO_CS_SPLIT == 2
        tmem_st32(sa + half * 32, pk);
#else
        tmem_st16(sa + half * 16, pk);
#endif
        tmem_st_wait();
#ifdef FO_CS_TIMING
        const long long tp4 = clock64();
#endif
#if FO_CS_ODONE_ALL
        // every o_done phase is awaited (PV_{j-1} has long finished by the time
        // P_j is stored, so this costs nothing) and no phase goes unobserved
        if (j > 0) mbar_wait_small(&bars->o_done, (o_base + j - 1) & 1, p.status);
        if (j > 0 && __any_sync(0xffffffffu, need)) {
#else
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          // PV_{j-1} must be complete before O can be rescaled for P_j (see fo_attention.cu)
          mbar_wait_small(&bars->o_done, (o_base + j - 1) & 1, p.status);
#endif
          tc_fence_after();
          const uint32_t oa = tbase + lane_off + TM_O + col0;
#pragma unroll 1
          for (int c = 0; c < NCH; ++c) {  // this warp's columns of O (rare path: kept compact)
            uint32_t o[32];
            tmem_ld32(oa + c * 32, o);
            tmem_ld_wait();
            reg_fence_cs(o);
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * corr);
            tmem_st32(oa + c * 32, o);
          }
          if (FO_CS_TC_ROWSUM && half == 0) {  // and the row-sum columns
            uint32_t l16[16];
            tmem_ld16(tbase + lane_off + TM_L, l16);
            tmem_ld_wait();
            reg_fence_cs(l16);
#pragma unroll
            for (int k = 0; k < 16; ++k) l16[k] = __float_as_uint(__uint_as_float(l16[k]) * corr);
            tmem_st16(tbase + lane_off + TM_L, l16);
          }
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();  // every lane's P / O stores are complete (tcgen05.wait::st above)
        if (lane == 0) mbar_arrive(&bars->p_full[sb]);
#ifdef FO_CS_TIMING
        if (tmr && j > 0) {
          const long long tp5 = clock64();
          g_sb += tp5 - tw1;  // S landed -> P stored (softmax busy)
          ++g_st;
          g_ph[0] += tp1 - tw1;  // S: TMEM -> registers
          g_ph[1] += tp2 - tp1;  // row max + partner exchange
          g_ph[2] += tp3 - tp2;  // exponentials + pack
          g_ph[3] += tp4 - tp3;  // P: registers -> TMEM
          g_ph[4] += tp5 - tp4;  // rescale check, arrive
        }
#endif
      }
      // ---------------- epilogue: this half of O / l -> bf16 -> HBM (+ cache push)
#ifdef FO_CS_TIMING
      if (tmr) t_mark = global_ns();
#endif
      mbar_wait_small(&bars->o_last, qi & 1, p.status);
#ifdef FO_CS_TIMING
      if (tmr) {
        const unsigned long long t = global_ns();
        g_a += t - t_mark;  // last P stored -> last PV complete
        t_mark = t;
        ++n_it;
      }
#endif
      o_base += n - 1;  // o_done phases of this item
      tc_fence_after();
#ifdef FO_CS_TIMING
      te_prev = clock64();
      auto ep_mark = [&](int k) {
        const long long t = clock64();
        if (tmr) g_ep[k] += t - te_prev;
        te_prev = t;
      };
#define FO_EP_MARK(k) ep_mark(k)
#else
#define FO_EP_MARK(k) ((void)0)
#endif
      float l_row;
      if (FO_CS_TC_ROWSUM) {
        uint32_t lsum[16];
        tmem_ld16(tbase + lane_off + TM_L, lsum);
        tmem_ld_wait();
        reg_fence_cs(lsum);
        l_row = __uint_as_float(lsum[0]);
      } else {
        // combine the two halves' partial sums (both scaled by the same maxima)
        bars->xsum[half][r] = l2.x + l2.y;  // SPLIT == 2 here (static_assert above)
        named_bar_sync(pair_bar, 64);
        l_row = bars->xsum[0][r] + bars->xsum[1][r];
      }
      const float inv_l = 1.f / l_row;
      FO_EP_MARK(0);  // l from TMEM
      const int ib = i + rank;  // this CTA's query block (a pair's missing partner: ib == t_q)
      const int row = ib * kTile + r;
      const bool row_ok = row < p.S;
      const int vn = min(valid_old + 1, p.order_d + 1);
      {
        int w_n;
        int2 it_n;
        have = sched_cur.next(k + 1, w_n, it_n);
        it_cur = it_n;
        valid_cur = have ? valid_of(it_n) : 0;
      }
      if (r == 0 && half == 0) {
#ifdef FO_CS_TIMING
        atomicAdd(&g_cs_timing[16 * blockIdx.x + 3], (unsigned long long)n);
#endif
        if (p.pairs && ib < p.t_q)
          atomicAdd(reinterpret_cast<unsigned long long*>(&p.pairs[h]),
                    static_cast<unsigned long long>(n));
        if (p.cache && p.valid) p.valid[(size_t)h * p.t_q + ib] = vn;
      }
      FO_EP_MARK(1);  // next item's record, counters
      const uint32_t oa = tbase + lane_off + TM_O + col0;
#if FO_CS_TMA_OUT
      // this warp's staging box: rows q4*32.., its columns; chunk q of row r at
      // q ^ ((r >> 1) & 3) (SW64, conflict-free for 8 consecutive rows)
      const int wslot = warp - 4;
      const uint32_t ost = smem_u32(sOst) + wslot * 2048 + lane * 64;
      const int osw = (lane >> 1) & 3;
#endif
#pragma unroll 1
      for (int c = 0; c < NCH; ++c) {
        uint32_t o[32];
        tmem_ld32(oa + c * 32, o);
        tmem_ld_wait();
        reg_fence_cs(o);
        FO_EP_MARK(2 + 2 * c);  // O chunk from TMEM (c = 0: marks 2, c = 1: marks 4)
        float of[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) of[k] = __uint_as_float(o[k]) * inv_l;
#if FO_CS_TMA_OUT
        {
          uint4 pk4[4];
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            pk4[v4].x = pack_bf16x2(of[v4 * 8 + 0], of[v4 * 8 + 1]);
            pk4[v4].y = pack_bf16x2(of[v4 * 8 + 2], of[v4 * 8 + 3]);
            pk4[v4].z = pack_bf16x2(of[v4 * 8 + 4], of[v4 * 8 + 5]);
            pk4[v4].w = pack_bf16x2(of[v4 * 8 + 6], of[v4 * 8 + 7]);
          }
          // the previous store from this box has read it (usually long done)
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) sts128(ost + ((v4 ^ osw) << 4), pk4[v4]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {  // rows past the end of the sequence are clipped by the TMA unit
            tma_store_2d(&om, sOst + wslot * 2048, h * kTile + col0 + c * 32, ib * kTile + q4 * 32);
            bulk_commit();
          }
        }
#endif
        if (row_ok) {
          const size_t off = (size_t)row * HD + (size_t)h * kTile + col0 + c * 32;
#if !FO_CS_TMA_OUT
          uint4 pk4[4];
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            pk4[v4].x = pack_bf16x2(of[v4 * 8 + 0], of[v4 * 8 + 1]);
            pk4[v4].y = pack_bf16x2(of[v4 * 8 + 2], of[v4 * 8 + 3]);
            pk4[v4].z = pack_bf16x2(of[v4 * 8 + 4], of[v4 * 8 + 5]);
            pk4[v4].w = pack_bf16x2(of[v4 * 8 + 6], of[v4 * 8 + 7]);
          }
          st_global_256(p.out + off, pk4[0], pk4[1]);
          st_global_256(p.out + off + 16, pk4[2], pk4[3]);
#endif
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
      FO_EP_MARK(3);  // the last chunk's scale, pack, stage, TMA store (chunk 0's land in 3 too)
      tc_fence_before();
      mbar_arrive(&bars->o_free);
      FO_EP_MARK(5);
#undef FO_EP_MARK
#ifdef FO_CS_TIMING
      if (tmr) {
        const unsigned long long t = global_ns();
        g_b += t - t_mark;  // epilogue
        t_mark = t;
      }
#endif
    }
#ifdef FO_CS_TIMING
    if (tmr) {
      g_cs_timing[16 * blockIdx.x + 4] = g_a;
      g_cs_timing[16 * blockIdx.x + 5] = g_b;
      g_cs_timing[16 * blockIdx.x + 6] = g_c;
      g_cs_timing[16 * blockIdx.x + 7] = n_it;
      g_cs_timing[16 * blockIdx.x + 12] = g_sw;
      g_cs_timing[16 * blockIdx.x + 13] = g_sb;
      g_cs_timing[16 * blockIdx.x + 14] = g_st;
      for (int k = 0; k < 5; ++k) g_cs_ph[5 * blockIdx.x + k] = g_ph[k];
      for (int k = 0; k < 6; ++k) g_cs_ep[6 * blockIdx.x + k] = g_ep[k];
    }
#endif
#if FO_CS_TMA_OUT
    if (lane == 0) bulk_wait<0>();  // this warp's O stores are complete
    __syncwarp();
#endif
    if (p.fc_cache)
      forecast_cached_tiles<SOFTMAX_THREADS>(p, threadIdx.x - 128, 8, &bars->fc_tile);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal into it
#ifdef FO_CS_TIMING
  if (threadIdx.x == 0) g_cs_timing[16 * blockIdx.x + 1] = global_ns();
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

#ifdef FO_CS_TIMING
extern "C" __attribute__((visibility("default"))) int fo_debug_cs_timing(unsigned long long* out,
                                                                       int n) {
  return (int)cudaMemcpyFromSymbol(out, g_cs_timing, sizeof(unsigned long long) * 16 * n);
}
extern "C" __attribute__((visibility("default"))) int fo_debug_cs_epilogue(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_cs_ep, sizeof(long long) * 6 * n);
}
extern "C" __attribute__((visibility("default"))) int fo_debug_cs_phases(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_cs_ph, sizeof(long long) * 5 * n);
}
#endif

void launch_attention_cs(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                         const CUtensorMap& om, const AttnParams& p, int grid, bool pair,
                         cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(sparse_attention_cs_kernel<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, attn_cs::SMEM_BYTES);
    cudaFuncSetAttribute(sparse_attention_cs_kernel<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, attn_cs::SMEM_BYTES);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (FO_PDL) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // fo_common.cuh
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (pair) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  cfg.gridDim = dim3(pair ? grid & ~1 : grid);
  cfg.blockDim = dim3(attn_cs::NTHREADS);
  cfg.dynamicSmemBytes = attn_cs::SMEM_BYTES;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  note_launch();
  if (pair)
    cudaLaunchKernelEx(&cfg, sparse_attention_cs_kernel<true>, qm, km, vm, om, p);
  else
    cudaLaunchKernelEx(&cfg, sparse_attention_cs_kernel<false>, qm, km, vm, om, p);
}

}  // namespace fo
