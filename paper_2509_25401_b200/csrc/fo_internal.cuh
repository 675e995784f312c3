// Internal declarations shared by the kernel translation units and the C-ABI.
#pragma once
#include "fo_common.cuh"

namespace fo {

// counts every kernel launch the library makes (fo_kernel_launches in the C ABI)
void note_launch();

__host__ __device__ constexpr int ceil_div_d(int a, int b) { return (a + b - 1) / b; }

// Per-layer schedule derived from the symbols (built by plan_kernel).
struct PlanView {
  int* counts;                // [0] attention items, [1] GEMM-Q (= active) tiles,
                              // [2] fused-forecast tile cursor, [3] CTAs done (both self-resetting),
                              // [4] 1: items cover CTA pairs of query blocks (pool_n even),
                              // [5] attention schedule slots per wave (CTAs or clusters),
                              // [6] attention waves of the balanced schedule,
                              // [7] GEMM-Q jobs (gq_jobs)
  int2* items;                // [H*rows] attention work: x = (h<<20)|i, y = #KV blocks; sorted desc
  int* gq_items;              // [H*rows] GEMM-Q tiles (h<<20)|i in (block, head) order, then
                              // the cached tiles in the same order from index counts[1]
  unsigned long long* hmask;  // [rows] bit h set = head h computed for block i
  int* orders;                // [rows] cached-bias orders per block (0 = no cached heads)
  long long* pairs_pred;      // [H] mask-predicted computed pairs
  int* scratch;               // [H*rows] plan-internal scratch (per-row KV counts)
  int* att_sched;             // [H*rows + 1024] attention item of (wave k, CTA b) at k*P + b, -1 none
  int2* gq_jobs;              // [gq_jobs_cap] GEMM-Q jobs of the CTA-pair kernel (counts[7] of
                              // them): x = i0 | (i1 + 1) << 16 (query blocks of CTA 0 / 1, i1 = -1:
                              // none), y = h | n256 << 8 (n256: heads h, h+1 as one N=256 tile,
                              // else head h alone, N=128); ordered by i0
};

// GEMM-Q job capacity: per head pair, three block lists (both heads / only the
// first / only the second active) cut into jobs of two blocks
__host__ __device__ inline int gq_jobs_cap(int H, int rows) {
  return H * rows / 2 + 3 * ((H + 1) / 2) + 64;
}

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline size_t plan_layout(int H, int rows, char* base, PlanView* pv) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align16(off + bytes);
    return o;
  };
  size_t o_counts = take(8 * sizeof(int));
  size_t o_items = take((size_t)H * rows * sizeof(int2));
  size_t o_gq = take((size_t)H * rows * sizeof(int));
  size_t o_hm = take((size_t)rows * sizeof(unsigned long long));
  size_t o_ord = take((size_t)rows * sizeof(int));
  size_t o_pairs = take((size_t)H * sizeof(long long));
  size_t o_scr = take((size_t)H * rows * sizeof(int));
  size_t o_sched = take(((size_t)H * rows + 1024) * sizeof(int));
  size_t o_gq2 = take(2 * (size_t)gq_jobs_cap(H, rows) * sizeof(int2));  // + sort scratch
  if (pv) {
    pv->counts = reinterpret_cast<int*>(base + o_counts);
    pv->items = reinterpret_cast<int2*>(base + o_items);
    pv->gq_items = reinterpret_cast<int*>(base + o_gq);
    pv->hmask = reinterpret_cast<unsigned long long*>(base + o_hm);
    pv->orders = reinterpret_cast<int*>(base + o_ord);
    pv->pairs_pred = reinterpret_cast<long long*>(base + o_pairs);
    pv->scratch = reinterpret_cast<int*>(base + o_scr);
    pv->att_sched = reinterpret_cast<int*>(base + o_sched);
    pv->gq_jobs = reinterpret_cast<int2*>(base + o_gq2);
  }
  return off;
}

__global__ void encode_symbols_kernel(const uint8_t* cache_bits, const uint8_t* skip_bits, int H,
                                      int rows, int cols, int pool_n, uint8_t* s_c, uint8_t* s_s,
                                      uint32_t* status);
__global__ void decode_symbols_kernel(const uint8_t* s_c, const uint8_t* s_s, int H, int rows,
                                      int cols, int pool_n, uint8_t* active, uint8_t* pair_bits);
__global__ void plan_kernel(const uint8_t* s_c, const uint8_t* s_s, int H, int rows, int cols,
                            int pool_n, int dense, const int32_t* valid, int order_d, int ctas,
                            int pair_items, PlanView pv, uint32_t* status);
// CTA-pair attention with K/V multicast: sparse plans over even pool_n (their
// query blocks 2c, 2c+1 share one compressed skip row)
#ifndef FO_ATTN_PAIR
#define FO_ATTN_PAIR 1
#endif
inline bool attention_pairs(int pool_n, int dense) { return FO_ATTN_PAIR && !dense && pool_n % 2 == 0; }
__global__ void compare_active_kernel(const uint8_t* s_c_a, const uint8_t* s_c_b, int H, int rows,
                                      int pool_n, uint32_t* status);

// ---------------------------------------------------------------------------
// attention
// ---------------------------------------------------------------------------
constexpr int kTile = 128;  // b_q = b_k = 128 tokens, head_dim 128

struct AttnParams {
  int S, H, t_q, t_kv, pool_n, comp_rows, row_stride;
  int dense;  // update mode: every (h, i, j) computed
  float scale_log2;
  const uint8_t* s_s;
  const int2* items;
  const int* n_items;
  const int* sched;       // plan att_sched: item of (wave k, CTA b) at k*gridDim.x + b
  const int* n_waves;     // plan counts[6]
  __nv_bfloat16* out;     // [S, H*128]
  __nv_bfloat16* cache;   // update mode: [order+1, S, H*128] diff stacks (in place) or null
  int32_t* valid;         // update mode: [H, t_q] valid orders or null
  int order_d;
  long long* pairs;       // [H] instrumented computed pairs, or null
  uint32_t* status;
  long long* dbg;         // FO_ATTN_TIMING builds: per-CTA phase cycle counters
  // fused OP_reuse (mode="materialize"): once a CTA's attention items are done,
  // its softmax warps forecast cached tiles into `out` (fc_cache null = off)
  const __nv_bfloat16* fc_cache;  // [order+1, S, H*128] diff stacks
  const int32_t* fc_valid;        // [H, t_q]
  int* fc_counts;                 // plan counts: [1] active tiles, [2] cursor, [3] CTAs done
  const int* fc_tiles;            // plan gq_items (cached tiles from index counts[1])
  float fc_coef[4];
};

// OP_reuse for the cached tiles of one layer (attention.py:96-113,212-216):
// out[tile] = sum_{d < min(order+1, valid)} coef[d] * stack[d][tile]. Run by
// the NT softmax threads of every CTA after its attention items: tiles are
// taken from a global cursor, so CTAs that finish their items early absorb
// the forecast work. Each thread streams 2048/NT 16-byte chunks per tile with
// all loads in flight. The last CTA out resets the cursor (graph replays).
template <int NT>
__device__ __forceinline__ void forecast_cached_tiles(const AttnParams& p, int s, int bar_id,
                                                      int* sh_tile) {
  constexpr int PER = 4;  // 16-byte chunks per thread in flight (x up to 4 orders)
  const int n_cached = p.H * p.t_q - p.fc_counts[1];
  const size_t HD = (size_t)p.H * kTile, SS = (size_t)p.S * HD;
  for (;;) {
    if (s == 0) *sh_tile = atomicAdd(&p.fc_counts[2], 1);
    named_bar_sync(bar_id, NT);
    const int k = *sh_tile;
    named_bar_sync(bar_id, NT);
    if (k >= n_cached) break;
    const int code = p.fc_tiles[p.fc_counts[1] + k];
    const int h = code >> 20, i = code & 0xFFFFF;
    const int n = min(p.order_d + 1, p.fc_valid[(size_t)h * p.t_q + i]);
    const int chunks = min(kTile, p.S - i * kTile) * 16;
#pragma unroll 1
    for (int e0 = s; e0 < chunks; e0 += PER * NT) {
    uint4 w[PER][4];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = e0 + u * NT;
      const size_t off = (size_t)(i * kTile + (e >> 4)) * HD + (size_t)h * kTile + (e & 15) * 8;
#pragma unroll
      for (int d = 0; d < 4; ++d)
        if (e < chunks && d < n)
          w[u][d] = __ldcs(reinterpret_cast<const uint4*>(p.fc_cache + d * SS + off));
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = e0 + u * NT;
      if (e >= chunks) continue;
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        if (d >= n) break;
        const uint32_t w4[4] = {w[u][d].x, w[u][d].y, w[u][d].z, w[u][d].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2 * q] = fmaf(p.fc_coef[d], bf16lo(w4[q]), acc[2 * q]);
          acc[2 * q + 1] = fmaf(p.fc_coef[d], bf16hi(w4[q]), acc[2 * q + 1]);
        }
      }
      uint4 pk;
      pk.x = pack_bf16x2(acc[0], acc[1]);
      pk.y = pack_bf16x2(acc[2], acc[3]);
      pk.z = pack_bf16x2(acc[4], acc[5]);
      pk.w = pack_bf16x2(acc[6], acc[7]);
      const size_t off = (size_t)(i * kTile + (e >> 4)) * HD + (size_t)h * kTile + (e & 15) * 8;
      __stcs(reinterpret_cast<uint4*>(p.out + off), pk);
    }
    }
  }
  if (s == 0) {
    __threadfence();
    if (atomicAdd(&p.fc_counts[3], 1) == (int)gridDim.x - 1) {
      p.fc_counts[2] = 0;
      p.fc_counts[3] = 0;
      __threadfence();
    }
  }
}

void launch_attention(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                      const AttnParams& p, int grid, cudaStream_t stream);
// two softmax warpgroups splitting every tile's key columns (fo_attention_cs.cu)
void launch_attention_cs(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                         const CUtensorMap& om, const AttnParams& p, int grid, bool pair,
                         cudaStream_t stream);

// ---------------------------------------------------------------------------
// GEMMs
// ---------------------------------------------------------------------------
struct GemmQParams {
  int S, dm, H, t_q, dense;
  const int2* jobs;       // sparse phase: plan gq_jobs (CTA-pair jobs, see PlanView)
  const int* n_jobs;      // their count (plan counts[7])
  const float* norm_w;    // [H, 128]
  const float* rope_cos;  // [S, 64]
  const float* rope_sin;  // [S, 64]
  float eps;
  __nv_bfloat16* q;  // [S, H*128]
  // fused dispatch projection (fo_gemm_qkv): W holds [W_q; W_k; W_v] and the
  // launch also runs the dense K (RMSNorm + RoPE) and V (plain) projections
  int qkv;
  __nv_bfloat16* k_out;  // [S, H*128]
  __nv_bfloat16* v_out;  // [S, H*128]
  const float* k_norm;   // [H, 128]
};
// GEMM-Q on CTA pairs (cta_group::2), persistent: every tile of the dense phase
// and of the sparse phase in one launch. xm: x with a 128-row box; wm / wm64:
// W_q with 128- and 64-row boxes (N=256 and N=128 jobs)
void launch_gemm_q2(const CUtensorMap& xm, const CUtensorMap& wm, const CUtensorMap& wm64,
                    const GemmQParams& p, cudaStream_t stream);

struct GemmOParams {
  int S, dm, H, t_q, order_d;
  int update;                            // 1: update (writes bias), 0: dispatch (reads bias)
  int i_begin, i_end;                    // dispatch: query-block range [i_begin, i_end)
  const unsigned long long* hmask;       // [t_q]
  const int* orders;                     // [t_q]
  float coef[4];                         // dispatch forecast coefficients c_d
  __nv_bfloat16* out;                    // [S, dm]
  __nv_bfloat16* bias;                   // [order+1, S, dm]
  uint32_t* status;
};
// dispatch (K4): 2-CTA clusters, bias chunks through a TMA ring
void launch_gemm_o(const CUtensorMap& am, const CUtensorMap& cm, const CUtensorMap& wm,
                   const CUtensorMap& om, const GemmOParams& p, int max_ctas, cudaStream_t stream);
// update (K5): 2-CTA clusters; cm / bm are 3-D [order+1][S][cols] maps
void launch_gemm_o_update(const CUtensorMap& am, const CUtensorMap& cm, const CUtensorMap& wm,
                          const CUtensorMap& om, const CUtensorMap& bm, const GemmOParams& p,
                          cudaStream_t stream);

// elementwise helpers
void launch_forecast_materialize(const __nv_bfloat16* cache, int S, int H, int t_q, int order_d,
                                 const unsigned long long* hmask, const int32_t* valid,
                                 const float* coef, __nv_bfloat16* out, cudaStream_t stream);
void launch_check_finite(const void* data, long long rows, int cols,
                         const unsigned long long* hmask, uint32_t* status, cudaStream_t stream);
void launch_synthetic_x(const float* x0, const float* a, const float* b, size_t n, int kind,
                        float c1, float c2, float s, __nv_bfloat16* out, cudaStream_t stream);
void launch_cache_push(const __nv_bfloat16* o, __nv_bfloat16* cache, int32_t* valid, int S, int H,
                       int t_q, int order_d, const uint8_t* sel, int one_tile,
                       cudaStream_t stream);

// update-step mask policy (fo_policy.cu)
constexpr int kPolicyMaxBlocks = 1024;  // compressed blocks per side
size_t policy_workspace_bytes(int H, int rows_c);
cudaError_t launch_generate_masks(const __nv_bfloat16* q, const __nv_bfloat16* k, int S, int H,
                                  int n_t, int pool_n, double tau_q, double tau_kv, double s_q,
                                  int guard, uint8_t* cache_bits, uint8_t* skip_bits, void* ws,
                                  cudaStream_t stream);
// the reference's policy building blocks one stage at a time (policy.py:21-178)
size_t policy_map_workspace_bytes(int H, int rows_q, int rows_k);
cudaError_t launch_policy_map(const void* q, const void* k, int is_f32, int S_q, int S_k, int H,
                              int d, int pool_q, int pool_k, float* p_tilde, void* ws,
                              cudaStream_t stream);
cudaError_t launch_policy_scores(const float* p_tilde, int H, int rows, int cols, int n_t,
                                 double* contribution, double* guidance, cudaStream_t stream);
cudaError_t launch_policy_select_cached(const double* contribution, const double* guidance, int H,
                                        int V, double tau_q, uint8_t* cached, cudaStream_t stream);
cudaError_t launch_policy_select_skip(const float* p_tilde, const uint8_t* compute, int H, int rows,
                                      int cols, int n_t, double tau_kv, int guard, uint8_t* keep,
                                      cudaStream_t stream);

// tile-level building blocks and dense numerics (fo_numerics.cu)
int max_row_width();
cudaError_t launch_online_softmax_update(const float* m, const float* l, const float* acc,
                                         const float* scores, const float* v, int rows, int cols,
                                         int d, float* m_out, float* l_out, float* acc_out,
                                         cudaStream_t st);
cudaError_t launch_online_softmax_finalize(const float* acc, const float* l, int rows, int d,
                                           float* out, uint32_t* status, cudaStream_t st);
cudaError_t launch_update_entry(const float* old, const float* o, size_t tile, int order, int valid,
                                float* stack, cudaStream_t st);
cudaError_t launch_forecast_entry(const float* stack, size_t tile, int n_orders, const float* coef,
                                  float* out, cudaStream_t st);
cudaError_t launch_mean_pool(const float* x, int n, int d, int pool, float* out, cudaStream_t st);
cudaError_t launch_rms_norm(const float* x, const float* w, int n, int d, double eps, float* out,
                            cudaStream_t st);
cudaError_t launch_rope(const float* x, const float* cs, const float* sn, int n, int d, float* out,
                        cudaStream_t st);
cudaError_t launch_row_softmax(const float* s, int n, int d, float* out, cudaStream_t st);
cudaError_t launch_matmul_f32(const float* a, const float* b, float* c, int m, int n, int k,
                              int accumulate, cudaStream_t st);
cudaError_t launch_masked_block_attention_f32(const float* q, const float* k, const float* v, int n,
                                              int d, const uint8_t* active,
                                              const uint8_t* pair_bits, int b_q, int b_k,
                                              float scale, float* out, unsigned long long* pairs,
                                              uint32_t* status, cudaStream_t st);

}  // namespace fo
