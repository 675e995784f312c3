// Internal declarations shared by the kernel translation units and the C-ABI.
#pragma once
#include "fo_common.cuh"

namespace fo {

__host__ __device__ constexpr int ceil_div_d(int a, int b) { return (a + b - 1) / b; }

// Per-layer schedule derived from the symbols (built by plan_kernel).
struct PlanView {
  int* counts;                // [0] attention items, [1] GEMM-Q tiles
  int2* items;                // [H*rows] attention work: x = (h<<20)|i, y = #KV blocks; sorted desc
  int* gq_items;              // [H*rows] GEMM-Q tiles (h<<20)|i in (block, head) order
  unsigned long long* hmask;  // [rows] bit h set = head h computed for block i
  int* orders;                // [rows] cached-bias orders per block (0 = no cached heads)
  long long* pairs_pred;      // [H] mask-predicted computed pairs
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline size_t plan_layout(int H, int rows, char* base, PlanView* pv) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align16(off + bytes);
    return o;
  };
  size_t o_counts = take(4 * sizeof(int));
  size_t o_items = take((size_t)H * rows * sizeof(int2));
  size_t o_gq = take((size_t)H * rows * sizeof(int));
  size_t o_hm = take((size_t)rows * sizeof(unsigned long long));
  size_t o_ord = take((size_t)rows * sizeof(int));
  size_t o_pairs = take((size_t)H * sizeof(long long));
  if (pv) {
    pv->counts = reinterpret_cast<int*>(base + o_counts);
    pv->items = reinterpret_cast<int2*>(base + o_items);
    pv->gq_items = reinterpret_cast<int*>(base + o_gq);
    pv->hmask = reinterpret_cast<unsigned long long*>(base + o_hm);
    pv->orders = reinterpret_cast<int*>(base + o_ord);
    pv->pairs_pred = reinterpret_cast<long long*>(base + o_pairs);
  }
  return off;
}

__global__ void encode_symbols_kernel(const uint8_t* cache_bits, const uint8_t* skip_bits, int H,
                                      int rows, int cols, int pool_n, uint8_t* s_c, uint8_t* s_s,
                                      uint32_t* status);
__global__ void decode_symbols_kernel(const uint8_t* s_c, const uint8_t* s_s, int H, int rows,
                                      int cols, int pool_n, uint8_t* active, uint8_t* pair_bits);
__global__ void plan_kernel(const uint8_t* s_c, const uint8_t* s_s, int H, int rows, int cols,
                            int pool_n, int dense, const int32_t* valid, int order_d, PlanView pv,
                            uint32_t* status);
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
  __nv_bfloat16* out;     // [S, H*128]
  __nv_bfloat16* cache;   // update mode: [order+1, S, H*128] diff stacks (in place) or null
  int32_t* valid;         // update mode: [H, t_q] valid orders or null
  int order_d;
  long long* pairs;       // [H] instrumented computed pairs, or null
  uint32_t* status;
  long long* dbg;         // FO_ATTN_TIMING builds: per-CTA phase cycle counters
};

void launch_attention(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                      const AttnParams& p, int grid, cudaStream_t stream);
// two softmax warpgroups splitting every tile's key columns (fo_attention_cs.cu)
void launch_attention_cs(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                         const AttnParams& p, int grid, cudaStream_t stream);

// ---------------------------------------------------------------------------
// GEMMs
// ---------------------------------------------------------------------------
struct GemmQParams {
  int S, dm, H, t_q, dense;
  const int* gq_items;
  const int* n_gq;
  const float* norm_w;  // [H, 128]
  const float* rope_cos;  // [S, 64]
  const float* rope_sin;  // [S, 64]
  float eps;
  __nv_bfloat16* q;  // [S, H*128]
};
void launch_gemm_q(const CUtensorMap& xm, const CUtensorMap& wm, const GemmQParams& p, int grid,
                   cudaStream_t stream);

struct GemmOParams {
  int S, dm, H, t_q, order_d;
  int update;                            // 1: update (writes bias), 0: dispatch (reads bias)
  const unsigned long long* hmask;       // [t_q]
  const int* orders;                     // [t_q]
  float coef[4];                         // dispatch forecast coefficients c_d
  __nv_bfloat16* out;                    // [S, dm]
  __nv_bfloat16* bias;                   // [order+1, S, dm]
  uint32_t* status;
};
void launch_gemm_o(const CUtensorMap& am, const CUtensorMap& cm, const CUtensorMap& wm,
                   const CUtensorMap& om, const GemmOParams& p, int grid, cudaStream_t stream);

// elementwise helpers
void launch_forecast_materialize(const __nv_bfloat16* cache, int S, int H, int t_q, int order_d,
                                 const unsigned long long* hmask, const int32_t* valid,
                                 const float* coef, __nv_bfloat16* out, cudaStream_t stream);
void launch_cache_push(const __nv_bfloat16* o, __nv_bfloat16* cache, int32_t* valid, int S, int H,
                       int t_q, int order_d, const uint8_t* sel, cudaStream_t stream);

// update-step mask policy (fo_policy.cu)
constexpr int kPolicyMaxBlocks = 1024;  // compressed blocks per side
size_t policy_workspace_bytes(int H, int rows_c);
cudaError_t launch_generate_masks(const __nv_bfloat16* q, const __nv_bfloat16* k, int S, int H,
                                  int n_t, int pool_n, double tau_q, double tau_kv, double s_q,
                                  int guard, uint8_t* cache_bits, uint8_t* skip_bits, void* ws,
                                  cudaStream_t stream);

}  // namespace fo
