// C ABI (include/flashomni_b200.h): argument validation, TMA descriptor
// construction and kernel launches. No allocation, no synchronisation.
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/flashomni_b200.h"
#include "fo_internal.cuh"

using namespace fo;

namespace fo {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace fo

namespace {
thread_local char g_err[512] = "";

// One NVTX range per compute entry point, named after it (header-only NVTX3:
// a no-op unless a tool such as ncu / nsys injects itself). Lets a profiler
// select an operator's kernels: ncu --nvtx --nvtx-include "fo_sparse_attention/"
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define FO_RANGE() NvtxRange fo_nvtx_range_(__func__)

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FO_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return FO_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 row-major [rows, cols] map with a box of box_cols x box_rows
int make_map_ex(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                uint32_t box_rows, CUtensorMapSwizzle swz, const char* name) {
  auto fn = encode_fn();
  if (!fn) return fail(FO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(FO_ERR_PARAM, "%s: base address not 16-byte aligned", name);
  if ((cols * 2) % 16 != 0) return fail(FO_ERR_SHAPE, "%s: row pitch not a multiple of 16 B", name);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FO_ERR_CUDA, "%s: cuTensorMapEncodeTiled failed (%d)", name, (int)r);
  return FO_OK;
}

// 3-D bf16 [slabs, rows, cols] map (box box_cols x box_rows x 1): stacked
// per-order tensors whose row coordinate is clipped / zero-filled per slab
int make_map3(CUtensorMap* m, const void* base, uint64_t slabs, uint64_t rows, uint64_t cols,
              uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz, const char* name) {
  auto fn = encode_fn();
  if (!fn) return fail(FO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(FO_ERR_PARAM, "%s: base address not 16-byte aligned", name);
  if ((cols * 2) % 16 != 0) return fail(FO_ERR_SHAPE, "%s: row pitch not a multiple of 16 B", name);
  cuuint64_t dims[3] = {cols, rows, slabs};
  cuuint64_t strides[2] = {cols * 2, rows * cols * 2};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FO_ERR_CUDA, "%s: cuTensorMapEncodeTiled failed (%d)", name, (int)r);
  return FO_OK;
}

// box = 64 columns (128 B) x box_rows, SW128: the MMA operand tiles
// outputs written by row-per-thread 256-bit stores (attention O, GEMM-Q,
// GEMM-O update out / bias) must start on a 32-byte boundary
static int check_align32(const void* ptr, const char* name) {
  if (ptr && (reinterpret_cast<uintptr_t>(ptr) & 31) != 0)
    return fail(FO_ERR_PARAM, "%s: base address not 32-byte aligned", name);
  return FO_OK;
}

int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
             const char* name) {
  return make_map_ex(m, base, rows, cols, 64, box_rows, CU_TENSOR_MAP_SWIZZLE_128B, name);
}

// Attention kernel: the column-split softmax kernel (fo_attention_cs.cu) by
// default; FO_ATTN_IMPL=v1 selects the single-warpgroup one (read once per
// process; both meet the same parity tests)
int attention_impl() {
  static int impl = -1;
  if (impl < 0) {
    const char* e = getenv("FO_ATTN_IMPL");
    impl = (e && strcmp(e, "v1") == 0) ? 0 : 1;
  }
  return impl;
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

PlanView plan_view(const void* ws, int H, int rows) {
  PlanView pv;
  plan_layout(H, rows, reinterpret_cast<char*>(const_cast<void*>(ws)), &pv);
  return pv;
}

int check_symbol_dims(int heads, int rows, int cols, int pool_n) {
  if (heads < 1 || heads > 64) return fail(FO_ERR_PARAM, "heads must be in [1, 64], got %d", heads);
  if (rows < 1 || cols < 1) return fail(FO_ERR_SHAPE, "symbol grid %dx%d is empty", rows, cols);
  if (rows >= (1 << 20)) return fail(FO_ERR_PARAM, "too many query blocks (%d)", rows);
  if (pool_n < 1) return fail(FO_ERR_CONSISTENCY, "pool_n must be >= 1, got %d", pool_n);
  return FO_OK;
}

int check_head_dim(int head_dim) {
  if (head_dim != kTile)
    return fail(FO_ERR_PARAM, "B200 kernels are built for head_dim = %d, got %d", kTile, head_dim);
  return FO_OK;
}
}  // namespace

#ifdef FO_ATTN_TIMING
static long long* fo_dbg_ptr = nullptr;
extern "C" __attribute__((visibility("default"))) int fo_debug_timing(long long* host) {
  if (!fo_dbg_ptr) return 1;
  cudaMemcpy(host, fo_dbg_ptr, 148 * 32 * sizeof(long long), cudaMemcpyDeviceToHost);
  return 0;
}
#endif

extern "C" {

long long fo_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int fo_abi_version(void) { return 1; }
const char* fo_last_error(void) { return g_err; }
int fo_num_sms(void) { return num_sms(); }

size_t fo_plan_workspace_bytes(int heads, int rows) { return plan_layout(heads, rows, nullptr, nullptr); }

size_t fo_plan_schedule_offset(int heads, int rows) {
  PlanView pv;
  plan_layout(heads, rows, nullptr, &pv);
  return reinterpret_cast<size_t>(pv.att_sched);
}

void fo_plan_offsets(int heads, int rows, size_t offsets[7]) {
  PlanView pv;
  plan_layout(heads, rows, nullptr, &pv);
  offsets[0] = reinterpret_cast<size_t>(pv.counts);
  offsets[1] = reinterpret_cast<size_t>(pv.items);
  offsets[2] = reinterpret_cast<size_t>(pv.gq_items);
  offsets[3] = reinterpret_cast<size_t>(pv.hmask);
  offsets[4] = reinterpret_cast<size_t>(pv.orders);
  offsets[5] = reinterpret_cast<size_t>(pv.pairs_pred);
  offsets[6] = reinterpret_cast<size_t>(pv.gq_jobs);
}

int fo_encode_symbols(const uint8_t* cache_bits, const uint8_t* skip_bits, int heads, int rows,
                      int cols, int pool_n, uint8_t* s_c, uint8_t* s_s, uint32_t* status,
                      void* stream) {
  FO_RANGE();
  int rc = check_symbol_dims(heads, rows, cols, pool_n);
  if (rc) return rc;
  const int comp_rows = ceil_div_d(rows, pool_n);
  const long long warps = (long long)heads * (comp_rows + 1);
  const int threads = 256;
  const long long blocks = (warps * 32 + threads - 1) / threads;
  note_launch();
  encode_symbols_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      cache_bits, skip_bits, heads, rows, cols, pool_n, s_c, s_s, status);
  return check_launch("encode_symbols");
}

int fo_decode_symbols(const uint8_t* s_c, const uint8_t* s_s, int heads, int rows, int cols,
                      int pool_n, uint8_t* active, uint8_t* pair_bits, void* stream) {
  FO_RANGE();
  int rc = check_symbol_dims(heads, rows, cols, pool_n);
  if (rc) return rc;
  const long long total = (long long)heads * rows * cols;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
  note_launch();
  decode_symbols_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(s_c, s_s, heads, rows, cols,
                                                                  pool_n, active, pair_bits);
  return check_launch("decode_symbols");
}

int fo_plan(const uint8_t* s_c, const uint8_t* s_s, int heads, int rows, int cols, int pool_n,
            int dense, const int32_t* valid, int order_d, void* plan_ws, uint32_t* status,
            void* stream) {
  FO_RANGE();
  int rc = check_symbol_dims(heads, rows, cols, pool_n);
  if (rc) return rc;
  if (!plan_ws) return fail(FO_ERR_PARAM, "plan workspace is NULL");
  PlanView pv = plan_view(plan_ws, heads, rows);
  // hist [nseg][cols+2] + scan [1024] + bin_of_rank [1024] + wave_len [1024]
  const bool head_major = (size_t)(heads * (cols + 2) + 3072) * sizeof(int) <= 160 * 1024;
  const size_t smem = (size_t)((head_major ? heads : 1) * (cols + 2) + 3072) * sizeof(int);
  if (smem > 200 * 1024) return fail(FO_ERR_PARAM, "too many key blocks (%d)", cols);
  if (num_sms() > 256) return fail(FO_ERR_CUDA, "the balanced schedule supports up to 256 SMs");
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  if (rows > 65535) return fail(FO_ERR_PARAM, "too many query blocks for the plan (%d)", rows);
  note_launch();
  // CTA-pair attention for even pool_n (sparse): the schedule has one slot per cluster
  // (the v1 kernel, FO_ATTN_IMPL=v1, runs one block per item)
  const bool pair = attention_impl() == 1 && attention_pairs(pool_n, dense);
  const int slots = pair ? num_sms() / 2 : num_sms();
  plan_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(s_c, s_s, heads, rows, cols, pool_n, dense,
                                                       valid, order_d, slots, pair ? 1 : 0, pv,
                                                       status);
  return check_launch("plan");
}

static int attention_common(const void* q, const void* k, const void* v, int seq, int heads,
                            int head_dim, const uint8_t* s_s, int rows, int cols, int pool_n,
                            const void* plan_ws, float scale, int update_mode, void* out,
                            void* cache, int32_t* valid, int order_d, int64_t* pairs,
                            uint32_t* status, const void* fc_cache, const int32_t* fc_valid,
                            const float* fc_coef, void* stream) {
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  rc = check_symbol_dims(heads, rows, cols, pool_n);
  if (rc) return rc;
  if ((rc = check_align32(out, "out"))) return rc;
  if (seq < 1) return fail(FO_ERR_SHAPE, "empty sequence");
  const int t = ceil_div_d(seq, kTile);
  if (rows != t || cols != t)
    return fail(FO_ERR_SHAPE, "symbols dimensioned %dx%d, expected %dx%d", rows, cols, t, t);
  if (order_d < 0 || order_d > 3) return fail(FO_ERR_PARAM, "order_d must be in [0, 3], got %d", order_d);
  if (!plan_ws) return fail(FO_ERR_PARAM, "plan workspace is NULL");
  if (cols > 2048) return fail(FO_ERR_PARAM, "at most 2048 key blocks (262,144 tokens), got %d", cols);
  CUtensorMap qm, km, vm;
  const uint64_t HD = (uint64_t)heads * kTile;
  if ((rc = make_map(&qm, q, seq, HD, kTile, "q"))) return rc;
  if ((rc = make_map(&km, k, seq, HD, kTile, "k"))) return rc;
  if ((rc = make_map(&vm, v, seq, HD, kTile, "v"))) return rc;
  PlanView pv = plan_view(plan_ws, heads, rows);
  AttnParams p;
  p.S = seq;
  p.H = heads;
  p.t_q = rows;
  p.t_kv = cols;
  p.pool_n = pool_n;
  p.comp_rows = ceil_div_d(rows, pool_n);
  p.row_stride = ceil_div_d(ceil_div_d(cols, pool_n), 8);
  p.dense = update_mode ? 1 : 0;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.s_s = s_s;
  p.items = pv.items;
  p.n_items = pv.counts;
  p.sched = pv.att_sched;
  p.n_waves = pv.counts + 6;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.cache = update_mode ? static_cast<__nv_bfloat16*>(cache) : nullptr;
  p.valid = update_mode ? valid : nullptr;
  p.order_d = order_d;
  p.pairs = reinterpret_cast<long long*>(pairs);
  p.status = status;
  p.dbg = nullptr;
  p.fc_cache = static_cast<const __nv_bfloat16*>(fc_cache);
  p.fc_valid = fc_valid;
  p.fc_counts = pv.counts;
  p.fc_tiles = pv.gq_items;
  for (int d = 0; d < 4; ++d) p.fc_coef[d] = (fc_coef && d <= order_d) ? fc_coef[d] : 0.f;
#ifdef FO_ATTN_TIMING
  static long long* g_dbg = nullptr;
  if (!g_dbg) {
    cudaMalloc(&g_dbg, 148 * 32 * sizeof(long long));
    cudaMemset(g_dbg, 0, 148 * 32 * sizeof(long long));
  }
  p.dbg = g_dbg;
  fo_dbg_ptr = g_dbg;
#endif
  if (!update_mode && !s_s) return fail(FO_ERR_PARAM, "s_s is NULL");
  if (attention_impl() == 1) {
    // O leaves through 32 x 32 SW64 TMA boxes (one per softmax warp and chunk)
    CUtensorMap om;
    if ((rc = make_map_ex(&om, out, seq, HD, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "out"))) return rc;
    // pooled symbols (pool_n even, sparse): CTA pairs with K/V multicast; the
    // plan was built with the matching pair items (fo_plan)
    const bool pair = attention_pairs(pool_n, update_mode);
    launch_attention_cs(qm, km, vm, om, p, num_sms(), pair, (cudaStream_t)stream);
  }
  else
    launch_attention(qm, km, vm, p, num_sms(), (cudaStream_t)stream);
  return check_launch("sparse_attention");
}

int fo_sparse_attention(const void* q, const void* k, const void* v, int seq, int heads,
                        int head_dim, const uint8_t* s_s, int rows, int cols, int pool_n,
                        const void* plan_ws, float scale, int update_mode, void* out, void* cache,
                        int32_t* valid, int order_d, int64_t* pairs, uint32_t* status,
                        void* stream) {
  FO_RANGE();
  return attention_common(q, k, v, seq, heads, head_dim, s_s, rows, cols, pool_n, plan_ws, scale,
                          update_mode, out, cache, valid, order_d, pairs, status, nullptr, nullptr,
                          nullptr, stream);
}

int fo_sparse_attention_reuse(const void* q, const void* k, const void* v, int seq, int heads,
                              int head_dim, const uint8_t* s_s, int rows, int cols, int pool_n,
                              const void* plan_ws, float scale, const void* cache,
                              const int32_t* valid, int order_d, const float* coef, void* out,
                              int64_t* pairs, uint32_t* status, void* stream) {
  FO_RANGE();
  if (!cache || !valid || !coef)
    return fail(FO_ERR_STATE, "materialize mode needs the feature cache, its valid orders and coef");
  return attention_common(q, k, v, seq, heads, head_dim, s_s, rows, cols, pool_n, plan_ws, scale,
                          0, out, nullptr, nullptr, order_d, pairs, status, cache, valid, coef,
                          stream);
}

int fo_forecast_materialize(const void* cache, int seq, int heads, int head_dim, int rows,
                            int order_d, const void* plan_ws, const int32_t* valid,
                            const float* coef, void* out, void* stream) {
  FO_RANGE();
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  if (rows != ceil_div_d(seq, kTile)) return fail(FO_ERR_SHAPE, "rows != ceil(seq/128)");
  if (order_d < 0 || order_d > 3) return fail(FO_ERR_PARAM, "order_d must be in [0, 3]");
  if (!cache || !valid || !coef || !plan_ws || !out)
    return fail(FO_ERR_PARAM, "forecast_materialize: NULL operand");
  float c[4] = {0, 0, 0, 0};
  for (int d = 0; d <= order_d; ++d) c[d] = coef[d];
  PlanView pv = plan_view(plan_ws, heads, rows);
  launch_forecast_materialize(static_cast<const __nv_bfloat16*>(cache), seq, heads, rows, order_d,
                              pv.hmask, valid, c, static_cast<__nv_bfloat16*>(out),
                              (cudaStream_t)stream);
  return check_launch("forecast_materialize");
}

int fo_check_finite(const void* data, long long rows, int cols, const void* plan_ws, int heads,
                    uint32_t* status, void* stream) {
  FO_RANGE();
  if (!data || !status) return fail(FO_ERR_PARAM, "check_finite: NULL operand");
  if (cols % 8 != 0) return fail(FO_ERR_SHAPE, "check_finite: %d columns, need a multiple of 8", cols);
  if ((reinterpret_cast<uintptr_t>(data) & 15) != 0)
    return fail(FO_ERR_PARAM, "check_finite: base address not 16-byte aligned");
  const unsigned long long* hmask = nullptr;
  if (plan_ws) {
    if (cols != heads * kTile) return fail(FO_ERR_SHAPE, "check_finite: masked check needs H*128 columns");
    hmask = plan_view(plan_ws, heads, ceil_div_d((int)rows, kTile)).hmask;
  }
  launch_check_finite(data, rows, cols, hmask, status, (cudaStream_t)stream);
  return check_launch("check_finite");
}

int fo_synthetic_x(const float* x0, const float* a, const float* b, size_t n, int kind, float c1,
                   float c2, float s, void* out, void* stream) {
  FO_RANGE();
  if (!x0 || !a || !b || !out) return fail(FO_ERR_PARAM, "synthetic_x: NULL operand");
  if (kind < 0 || kind > 2) return fail(FO_ERR_PARAM, "synthetic_x: unknown workload kind %d", kind);
  launch_synthetic_x(x0, a, b, n, kind, c1, c2, s, static_cast<__nv_bfloat16*>(out),
                     (cudaStream_t)stream);
  return check_launch("synthetic_x");
}

int fo_cache_push(const void* o, void* cache, int32_t* valid, int seq, int heads, int head_dim,
                  int rows, int order_d, const uint8_t* select, void* stream) {
  FO_RANGE();
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  if (rows != ceil_div_d(seq, kTile)) return fail(FO_ERR_SHAPE, "rows != ceil(seq/128)");
  if (order_d < 0 || order_d > 3) return fail(FO_ERR_PARAM, "order_d must be in [0, 3]");
  launch_cache_push(static_cast<const __nv_bfloat16*>(o), static_cast<__nv_bfloat16*>(cache), valid,
                    seq, heads, rows, order_d, select, -1, (cudaStream_t)stream);
  return check_launch("cache_push");
}

int fo_cache_push_tile(const void* tile, void* cache, int32_t* valid, int seq, int heads,
                       int head_dim, int rows, int order_d, int head, int block, void* stream) {
  FO_RANGE();
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  if (!tile || !cache || !valid) return fail(FO_ERR_PARAM, "cache_push_tile: null pointer");
  if (rows != ceil_div_d(seq, kTile)) return fail(FO_ERR_SHAPE, "rows != ceil(seq/128)");
  if (order_d < 0 || order_d > 3) return fail(FO_ERR_PARAM, "order_d must be in [0, 3]");
  if (head < 0 || head >= heads || block < 0 || block >= rows)
    return fail(FO_ERR_BOUNDS, "cache_push_tile: entry (%d, %d) outside (%d, %d)", head, block,
                heads, rows);
  if (reinterpret_cast<uintptr_t>(tile) & 15) return fail(FO_ERR_PARAM, "cache_push_tile: tile misaligned");
  launch_cache_push(static_cast<const __nv_bfloat16*>(tile), static_cast<__nv_bfloat16*>(cache),
                    valid, seq, heads, rows, order_d, nullptr, head * rows + block,
                    (cudaStream_t)stream);
  return check_launch("cache_push_tile");
}

int fo_gemm_q(const void* x, int seq, int d_model, const void* w_qt, int heads, int head_dim,
              const float* norm_w, const float* rope_cos, const float* rope_sin, float eps,
              const void* plan_ws, int dense, void* q_out, void* stream) {
  FO_RANGE();
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  if (d_model % 64 != 0 || d_model < 64) return fail(FO_ERR_SHAPE, "d_model must be a multiple of 64");
  if ((rc = check_align32(q_out, "q_out"))) return rc;
  if (heads < 1 || heads > 64) return fail(FO_ERR_PARAM, "heads must be in [1, 64]");
  if (!dense && !plan_ws) return fail(FO_ERR_PARAM, "plan workspace is NULL");
  CUtensorMap xm, wm, wm64;
  if ((rc = make_map(&xm, x, seq, d_model, 128, "x"))) return rc;
  if ((rc = make_map(&wm, w_qt, (uint64_t)heads * kTile, d_model, 128, "w_q"))) return rc;
  if ((rc = make_map(&wm64, w_qt, (uint64_t)heads * kTile, d_model, 64, "w_q"))) return rc;
  const int t_q = ceil_div_d(seq, kTile);
  GemmQParams p;
  p.S = seq;
  p.dm = d_model;
  p.H = heads;
  p.t_q = t_q;
  p.dense = dense;
  if (!dense) {
    PlanView pv = plan_view(plan_ws, heads, t_q);
    p.jobs = pv.gq_jobs;
    p.n_jobs = pv.counts + 7;
  } else {
    p.jobs = nullptr;
    p.n_jobs = nullptr;
  }
  p.norm_w = norm_w;
  p.rope_cos = rope_cos;
  p.rope_sin = rope_sin;
  p.eps = eps;
  p.q = static_cast<__nv_bfloat16*>(q_out);
  p.qkv = 0;
  p.k_out = p.v_out = nullptr;
  p.k_norm = nullptr;
  // one persistent launch on CTA pairs for both phases (fo_gemm.cu gemm_q2_kernel)
  launch_gemm_q2(xm, wm, wm64, p, (cudaStream_t)stream);
  return check_launch("gemm_q");
}

int fo_gemm_qkv(const void* x, int seq, int d_model, const void* w_qkvt, int heads, int head_dim,
                const float* q_norm, const float* k_norm, const float* rope_cos,
                const float* rope_sin, float eps, const void* plan_ws, int dense, void* q_out,
                void* k_out, void* v_out, void* stream) {
  FO_RANGE();
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  if (d_model % 64 != 0 || d_model < 64) return fail(FO_ERR_SHAPE, "d_model must be a multiple of 64");
  if ((rc = check_align32(q_out, "q_out")) || (rc = check_align32(k_out, "k_out")) ||
      (rc = check_align32(v_out, "v_out")))
    return rc;
  if (!x || !w_qkvt || !q_out || !k_out || !v_out)
    return fail(FO_ERR_PARAM, "gemm_qkv: null pointer");
  // Q's and K's norm weights share the 64-head shared-memory table
  if (heads < 1 || heads > 32) return fail(FO_ERR_PARAM, "gemm_qkv: heads must be in [1, 32]");
  if (!dense && !plan_ws) return fail(FO_ERR_PARAM, "plan workspace is NULL");
  CUtensorMap xm, wm, wm64;
  const uint64_t rows_w = 3 * (uint64_t)heads * kTile;
  if ((rc = make_map(&xm, x, seq, d_model, 128, "x"))) return rc;
  if ((rc = make_map(&wm, w_qkvt, rows_w, d_model, 128, "w_qkv"))) return rc;
  if ((rc = make_map(&wm64, w_qkvt, rows_w, d_model, 64, "w_qkv"))) return rc;
  const int t_q = ceil_div_d(seq, kTile);
  GemmQParams p;
  p.S = seq;
  p.dm = d_model;
  p.H = heads;
  p.t_q = t_q;
  p.dense = dense;
  if (!dense) {
    PlanView pv = plan_view(plan_ws, heads, t_q);
    p.jobs = pv.gq_jobs;
    p.n_jobs = pv.counts + 7;
  } else {
    p.jobs = nullptr;
    p.n_jobs = nullptr;
  }
  p.norm_w = q_norm;
  p.rope_cos = rope_cos;
  p.rope_sin = rope_sin;
  p.eps = eps;
  p.q = static_cast<__nv_bfloat16*>(q_out);
  p.qkv = 1;
  p.k_out = static_cast<__nv_bfloat16*>(k_out);
  p.v_out = static_cast<__nv_bfloat16*>(v_out);
  p.k_norm = k_norm;
  launch_gemm_q2(xm, wm, wm64, p, (cudaStream_t)stream);
  return check_launch("gemm_qkv");
}

static int gemm_o_common(const void* o, const void* cache, const void* w_outt, int seq, int heads,
                         int head_dim, int d_model, int order_d, const void* plan_ws,
                         GemmOParams& p, CUtensorMap& am, CUtensorMap& cm, CUtensorMap& wm) {
  int rc = check_head_dim(head_dim);
  if (rc) return rc;
  if (d_model % 128 != 0) return fail(FO_ERR_SHAPE, "d_model must be a multiple of 128");
  if (heads < 1 || heads > 64) return fail(FO_ERR_PARAM, "heads must be in [1, 64]");
  if (order_d < 0 || order_d > 3) return fail(FO_ERR_PARAM, "order_d must be in [0, 3]");
  if (!plan_ws) return fail(FO_ERR_PARAM, "plan workspace is NULL");
  const uint64_t HD = (uint64_t)heads * kTile;
  if ((rc = make_map(&am, o, seq, HD, 128, "o"))) return rc;
  if ((rc = make_map(&cm, cache ? cache : o, cache ? (uint64_t)(order_d + 1) * seq : seq, HD, 128,
                     "cache")))
    return rc;
  if ((rc = make_map(&wm, w_outt, d_model, HD, 128, "w_out"))) return rc;
  const int t_q = ceil_div_d(seq, kTile);
  PlanView pv = plan_view(plan_ws, heads, t_q);
  p.S = seq;
  p.dm = d_model;
  p.H = heads;
  p.t_q = t_q;
  p.order_d = order_d;
  p.i_begin = 0;
  p.i_end = t_q;
  p.hmask = pv.hmask;
  p.orders = pv.orders;
  for (int d = 0; d < 4; ++d) p.coef[d] = 0.f;
  p.status = nullptr;
  return FO_OK;
}

int fo_gemm_o_update(const void* o, const void* cache, const void* w_outt, int seq, int heads,
                     int head_dim, int d_model, int order_d, const void* plan_ws, void* out,
                     void* bias, uint32_t* status, void* stream) {
  FO_RANGE();
  GemmOParams p;
  CUtensorMap am, cm, wm;
  int rc = gemm_o_common(o, cache, w_outt, seq, heads, head_dim, d_model, order_d, plan_ws, p, am,
                         cm, wm);
  if (rc) return rc;
  if (!cache) return fail(FO_ERR_STATE, "update projection needs the refreshed feature cache");
  if (!out || !bias) return fail(FO_ERR_PARAM, "gemm_o_update: out / bias is NULL");
  p.update = 1;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.bias = static_cast<__nv_bfloat16*>(bias);
  p.status = status;
  // A tiles move in halves (64 rows), each multicast to both CTAs of a cluster;
  // the cache stacks and the bias are [order+1][S][cols] 3-D maps (a ragged
  // last block stays inside its order's slab)
  const uint64_t HD = (uint64_t)heads * kTile;
  CUtensorMap om, bm;
  if ((rc = make_map(&am, o, seq, HD, 64, "o"))) return rc;
  if ((rc = make_map3(&cm, cache, order_d + 1, seq, HD, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B,
                      "cache")))
    return rc;
  if ((rc = make_map_ex(&om, out, seq, d_model, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "out"))) return rc;
  if ((rc = make_map3(&bm, bias, order_d + 1, seq, d_model, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B,
                      "bias")))
    return rc;
  launch_gemm_o_update(am, cm, wm, om, bm, p, (cudaStream_t)stream);
  return check_launch("gemm_o_update");
}

int fo_gemm_o_dispatch(const void* o, const void* w_outt, const void* bias, const int32_t* orders,
                       int seq, int heads, int head_dim, int d_model, int order_d,
                       const float* coef, const void* plan_ws, void* out, void* stream) {
  return fo_gemm_o_dispatch_rows(o, w_outt, bias, orders, seq, heads, head_dim, d_model, order_d,
                                 coef, plan_ws, 0, ceil_div_d(seq, kTile), 0, out, stream);
}

int fo_gemm_o_dispatch_rows(const void* o, const void* w_outt, const void* bias,
                            const int32_t* orders, int seq, int heads, int head_dim, int d_model,
                            int order_d, const float* coef, const void* plan_ws, int block_begin,
                            int block_end, int max_sms, void* out, void* stream) {
  FO_RANGE();
  GemmOParams p;
  CUtensorMap am, cm, wm;
  int rc = gemm_o_common(o, nullptr, w_outt, seq, heads, head_dim, d_model, order_d, plan_ws, p,
                         am, cm, wm);
  if (rc) return rc;
  if (!orders || !bias) return fail(FO_ERR_STATE, "dispatch projection requires the update-step bias");
  if (!coef) return fail(FO_ERR_PARAM, "gemm_o_dispatch: coef is NULL");
  if (!out) return fail(FO_ERR_PARAM, "gemm_o_dispatch: out is NULL");
  if (block_begin < 0 || block_end > p.t_q || block_begin > block_end)
    return fail(FO_ERR_BOUNDS, "gemm_o_dispatch: block range [%d, %d) outside [0, %d)", block_begin,
                block_end, p.t_q);
  if (max_sms < 0 || max_sms == 1) return fail(FO_ERR_PARAM, "gemm_o_dispatch: max_sms=%d", max_sms);
  if (block_begin == block_end) return FO_OK;
  p.update = 0;
  p.i_begin = block_begin;
  p.i_end = block_end;
  p.orders = orders;
  for (int d = 0; d <= order_d; ++d) p.coef[d] = coef[d];
  p.out = static_cast<__nv_bfloat16*>(out);
  p.bias = static_cast<__nv_bfloat16*>(const_cast<void*>(bias));
  // epilogue chunks: 128 rows x 32 columns (64 B rows, SW64) of bias and out
  CUtensorMap bm, om;
  if ((rc = make_map_ex(&bm, bias, (uint64_t)(order_d + 1) * seq, d_model, 32, 128,
                        CU_TENSOR_MAP_SWIZZLE_64B, "bias")))
    return rc;
  // output: one 32-row x 32-column box per epilogue warp and chunk
  if ((rc = make_map_ex(&om, out, seq, d_model, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "out")))
    return rc;
  // o moves in half tiles (64 rows), each multicast to both CTAs of a cluster
  if ((rc = make_map(&am, o, seq, (uint64_t)heads * kTile, 64, "o"))) return rc;
  launch_gemm_o(am, bm, wm, om, p, max_sms > 0 ? max_sms : (1 << 30), (cudaStream_t)stream);
  return check_launch("gemm_o_dispatch");
}

int fo_check_active_match(const uint8_t* s_c_a, const uint8_t* s_c_b, int heads, int rows,
                          int pool_n, uint32_t* status, void* stream) {
  FO_RANGE();
  int rc = check_symbol_dims(heads, rows, 1, pool_n);
  if (rc) return rc;
  const int total = heads * rows;
  note_launch();
  compare_active_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(s_c_a, s_c_b, heads,
                                                                              rows, pool_n, status);
  return check_launch("check_active_match");
}

size_t fo_policy_workspace_bytes(int seq, int heads, int pool_n) {
  if (seq <= 0 || heads <= 0 || pool_n <= 0) return 0;
  const int rows_c = (seq + pool_n * kTile - 1) / (pool_n * kTile);
  return policy_workspace_bytes(heads, rows_c);
}

int fo_generate_masks(const void* q, const void* k, int seq, int heads, int n_text, int pool_n,
                      double tau_q, double tau_kv, double s_q, int guard, uint8_t* cache_bits,
                      uint8_t* skip_bits, void* workspace, size_t workspace_bytes, void* stream) {
  FO_RANGE();
  if (!q || !k || !cache_bits || !skip_bits || !workspace)
    return fail(FO_ERR_PARAM, "generate_masks: null pointer");
  if (seq <= 0 || heads <= 0) return fail(FO_ERR_SHAPE, "generate_masks: seq=%d heads=%d", seq, heads);
  if (pool_n <= 0) return fail(FO_ERR_PARAM, "pool_n must be >= 1, got %d", pool_n);
  if (n_text < 0 || n_text > seq)
    return fail(FO_ERR_PARAM, "n_text=%d outside [0, %d]", n_text, seq);
  // policy.py:101-102, 136-137, 168-169 (NaN fails these too)
  if (!(tau_q >= 0.0 && tau_q <= 1.0)) return fail(FO_ERR_PARAM, "tau_q must be in [0, 1], got %g", tau_q);
  if (!(tau_kv >= 0.0 && tau_kv <= 1.0))
    return fail(FO_ERR_PARAM, "tau_kv must be in [0, 1], got %g", tau_kv);
  if (!(s_q >= 0.0 && s_q <= 1.0)) return fail(FO_ERR_PARAM, "s_q must be in [0, 1], got %g", s_q);
  const int block = pool_n * kTile;
  const int rows_c = (seq + block - 1) / block;
  const int n_t = (n_text + block - 1) / block;
  if (rows_c > kPolicyMaxBlocks)
    return fail(FO_ERR_SHAPE, "generate_masks: %d compressed blocks exceed %d", rows_c,
                kPolicyMaxBlocks);
  if (n_t >= rows_c)  // CompressedAttnMap.__post_init__ (policy.py:33-37)
    return fail(FO_ERR_PARAM, "n_t=%d must leave at least one vision row (map has %d rows)", n_t,
                rows_c);
  if (workspace_bytes < policy_workspace_bytes(heads, rows_c))
    return fail(FO_ERR_PARAM, "generate_masks: workspace %zu B < %zu B", workspace_bytes,
                policy_workspace_bytes(heads, rows_c));
  cudaError_t e = launch_generate_masks(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), seq, heads, n_t,
      pool_n, tau_q, tau_kv, s_q, guard, cache_bits, skip_bits, workspace, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(FO_ERR_CUDA, "generate_masks: %s", cudaGetErrorString(e));
  return FO_OK;
}

// ---- the reference's policy building blocks, one stage per call (policy.py:21-178)
size_t fo_policy_map_workspace_bytes(int seq_q, int seq_k, int heads, int pool_q, int pool_k) {
  if (seq_q <= 0 || seq_k <= 0 || heads <= 0 || pool_q <= 0 || pool_k <= 0) return 0;
  return policy_map_workspace_bytes(heads, (seq_q + pool_q - 1) / pool_q,
                                    (seq_k + pool_k - 1) / pool_k);
}

int fo_policy_compressed_map(const void* q, const void* k, int is_f32, int seq_q, int seq_k,
                             int heads, int head_dim, int pool_q, int pool_k, float* p_tilde,
                             void* workspace, size_t workspace_bytes, void* stream) {
  FO_RANGE();
  if (!q || !k || !p_tilde || !workspace) return fail(FO_ERR_PARAM, "compressed_map: null pointer");
  if (seq_q <= 0 || seq_k <= 0 || heads <= 0)
    return fail(FO_ERR_SHAPE, "compressed_map: seq=%d/%d heads=%d", seq_q, seq_k, heads);
  if (head_dim < 1 || head_dim > kTile)
    return fail(FO_ERR_SHAPE, "compressed_map: head_dim %d outside [1, %d]", head_dim, kTile);
  if (pool_q < 1 || pool_k < 1)  // mean_pool_blocks (tensor.py:119-120)
    return fail(FO_ERR_PARAM, "pool must be >= 1, got %d / %d", pool_q, pool_k);
  const int rows = (seq_q + pool_q - 1) / pool_q, cols = (seq_k + pool_k - 1) / pool_k;
  if (rows > kPolicyMaxBlocks || cols > kPolicyMaxBlocks)
    return fail(FO_ERR_SHAPE, "compressed_map: %d x %d compressed blocks exceed %d", rows, cols,
                kPolicyMaxBlocks);
  if (workspace_bytes < policy_map_workspace_bytes(heads, rows, cols))
    return fail(FO_ERR_PARAM, "compressed_map: workspace %zu B too small", workspace_bytes);
  const uintptr_t al = is_f32 ? 8 : 4;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) % al)
    return fail(FO_ERR_PARAM, "compressed_map: q/k misaligned");
  cudaError_t e = launch_policy_map(q, k, is_f32, seq_q, seq_k, heads, head_dim, pool_q, pool_k,
                                    p_tilde, workspace, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(FO_ERR_CUDA, "compressed_map: %s", cudaGetErrorString(e));
  return FO_OK;
}

int fo_policy_block_scores(const float* p_tilde, int heads, int rows, int cols, int n_t,
                           double* contribution, double* guidance, void* stream) {
  FO_RANGE();
  if (!p_tilde || !contribution || !guidance) return fail(FO_ERR_PARAM, "block_scores: null pointer");
  if (heads <= 0 || rows <= 0 || cols <= 0 || rows > kPolicyMaxBlocks || cols > kPolicyMaxBlocks)
    return fail(FO_ERR_SHAPE, "block_scores: %d x %d map", rows, cols);
  if (n_t < 0 || n_t >= rows || n_t > cols)  // CompressedAttnMap (policy.py:33-37)
    return fail(FO_ERR_PARAM, "n_t=%d must leave at least one vision row (map has %d rows)", n_t, rows);
  cudaError_t e = launch_policy_scores(p_tilde, heads, rows, cols, n_t, contribution, guidance,
                                       (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(FO_ERR_CUDA, "block_scores: %s", cudaGetErrorString(e));
  return FO_OK;
}

int fo_policy_select_cached(const double* contribution, const double* guidance, int heads, int n,
                            double tau_q, uint8_t* cached, void* stream) {
  FO_RANGE();
  if (!contribution || !guidance || !cached) return fail(FO_ERR_PARAM, "select_cached: null pointer");
  if (heads <= 0 || n < 0 || n > kPolicyMaxBlocks) return fail(FO_ERR_SHAPE, "select_cached: n=%d", n);
  if (!(tau_q >= 0.0 && tau_q <= 1.0)) return fail(FO_ERR_PARAM, "tau_q must be in [0, 1], got %g", tau_q);
  if (n == 0) return FO_OK;
  cudaError_t e = launch_policy_select_cached(contribution, guidance, heads, n, tau_q, cached,
                                              (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(FO_ERR_CUDA, "select_cached: %s", cudaGetErrorString(e));
  return FO_OK;
}

int fo_policy_select_skip(const float* p_tilde, const uint8_t* compute, int heads, int rows,
                          int cols, int n_t, double tau_kv, int guard, uint8_t* keep, void* stream) {
  FO_RANGE();
  if (!p_tilde || !compute || !keep) return fail(FO_ERR_PARAM, "select_skip: null pointer");
  if (heads <= 0 || rows <= 0 || cols <= 0 || rows > kPolicyMaxBlocks || cols > kPolicyMaxBlocks)
    return fail(FO_ERR_SHAPE, "select_skip: %d x %d map", rows, cols);
  if (n_t < 0 || n_t > cols) return fail(FO_ERR_PARAM, "select_skip: n_t=%d", n_t);
  if (!(tau_kv >= 0.0 && tau_kv <= 1.0))
    return fail(FO_ERR_PARAM, "tau_kv must be in [0, 1], got %g", tau_kv);
  cudaError_t e = launch_policy_select_skip(p_tilde, compute, heads, rows, cols, n_t, tau_kv, guard,
                                            keep, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(FO_ERR_CUDA, "select_skip: %s", cudaGetErrorString(e));
  return FO_OK;
}

// ---- tile-level building blocks and dense numerics (fo_numerics.cu)
static int cuda_rc(cudaError_t e, const char* what) {
  return e == cudaSuccess ? FO_OK : fail(FO_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int fo_online_softmax_update(const float* m, const float* l, const float* acc, const float* scores,
                             const float* v, int rows, int cols, int d, float* m_out, float* l_out,
                             float* acc_out, void* stream) {
  if (!m || !l || !acc || !scores || !v || !m_out || !l_out || !acc_out)
    return fail(FO_ERR_PARAM, "online_softmax_update: null pointer");
  if (rows < 0 || cols <= 0 || d <= 0 || cols > max_row_width())
    return fail(FO_ERR_SHAPE, "online_softmax_update: rows=%d cols=%d d=%d", rows, cols, d);
  if (rows == 0) return FO_OK;
  return cuda_rc(launch_online_softmax_update(m, l, acc, scores, v, rows, cols, d, m_out, l_out,
                                              acc_out, (cudaStream_t)stream),
                 "online_softmax_update");
}

int fo_online_softmax_finalize(const float* acc, const float* l, int rows, int d, float* out,
                               uint32_t* status, void* stream) {
  if (!acc || !l || !out || !status) return fail(FO_ERR_PARAM, "online_softmax_finalize: null pointer");
  if (rows < 0 || d <= 0) return fail(FO_ERR_SHAPE, "online_softmax_finalize: rows=%d d=%d", rows, d);
  if (rows == 0) return FO_OK;
  return cuda_rc(launch_online_softmax_finalize(acc, l, rows, d, out, status, (cudaStream_t)stream),
                 "online_softmax_finalize");
}

int fo_update_entry(const float* old_stack, int old_valid, const float* o_new, long long tile,
                    int order, float* stack, void* stream) {
  if (!o_new || !stack || (old_valid > 0 && !old_stack))
    return fail(FO_ERR_PARAM, "update_entry: null pointer");
  if (order < 0 || order > 7 || tile < 0) return fail(FO_ERR_PARAM, "update_entry: order %d", order);
  if (tile == 0) return FO_OK;
  const int valid = old_valid > 0 ? (old_valid + 1 < order + 1 ? old_valid + 1 : order + 1) : 1;
  return cuda_rc(launch_update_entry(old_stack, o_new, (size_t)tile, order, valid, stack,
                                     (cudaStream_t)stream),
                 "update_entry");
}

int fo_forecast_entry(const float* stack, long long tile, int n_orders, const float* coef,
                      float* out, void* stream) {
  if (!stack || !coef || !out) return fail(FO_ERR_PARAM, "forecast: null pointer");
  if (n_orders < 1 || n_orders > 8 || tile < 0) return fail(FO_ERR_PARAM, "forecast: n_orders %d", n_orders);
  if (tile == 0) return FO_OK;
  return cuda_rc(launch_forecast_entry(stack, (size_t)tile, n_orders, coef, out, (cudaStream_t)stream),
                 "forecast");
}

int fo_mean_pool_blocks(const float* x, int n, int d, int pool, float* out, void* stream) {
  if (!x || !out) return fail(FO_ERR_PARAM, "mean_pool_blocks: null pointer");
  if (pool < 1) return fail(FO_ERR_PARAM, "pool must be >= 1, got %d", pool);
  if (n < 0 || d <= 0) return fail(FO_ERR_SHAPE, "mean_pool_blocks: n=%d d=%d", n, d);
  if (n == 0) return FO_OK;
  return cuda_rc(launch_mean_pool(x, n, d, pool, out, (cudaStream_t)stream), "mean_pool_blocks");
}

int fo_rms_norm(const float* x, const float* weight, int n, int d, double eps, float* out,
                void* stream) {
  if (!x || !weight || !out) return fail(FO_ERR_PARAM, "rms_norm: null pointer");
  if (n < 0 || d <= 0 || d > max_row_width()) return fail(FO_ERR_SHAPE, "rms_norm: n=%d d=%d", n, d);
  if (n == 0) return FO_OK;
  return cuda_rc(launch_rms_norm(x, weight, n, d, eps, out, (cudaStream_t)stream), "rms_norm");
}

int fo_rope(const float* x, const float* cos_t, const float* sin_t, int n, int d, float* out,
            void* stream) {
  if (!x || !cos_t || !sin_t || !out) return fail(FO_ERR_PARAM, "rope: null pointer");
  if (n < 0 || d <= 0 || d % 2) return fail(FO_ERR_SHAPE, "rope: feature dim must be even, got %d", d);
  if (n == 0) return FO_OK;
  return cuda_rc(launch_rope(x, cos_t, sin_t, n, d, out, (cudaStream_t)stream), "rope");
}

int fo_row_softmax(const float* s, int n, int d, float* out, void* stream) {
  if (!s || !out) return fail(FO_ERR_PARAM, "row_softmax: null pointer");
  if (n < 0 || d <= 0 || d > max_row_width()) return fail(FO_ERR_SHAPE, "row_softmax: n=%d d=%d", n, d);
  if (n == 0) return FO_OK;
  return cuda_rc(launch_row_softmax(s, n, d, out, (cudaStream_t)stream), "row_softmax");
}

int fo_matmul_f32(const float* a, const float* b, float* c, int m, int n, int k, int accumulate,
                  void* stream) {
  FO_RANGE();
  if (!a || !b || !c) return fail(FO_ERR_PARAM, "matmul_f32: null pointer");
  if (m < 0 || n < 0 || k < 0 || m > 65535 * 64)
    return fail(FO_ERR_SHAPE, "matmul_f32: m=%d n=%d k=%d", m, n, k);
  if (m == 0 || n == 0) return FO_OK;
  return cuda_rc(launch_matmul_f32(a, b, c, m, n, k, accumulate, (cudaStream_t)stream),
                 "matmul_f32");
}

int fo_masked_block_attention_f32(const float* q, const float* k, const float* v, int n, int d,
                                  const uint8_t* active, const uint8_t* pair_bits, int b_q, int b_k,
                                  float scale, float* out, unsigned long long* pairs,
                                  uint32_t* status, void* stream) {
  FO_RANGE();
  if (!q || !k || !v || !active || !pair_bits || !out || !status)
    return fail(FO_ERR_PARAM, "masked_block_attention: null pointer");
  if (n < 0 || d < 1 || d > 256 || b_q < 1 || b_k < 1)
    return fail(FO_ERR_SHAPE, "masked_block_attention: n=%d d=%d (1..256) b_q=%d b_k=%d", n, d, b_q,
                b_k);
  if (n == 0) return FO_OK;
  return cuda_rc(launch_masked_block_attention_f32(q, k, v, n, d, active, pair_bits, b_q, b_k, scale,
                                                   out, pairs, status, (cudaStream_t)stream),
                 "masked_block_attention");
}

}  // extern "C"
