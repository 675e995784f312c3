/*
 * flashomni_b200.h — C ABI of the B200-native FlashOmni hot path.
 *
 * Everything is plain pointers, sizes and a cudaStream_t passed as void*;
 * all buffers are caller-allocated device memory and every call is
 * stream-ordered (nothing synchronises, nothing allocates). Device-detected
 * contract violations (an active query block with every key block skipped,
 * a cold cache entry, a non-uniform pool group, stale symbols) set bits in
 * a caller-owned uint32 status word in device memory; the host wrapper reads
 * it and raises the matching exception of reference errors.py:4-25.
 *
 * Layouts (bf16 unless stated):
 *   q, k, v, o        [seq, heads, 128]         token-major, = [seq, heads*128]
 *   x                 [seq, d_model]
 *   w_qt              [heads*128, d_model]      (reference w_q [heads, d_model, 128], transposed)
 *   w_outt            [d_model, heads*128]      (reference w_out [heads, 128, d_model], transposed)
 *   cache (diff stacks) [order_d+1, seq, heads*128]
 *   bias  (B_c)       [order_d+1, seq, d_model]
 *   valid             int32 [heads, rows]       valid difference orders per (head, block)
 *   s_c               uint8 [heads, ceil(ceil(rows/pool_n)/8)]
 *   s_s               uint8 [heads, ceil(rows/pool_n), ceil(ceil(cols/pool_n)/8)]
 * Blocks are b_q = b_k = 128 tokens; rows = cols = ceil(seq/128).
 * Alignment: TMA-read operands start on a 16-byte boundary; the outputs
 * written with 256-bit row stores (attention out, GEMM-Q q_out, GEMM-O
 * update out and bias) on a 32-byte boundary (FO_ERR_PARAM otherwise).
 */
#ifndef FLASHOMNI_B200_H
#define FLASHOMNI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FO_API __attribute__((visibility("default")))
#else
#define FO_API
#endif

/* return codes, one per reference exception class (errors.py:4-25) */
enum {
  FO_OK = 0,
  FO_ERR_SHAPE = 1,       /* ShapeError */
  FO_ERR_PARAM = 2,       /* ParameterError */
  FO_ERR_BOUNDS = 3,      /* BoundsError */
  FO_ERR_CONSISTENCY = 4, /* ConsistencyError */
  FO_ERR_STATE = 5,       /* StateError */
  FO_ERR_CUDA = 6         /* launch / driver failure */
};
/* device status-word bits */
#define FO_ST_CONSISTENCY 0x1u
#define FO_ST_STATE 0x2u
#define FO_ST_BOUNDS 0x4u
#define FO_ST_PARAM 0x8u
#define FO_ST_TIMEOUT 0x10u

FO_API int fo_abi_version(void);
FO_API const char* fo_last_error(void);
FO_API int fo_num_sms(void);
/* Kernels this library has launched since load (every <<<>>> / cudaLaunchKernelEx
 * site counts one): the bench's gpu_launches figure. */
FO_API long long fo_kernel_launches(void);

/* Schedule workspace for one layer's symbols (plan): byte size and the byte
 * offsets of {counts, items, gemm-q tiles, head masks, orders, pairs, gemm-q head-pair jobs}. */
FO_API size_t fo_plan_workspace_bytes(int heads, int rows);
FO_API void fo_plan_offsets(int heads, int rows, size_t offsets[7]);
/* Byte offset of the attention schedule in the plan workspace: int32
 * [n_waves, num_sms], the item each CTA runs in each wave (-1: none);
 * n_waves is counts[6]. */
FO_API size_t fo_plan_schedule_offset(int heads, int rows);

/* K1 symbol pack. Replaces encode_cache_mask / encode_skip_mask / build_symbols
 * (reference pkg/src/omniattn/symbols.py:65-81,145-160) for all heads at once.
 * cache_bits uint8 [heads, rows], skip_bits uint8 [heads, rows, cols] (nonzero = 1). */
FO_API int fo_encode_symbols(const uint8_t* cache_bits, const uint8_t* skip_bits, int heads, int rows,
                      int cols, int pool_n, uint8_t* s_c, uint8_t* s_s, uint32_t* status,
                      void* stream);

/* Device decode of every cache bit and pair bit with the same decoders the kernel
 * prologues use. Replaces decode_spatial / decode_reduction / decode_run
 * (symbols.py:163-198). active uint8 [heads, rows], pair_bits uint8 [heads, rows, cols]. */
FO_API int fo_decode_symbols(const uint8_t* s_c, const uint8_t* s_s, int heads, int rows, int cols,
                      int pool_n, uint8_t* active, uint8_t* pair_bits, void* stream);

/* Build the layer schedule from symbols: attention work items sorted by KV
 * count, GEMM-Q tile list, per-block head masks, cached-bias orders and the
 * mask-predicted pair counts. Raises CONSISTENCY for an active row with no key
 * block (pyref.py:43-46) and STATE for a cached tile with a cold cache
 * (attention.py:208-211, gemm.py:150-153) when `valid` is given.
 * dense=1 schedules every (head, block) with every key block (update step). */
FO_API int fo_plan(const uint8_t* s_c, const uint8_t* s_s, int heads, int rows, int cols, int pool_n,
            int dense, const int32_t* valid, int order_d, void* plan_ws, uint32_t* status,
            void* stream);

/* K2 / K2u sparse attention for all heads. Replaces sparse_attention(mode="bias")
 * (attention.py:150-221) and the backend entry masked_block_attention
 * (_kernels/pyref.py:14-48, _kernels/_core.pyx:14-101). Rows of cached blocks
 * are left untouched in `out`. update_mode=1 (plan built dense) also pushes
 * every tile into the diff stacks `cache` and bumps `valid`
 * (attention.py:71-85 via pipeline.py:274-278). pairs (int64 [heads], may be
 * NULL) accumulates the instrumented computed-pair count. */
FO_API int fo_sparse_attention(const void* q, const void* k, const void* v, int seq, int heads,
                        int head_dim, const uint8_t* s_s, int rows, int cols, int pool_n,
                        const void* plan_ws, float scale, int update_mode, void* out, void* cache,
                        int32_t* valid, int order_d, int64_t* pairs, uint32_t* status,
                        void* stream);

/* K2 in mode="materialize" as ONE launch (attention.py:150-221 with 212-216): the
 * computed tiles as fo_sparse_attention, and the cached tiles' OP_reuse
 * out = sum_{d < min(order_d+1, valid)} coef[d] * cache[d] fused into the same
 * persistent kernel (its softmax warps take cached tiles from a global cursor
 * once their attention items are done). cache [order_d+1, S, H*128] and valid
 * are read-only here; coef is a host array of order_d+1 floats. The plan must
 * be built with `valid` (cold-cache check). */
FO_API int fo_sparse_attention_reuse(const void* q, const void* k, const void* v, int seq, int heads,
                              int head_dim, const uint8_t* s_s, int rows, int cols, int pool_n,
                              const void* plan_ws, float scale, const void* cache,
                              const int32_t* valid, int order_d, const float* coef, void* out,
                              int64_t* pairs, uint32_t* status, void* stream);

/* OP_reuse for mode="materialize": cached tiles of `out` <- sum_d coef[d]*stack[d]
 * (attention.py:96-113,212-216). coef is a host array of order_d+1 floats. */
FO_API int fo_forecast_materialize(const void* cache, int seq, int heads, int head_dim, int rows,
                            int order_d, const void* plan_ws, const int32_t* valid,
                            const float* coef, void* out, void* stream);

/* Input validation of the reference's as_matrix (tensor.py:19-30): sets FO_ST_PARAM
 * when any bf16 of data [rows, cols] is NaN or Inf. With plan_ws (cols = heads*128)
 * only the tiles of active (block, head) pairs are checked, as sparse_attention
 * checks only the q rows it reads (attention.py:194-196). */
FO_API int fo_check_finite(const void* data, long long rows, int cols, const void* plan_ws, int heads,
                           uint32_t* status, void* stream);

/* SyntheticWorkload.x(t) of the reference run() (pipeline.py:160-171) as one pass:
 * out bf16 = bf16(f32(f64(x0) + f64(f32 terms))) with numpy's float32 products and
 * float64 sums. kind 0 drift (c1 = t, c2 = t*t/steps), 1 poly1 (c1 = s*t),
 * 2 poly2 (c1 = s*t, c2 = (s*t)^2); scalars already rounded to float32. */
FO_API int fo_synthetic_x(const float* x0, const float* a, const float* b, size_t n, int kind,
                          float c1, float c2, float s, void* out, void* stream);

/* FeatureCache.update for the selected (head, block) entries (select uint8
 * [heads, rows], NULL = all) (attention.py:71-85,128-131). */
FO_API int fo_cache_push(const void* o, void* cache, int32_t* valid, int seq, int heads, int head_dim,
                  int rows, int order_d, const uint8_t* select, void* stream);
/* FeatureCache.update of ONE entry (attention.py:128-131): tile bf16 [r, 128],
 * r = min(128, seq - 128*block), pushed into (head, block); BOUNDS outside the cache. */
FO_API int fo_cache_push_tile(const void* tile, void* cache, int32_t* valid, int seq, int heads,
                              int head_dim, int rows, int order_d, int head, int block,
                              void* stream);

/* K3 GEMM-Q: q = rope(rms_norm(x @ W_q[h])) for active (block, head) tiles only
 * (gemm.py:44-93, tensor.py:68-109). dense=1: every tile (update phase, plan
 * may be NULL). rope_cos/rope_sin fp32 [seq, 64] = cos/sin(pos * 1e4^(-2j/128)). */
FO_API int fo_gemm_q(const void* x, int seq, int d_model, const void* w_qt, int heads, int head_dim,
              const float* norm_w, const float* rope_cos, const float* rope_sin, float eps,
              const void* plan_ws, int dense, void* q_out, void* stream);

/* K5 GEMM-O update: B_c[d] = sum_{h cached next} stack_d^h W_h and
 * out = B_c[0] + sum_{h active next} o_h W_h (gemm.py:110-175): cached heads'
 * order-0 term comes from the cache's stack 0, not from o. cache is
 * [cache_order+1, seq, heads*128] (required: STATE when NULL). plan_ws is the
 * plan of the NEXT symbols built with `valid`; orders are taken from it. */
FO_API int fo_gemm_o_update(const void* o, const void* cache, const void* w_outt, int seq, int heads,
                     int head_dim, int d_model, int order_d, const void* plan_ws, void* out,
                     void* bias, uint32_t* status, void* stream);

/* K4 GEMM-O dispatch: out = sum_{h active} o_h W_h + sum_d coef[d] * B_c[d]
 * (gemm.py:178-229). orders int32 [rows] from the update step; coef host floats. */
FO_API int fo_gemm_o_dispatch(const void* o, const void* w_outt, const void* bias, const int32_t* orders,
                       int seq, int heads, int head_dim, int d_model, int order_d,
                       const float* coef, const void* plan_ws, void* out, void* stream);

/* fo_gemm_o_dispatch restricted to query blocks [block_begin, block_end) (rows
 * 128*block_begin .. of `out`; other rows untouched) on at most max_sms SMs (0 =
 * all): the row-chunked dispatch the multi-GPU step overlaps with the
 * all-reduce of the previous chunk. BOUNDS for a range outside
 * [0, rows). */
FO_API int fo_gemm_o_dispatch_rows(const void* o, const void* w_outt, const void* bias,
                                   const int32_t* orders, int seq, int heads, int head_dim,
                                   int d_model, int order_d, const float* coef, const void* plan_ws,
                                   int block_begin, int block_end, int max_sms, void* out,
                                   void* stream);

/* The dispatch step's three projections in ONE launch (pipeline.py:223-234 +
 * gemm.py:44-93): q (GEMM-Q, RMSNorm + RoPE; only the plan's active tiles, or
 * every tile with dense=1), k (dense, RMSNorm + RoPE with k_norm) and v (dense,
 * plain) from one read of x. w_qkvt: bf16 [3*heads*128, d_model] = [W_q^T;
 * W_k^T; W_v^T]. heads <= 32. */
FO_API int fo_gemm_qkv(const void* x, int seq, int d_model, const void* w_qkvt, int heads,
                       int head_dim, const float* q_norm, const float* k_norm,
                       const float* rope_cos, const float* rope_sin, float eps,
                       const void* plan_ws, int dense, void* q_out, void* k_out, void* v_out,
                       void* stream);

/* Stale-symbol check (gemm.py:201-209): STATE if the decoded cache bits differ. */
FO_API int fo_check_active_match(const uint8_t* s_c_a, const uint8_t* s_c_b, int heads, int rows,
                          int pool_n, uint32_t* status, void* stream);

/* Update-step mask policy, all heads at once (replaces policy.py:196-234
 * generate_masks, called per head from pipeline.py:260-270). q, k: bf16
 * [seq, heads, 128] (head_dim 128, b_q = b_k = 128). n_text: leading text
 * tokens. tau_q / tau_kv / s_q in [0, 1] (ramp_threshold is applied by the
 * caller, policy.py:181-187). guard != 0 protects text columns and the
 * diagonal. Outputs, True = compute: cache_bits u8 [heads, t_q], skip_bits u8
 * [heads, t_q, t_q]; feed them to fo_encode_symbols. Decisions match the
 * reference's float32 / float64 numpy bit for bit (see fo_policy.cu).
 * Errors: PARAM for thresholds outside [0, 1] or a text prefix that leaves no
 * vision row (policy.py:33-37), SHAPE for more than 1024 compressed blocks
 * per side. */
FO_API size_t fo_policy_workspace_bytes(int seq, int heads, int pool_n);
FO_API int fo_generate_masks(const void* q, const void* k, int seq, int heads, int n_text,
                             int pool_n, double tau_q, double tau_kv, double s_q, int guard,
                             uint8_t* cache_bits, uint8_t* skip_bits, void* workspace,
                             size_t workspace_bytes, void* stream);

/* ---- The reference's policy building blocks, one stage per call ----------
 * (policy.py:21-178; fo_generate_masks runs all of them fused.) q, k:
 * [seq, heads, 128] bf16 (is_f32 = 0) or float32 (is_f32 = 1); a head
 * dimension head_dim < 128 is zero-padded by the caller (the scores divide by
 * sqrt(head_dim)). */
/* compressed_attention (policy.py:44-55): mean-pool q by pool_q and k by
 * pool_k tokens (tensor.py:112-126), scores / sqrt(d) in float64, row softmax
 * -> p_tilde float32 [heads, ceil(seq_q/pool_q), ceil(seq_k/pool_k)]. */
FO_API size_t fo_policy_map_workspace_bytes(int seq_q, int seq_k, int heads, int pool_q,
                                            int pool_k);
FO_API int fo_policy_compressed_map(const void* q, const void* k, int is_f32, int seq_q, int seq_k,
                                    int heads, int head_dim, int pool_q, int pool_k,
                                    float* p_tilde, void* workspace, size_t workspace_bytes,
                                    void* stream);
/* vision_to_text_contribution / text_to_vision_guidance (policy.py:58-77):
 * float64 contribution [heads, cols - n_t], guidance [heads, rows - n_t]. */
FO_API int fo_policy_block_scores(const float* p_tilde, int heads, int rows, int cols, int n_t,
                                  double* contribution, double* guidance, void* stream);
/* select_cached_blocks (policy.py:93-111): cached u8 [heads, n], 1 = cached. */
FO_API int fo_policy_select_cached(const double* contribution, const double* guidance, int heads,
                                   int n, double tau_q, uint8_t* cached, void* stream);
/* select_skip_blocks (policy.py:124-159): compute u8 [heads, rows] (1 = row
 * computed) -> keep u8 [heads, rows, cols], 1 = compute the pair. */
FO_API int fo_policy_select_skip(const float* p_tilde, const uint8_t* compute, int heads, int rows,
                                 int cols, int n_t, double tau_kv, int guard, uint8_t* keep,
                                 void* stream);

/* ---- Tile-level building blocks and dense numerics (float32 device buffers) */
/* online_softmax_update (attention.py:39-49) over one score block: m, l [rows],
 * acc [rows, d], scores [rows, cols], v [cols, d] -> m_out, l_out, acc_out. */
FO_API int fo_online_softmax_update(const float* m, const float* l, const float* acc,
                                    const float* scores, const float* v, int rows, int cols, int d,
                                    float* m_out, float* l_out, float* acc_out, void* stream);
/* online_softmax_finalize (attention.py:52-55): out = acc / l; a row with
 * l <= 0 sets FO_ST_CONSISTENCY. */
FO_API int fo_online_softmax_finalize(const float* acc, const float* l, int rows, int d, float* out,
                                      uint32_t* status, void* stream);
/* update_entry (attention.py:71-85) for one tile of `tile` floats: old_stack
 * [order+1, tile] with old_valid levels (0 / NULL: no entry) -> stack
 * [order+1, tile]; valid orders become min(old_valid + 1, order + 1). */
FO_API int fo_update_entry(const float* old_stack, int old_valid, const float* o_new,
                           long long tile, int order, float* stack, void* stream);
/* forecast (attention.py:96-113): out = sum_{d < n_orders} coef[d] * stack[d];
 * coef is a host array. */
FO_API int fo_forecast_entry(const float* stack, long long tile, int n_orders, const float* coef,
                             float* out, void* stream);
/* tensor.py numerics: mean_pool_blocks (112-126), rms_norm (68-80), rope (83-109;
 * cos/sin tables float32 [n, d/2]), row_softmax (42-47). x [n, d]. */
FO_API int fo_mean_pool_blocks(const float* x, int n, int d, int pool, float* out, void* stream);
FO_API int fo_rms_norm(const float* x, const float* weight, int n, int d, double eps, float* out,
                       void* stream);
FO_API int fo_rope(const float* x, const float* cos_t, const float* sin_t, int n, int d, float* out,
                   void* stream);
FO_API int fo_row_softmax(const float* s, int n, int d, float* out, void* stream);

/* C [m, n] (+)= A [m, k] B [k, n], float32 row-major (accumulate != 0: C += AB,
 * one rounding of the product then of the sum, like numpy's `c += a @ b`). The
 * product of the reference-signature GEMM paths at shapes the tcgen05 kernels
 * do not tile (gemm.py:44-229 with numpy float32 matmul). */
FO_API int fo_matmul_f32(const float* a, const float* b, float* c, int m, int n, int k,
                         int accumulate, void* stream);

/* The reference tile-kernel protocol at any block size and head dim, fp32
 * (replaces _kernels/pyref.py:14-48 masked_block_attention and
 * _kernels/_core.pyx:14-101): q, k, v float32 [n, d] (d <= 256); active
 * uint8 [t_q]; pair_bits uint8 [t_q, t_kv] (t = ceil(n / b)). Writes the rows
 * of active blocks of out (others untouched), adds the computed pair count to
 * *pairs (optional) and raises CONSISTENCY in *status for an active block
 * with no key block (the reference's l <= 0 error). The tcgen05 kernel
 * (fo_sparse_attention) is the path for 128-token blocks. */
FO_API int fo_masked_block_attention_f32(const float* q, const float* k, const float* v, int n,
                                         int d, const uint8_t* active, const uint8_t* pair_bits,
                                         int b_q, int b_k, float scale, float* out,
                                         unsigned long long* pairs, uint32_t* status,
                                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FLASHOMNI_B200_H */
