/*
 * swiftdec_b200.h — C ABI of the B200 decode-step library (libswiftdec_b200.so).
 *
 * Drop-in boundary for the TokenSwift decode step (arXiv 2502.18890). The
 * reference (swiftdec, pure Python/numpy) has no native FFI; the entry points
 * below are what a ctypes binding inside swiftdec would call in place of the
 * numpy code cited beside each one (paths relative to
 * /root/reference/pkg/src/swiftdec/). INTEGRATION.md shows that binding.
 *
 * Conventions
 *  - Every pointer is DEVICE memory unless its name ends in `_host`.
 *  - Sizes are element counts. `stream` is a cudaStream_t.
 *  - dtype codes: SD_F32 = 0 (float), SD_BF16 = 1 (__nv_bfloat16), SD_F64 = 2.
 *  - Functions never allocate, never synchronise the host, keep no global
 *    mutable state, and return SD_OK or an error code; sd_last_error() gives
 *    a message for the calling thread. Argument validation that raises typed
 *    exceptions in the reference stays in the host layer.
 *  - KV layout, one layer: [kv_head][row][head_dim], `head_stride` elements
 *    between heads (= capacity * head_dim). Layers are `layer_stride` apart.
 */
#ifndef SWIFTDEC_B200_H
#define SWIFTDEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* exported even when the library is compiled with -fvisibility=hidden */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define SD_OK 0
#define SD_EINVAL 1
#define SD_ECUDA 2
#define SD_EUNSUPPORTED 3

#define SD_F32 0
#define SD_BF16 1
#define SD_F64 2

/* fixed capacities of the device tree / step-result records */
#define SD_TREE_MAX_ROWS 256   /* 1 + nodes */
#define SD_TREE_MAX_PATHS 512
#define SD_TREE_MAX_DEPTH 8
#define SD_MASK_WORDS 8        /* SD_TREE_MAX_ROWS / 32 */

typedef void* sd_stream_t;

int sd_version(void);
const char* sd_last_error(void);

/* Post-process a captured step graph (cudaGraph_t, before instantiation):
 * programmatic edges from a kernel outside this library (cuBLAS) to one of
 * ours are moved to the predecessor's launch-completion port, so our kernel
 * launches while the library kernel runs and waits in griddepcontrol.wait.
 * Not a reference interface: graph scheduling of the step. */
int sd_graph_relax_library_edges(void* graph, int* relaxed_out);

/* ---- dense-layer plumbing (model.py:234-236, 278, 306-311) ---- */
/* h[t,:] = embed[tokens[t],:] (as f32) */
int sd_embed(const int32_t* tokens, int T, const void* embed, int dtype, int d, float* h, sd_stream_t stream);
/* h += delta (if delta); x = h * gain / sqrt(mean(h^2) + eps) -> x (x_dtype).
 * delta may be `delta_splits` split-K slices `delta_split_stride` floats apart
 * (sd_gemm output), summed in slice order. */
int sd_add_rmsnorm(float* h, const float* delta, int T, int d, const float* gain, float eps,
                   void* x, int x_dtype, int delta_splits, int64_t delta_split_stride, sd_stream_t stream);
/* out = a / (1 + exp(-a)) */
int sd_silu(const float* a, void* out, int out_dtype, size_t n, sd_stream_t stream);
/* sd_silu over a [T][N] projection whose rows past *rows_dev (the tree record's
 * live row count; NULL: all T) are padding and left untouched. */
int sd_silu_rows(const float* a, void* out, int out_dtype, int T, int N, const int32_t* rows_dev,
                 sd_stream_t stream);
/* out = a + b (f32), cast_out = (cast_dtype) out (nullable) */
int sd_add_cast(const float* a, const float* b, float* out, void* cast_out, int cast_dtype, size_t n,
                sd_stream_t stream);

/* ---- RoPE + KV staging (model.py:216-232, 276-289; kvcache.py:91-96) ----
 * qkv: [T][(H + 2*Hk) * dh] f32 (columns q | k | v). Interleaved-pair RoPE at
 * positions[t] from fp64-derived cos/sin tables [max_pos][dh/2] (f32).
 * q_rot = rope(q) * q_scale -> [T][H][dh] (q_dtype); q_pre = q (f32, nullable).
 * k_raw (nullable), k_rot, v written at row (row_offset + t) of each kv head.
 * qkv may be `qkv_splits` split-K slices (sd_gemm) `qkv_split_stride` floats
 * apart, summed in slice order.
 * rows_dev (nullable): rows t >= *rows_dev are skipped. row_offset < 0: rows go
 * to positions[0] + t (device-resident offset; k_raw / k_rot / v then point
 * at row 0 of the layer). Launched as a programmatic dependent: positions,
 * rows_dev and the tables are read before the dependency wait, so they must
 * come from an ordinary launch or copy (tree record, host fill), not from a
 * kernel of the same programmatic-dependent chain; qkv may. */
int sd_rope_stage(const float* qkv, int T, int H, int Hk, int dh, const int32_t* positions,
                  const float* rope_cos, const float* rope_sin, float q_scale,
                  void* q_rot, int q_dtype, float* q_pre,
                  void* k_raw, void* k_rot, void* v, int kv_dtype, int64_t head_stride, int64_t row_offset,
                  const int32_t* rows_dev, int qkv_splits, int64_t qkv_split_stride, sd_stream_t stream);

/* ---- split-KV attention: verify tree / draft / AR (model.py:238-247, 290-305) ----
 * Row t (query head j uses kv head j / (H/Hk)) attends to
 *   cache rows [0, ctx)  (src_kind 0: k_cache holds K_rot;
 *                          src_kind 1: k_cache holds K_raw of partial-cache
 *                          slots, rotated on load at rank ranks[slot] —
 *                          kvcache.py:158-165)
 *   + tree rows j <= t of the request with mask bit j set (mask_bits
 *     [T][mask_words]; NULL = causal). Self is always visible.
 * q: [T][H][dh] (q_dtype, already rotated and scaled). out: [T][H][dh].
 * T <= SD_TREE_MAX_ROWS. rows_dev (nullable): live row count <= T read on
 * device (rows beyond it produce zeros), so a padded verify forward needs no
 * host round trip. Partial-cache slots with rank < 0 are holes and skipped.
 * ctx_dev (nullable, src_kind 0): live cache length read on device; `ctx` is
 * then an upper bound that sizes the grid and workspace, and the tree rows are
 * taken from k_cache / v_cache right after the live rows (k_tree / v_tree are
 * ignored). With ctx_dev every argument is step-invariant, so the call can be
 * captured once in a CUDA graph and replayed as the cache grows.
 * Split boundaries depend on ctx only — the tensor-core path also on
 * kv_heads_total, the model's kv heads over all shards (0 = Hk) — so a kv
 * head's output is bitwise identical for any number of GPUs sharing the heads
 * (SURVEY H7). The tensor-core and draft
 * kernels are programmatic dependent launches: rows_dev, ctx_dev, ranks and
 * the committed cache rows are read before the dependency wait, so they must
 * not be written by the kernel launched immediately before (q, the tree rows
 * and the pending row may be). */
/* The workspace starts with SD_ATTN_WS_HEAD bytes of arrival counters: zero
 * them once when the workspace is allocated; every call leaves them zero. */
#define SD_ATTN_WS_HEAD 4096
size_t sd_attention_workspace_bytes(int T, int H, int dh, int ctx);
int sd_attention(const void* q, int q_dtype, int T, int H, int Hk, int dh,
                 int src_kind, const void* k_cache, const void* v_cache, int kv_dtype, int64_t head_stride,
                 int ctx, const int32_t* ranks, const float* rope_cos, const float* rope_sin,
                 const void* k_tree, const void* v_tree, int64_t tree_head_stride,
                 const uint32_t* mask_bits, int mask_words, const int32_t* rows_dev, const int32_t* ctx_dev,
                 const void* tmap_k_host, const void* tmap_v_host, int layer, int kv_heads_total,
                 void* out, int out_dtype, void* workspace, size_t workspace_bytes, sd_stream_t stream);
/* 128-byte TMA descriptor (CUtensorMap) over a whole [L][Hk][cap][128] bf16
 * cache array. When sd_attention gets descriptors for K_rot and V (and the
 * call is bf16 / head_dim 128 / src_kind 0), the cache chunks run on the
 * tcgen05 tensor-core kernel (TMA-fed, accumulators in TMEM) of `layer`;
 * k_cache / v_cache must then be that layer's slice of the described arrays. */
int sd_make_kv_tmap(const void* base, int L, int Hk, int cap, int dh, void* tmap_out_host);
/* Same descriptor with 64-slot boxes, over a partial cache's K_raw / V slot
 * arrays [L][Hk][slot_cap][128] bf16. When sd_attention gets these with
 * src_kind 1 (T == 1, bf16, head_dim 128, H / Hk <= 16), the draft attention
 * runs on the TMA-fed warp-level tensor-core kernel of `layer` (rank-RoPE in
 * registers, split merge and the pending row fused; replaces the reference's
 * draft_view + causal forward, kvcache.py:227-240, model.py:301-305). */
int sd_make_slot_tmap(const void* base, int L, int Hk, int cap, int dh, void* tmap_out_host);
/* DEBUG ONLY (the one piece of global state): route clock64 event stamps of
 * the tensor-core kernel's first CTA to int64 [4][64][8] at trace_dev (NULL
 * disables); force_chunks > 0 overrides the chunk count. Not used by the
 * product path. */
int sd_debug_tc_trace(void* trace_dev, int force_chunks);

/* ---- weight-streaming dense layers (model.py:283-285, 306-309) ----
 * Y = X[M][K] . W[K][N] (bf16 in, fp32 accumulate) on tcgen05, M <= 128
 * (decode rows), K % 64 == 0, N % 128 == 0. The weight is stored N-tiled,
 * [N/128][K][128] (sd_tile_weight from the row-major [K][N] reference layout),
 * stored as [N/128][2][K][64]) and described once by sd_make_weight_tmap.
 * epi SD_GEMM_EPI_F32: y holds S = sd_gemm_splits(M, N, K, epi) fp32 split-K
 * slices [S][M][ldy] whose in-order sum is Y (sd_add_rmsnorm / sd_rope_stage
 * take the slices directly). SD_GEMM_EPI_SILU_BF16: y = bf16 silu(Y) [M][ldy]
 * (the MLP's non-gated SiLU); for M <= 16 it is split-K too, reduced in split
 * order inside the kernel through `workspace` (sd_gemm_workspace_bytes; zero it
 * once before first use — the kernel leaves it zeroed). */
#define SD_GEMM_EPI_F32 0
#define SD_GEMM_EPI_SILU_BF16 1
#define SD_GEMM_EPI_ADDNORM 2 /* internal to sd_gemv_addnorm */
#define SD_GEMM_EPI_ROPE 3    /* internal to sd_gemv_rope */
int sd_tile_weight(const void* w, int K, int N, void* w_tiled, sd_stream_t stream);
int sd_make_weight_tmap(const void* w_tiled, int K, int N, void* tmap_out_host);
int sd_gemm_splits(int M, int N, int K, int epi);
size_t sd_gemm_workspace_bytes(int M, int N, int K);
int sd_gemm(const void* x, int M, int K, const void* w_tmap_host, int N, int epi, void* y, int64_t ldy,
            void* workspace, size_t workspace_bytes, sd_stream_t stream);

/* ---- few-row weight streaming (the verification forward's tree rows,
 * model.py:283-285, 306-309) ----
 * y = S = sd_gemm_rows_splits(K, N) fp32 split-K slices [S][T][N] whose in-order
 * sum is x[T][K] . W[K][N]; x, W bf16 (W row-major, the reference layout);
 * T <= 112, K % 32 == 0, N % 256 == 0. With rows_dev (device int: the tree
 * record's live row count) only rows < min(*rows_dev, T) are computed and
 * written. sd_add_rmsnorm / sd_rope_stage take the slices directly. */
int sd_gemm_rows_splits(int K, int N);
int sd_gemm_rows(const void* x, int T, int K, const void* w, int N, const int32_t* rows_dev, float* y,
                 sd_stream_t stream);

/* ---- single-row weight streaming (the draft forward's projections and draft
 * heads, model.py:104-120, 283-285, 306-309) ----
 * y[N] = x[K] . W[K][N]; x, W bf16 (W row-major, the reference layout), fp32
 * accumulate; epi SD_GEMM_EPI_F32 -> fp32 y, SD_GEMM_EPI_SILU_BF16 -> bf16 silu.
 * N % 8 == 0. K is split across CTAs and reduced in slice order by the last
 * CTA of each column block through `workspace` (sd_gemv_workspace_bytes; zero
 * it once, calls leave it zeroed). */
size_t sd_gemv_workspace_bytes(int K, int N);
int sd_gemv(const void* x, int K, const void* w, int N, int epi, void* y, void* workspace, size_t workspace_bytes,
            sd_stream_t stream);
/* Projection fused with the residual add + RMSNorm that follows it
 * (model.py:278, 306-311): h[N] += x[K] . W[K][N]; x_out = h * gain / rms(h)
 * (x_dtype SD_BF16 / SD_F32). The last column block to finish normalises the
 * row, so the pair is one launch; same workspace as sd_gemv. */
/* one row, the norm folded into the projection's input (model.py:306-311):
 * h_out = h_in + delta; x = bf16(rmsnorm(h_out) * gain) computed in the kernel;
 * y = x . W with the sd_gemv epilogues. h_out must not alias h_in. */
int sd_gemv_norm(const float* h_in, const float* delta, const float* gain, float eps, float* h_out, int K,
                 const void* w, int N, int epi, void* y, void* workspace, size_t workspace_bytes,
                 sd_stream_t stream);
/* The draft row's QKV projection with RoPE + staging as its epilogue (replaces
 * sd_gemv(_norm) + sd_rope_stage for one row, model.py:216-232, 283-289): the
 * input is bf16 x, or (h_in, delta, gain) as in sd_gemv_norm; the output is
 * q_rot [H][dh] (bf16, rotated at *pos and scaled by q_scale), k_rot [Hk][dh]
 * (rotated) and v [Hk][dh] (bf16); N = (H + 2 Hk) dh; cos/sin tables as
 * sd_rope_stage. */
int sd_gemv_rope(const void* x, const float* h_in, const float* delta, const float* gain, float eps, float* h_out,
                 int K, const void* w, int N, const int32_t* pos, const float* cos_table, const float* sin_table,
                 float q_scale, int H, int Hk, int dh, void* q_rot, void* k_rot, void* v, void* workspace,
                 size_t workspace_bytes, sd_stream_t stream);
int sd_gemv_addnorm(const void* x, int K, const void* w, int N, float* h, const float* gain, float eps, void* x_out,
                    int x_dtype, void* workspace, size_t workspace_bytes, sd_stream_t stream);

/* ---- Eq. 2 importance (kvcache.py:243-265) ----
 * scores[l][p - start] = sum_k sum_g q_sum[l][k*G+g] . K_raw[l][k][p], p in [start, end),
 * heads summed in ascending order. per_head (nullable): [L][Hk][end-start]. */
int sd_importance_scores(const float* q_sum, const void* k_raw, int kv_dtype, int64_t layer_stride,
                         int64_t head_stride, int L, int H, int Hk, int dh, int start, int end,
                         float* scores, float* per_head, sd_stream_t stream);
/* scores[l][i] = sum over kv heads (ascending) of per_head[l][k][i]; used after
 * an all-gather of per-head partials (sharded refresh). */
int sd_sum_head_scores(const float* per_head, int L, int Hk, int n, float* scores, sd_stream_t stream);

/* ---- partial cache build / maintenance (kvcache.py:191-354) ----
 * Device layout per layer l (slot_cap slots; every array [L][slot_cap]):
 *   ppos / prank / pscore  slot metadata: position, rank (dense position order
 *                          of the live slots: the draft rotation angle,
 *                          kvcache.py:158-165), score (NaN = unscored); holes
 *                          have pos = rank = -1
 *   pk / pv                K_raw / V as [L][Hk][slot_cap][dh]
 *   ring                   the body's slot ids in importance order (circular;
 *                          head / length in meta): the reference's body list
 *                          order (sink first, then body, kvcache.py:197)
 *   freel                  free-slot stack (holes below hi)
 *   meta [L][SD_PM_WORDS]  count, hi, ring head, ring length, free count, error
 * All bookkeeping lives on the device, so the per-step admit/evict runs inside
 * the step's CUDA graph without a host round trip. */
#define SD_PM_COUNT 0
#define SD_PM_HI 1
#define SD_PM_HEAD 2
#define SD_PM_LEN 3
#define SD_PM_NFREE 4
#define SD_PM_ERR 5
#define SD_PM_WORDS 8
size_t sd_refresh_workspace_bytes(int L, int n_cand, int take);
/* refresh / prefill_partial (kvcache.py:268-297, 327-329; engine.py:128-151):
 * one launch = Eq. 2 scores of positions [sink, upto) from q_sum and K_raw
 * (or the precomputed scores_in [L][upto-sink] of a sharded refresh), the
 * per-layer top-(budget-sink) by (-score, pos), the K_raw / V gather into
 * slots [0, budget) (sink, then the body in position order) and the
 * importance ring. */
int sd_partial_refresh(const float* q_sum, const float* scores_in, int L, int H, int Hk, int dh, int upto,
                       int sink, int budget, const void* full_k_raw, const void* full_v, int kv_dtype,
                       int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                       int64_t part_layer_stride, int64_t part_head_stride, int slot_cap, int32_t* ppos,
                       int32_t* prank, float* pscore, int32_t* ring, int32_t* freel, int32_t* meta,
                       void* workspace, size_t workspace_bytes, sd_stream_t stream);
/* mirror_partial (kvcache.py:300-319): slot s <- position s < upto, body ring
 * newest first. */
int sd_partial_mirror(int L, int Hk, int dh, int upto, int sink, const void* full_k_raw, const void* full_v,
                      int kv_dtype, int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                      int64_t part_layer_stride, int64_t part_head_stride, int slot_cap, int32_t* ppos,
                      int32_t* prank, float* pscore, int32_t* ring, int32_t* freel, int32_t* meta,
                      sd_stream_t stream);
/* admit (kvcache.py:215-225) of positions first..first+a-1 at the ring head,
 * then (evict != 0) evict_to_budget (kvcache.py:332-354) from the ring tail.
 * With `result` (engine, engine.py:281-283) a = result[SD_RES_ACCEPTED],
 * first = result[SD_RES_BASE], protected = a, read on the device; else the
 * host values (a <= 1024 per launch). A SinkViolation leaves the cache
 * unchanged and sets meta[l][SD_PM_ERR]. */
int sd_partial_step(int L, const int32_t* result, int a_host, int first_pos_host, int evict, int protected_host,
                    int sink, int budget, int Hk, int dh, const void* full_k_raw, const void* full_v, int kv_dtype,
                    int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                    int64_t part_layer_stride, int64_t part_head_stride, int slot_cap, int32_t* ppos,
                    int32_t* prank, float* pscore, int32_t* ring, int32_t* freel, int32_t* meta,
                    sd_stream_t stream);

/* ---- reconcile (kvcache.py:116-127) + last_queries (engine.py:280) ----
 * keep offsets / count read from the device step result. Rows base+keep[i] ->
 * base+i for K_raw, K_rot, V; q_sum[l][h] = sum_i q_pre[l][keep[i]][h]. */
int sd_reconcile(int L, const int32_t* result, int base_len, void* k_raw, void* k_rot, void* v, int kv_dtype,
                 int64_t layer_stride, int64_t head_stride, int Hk, int dh,
                 const float* q_pre, int q_rows, int H, float* q_sum, sd_stream_t stream);

/* ---- sampling (sampling.py:142-224, engine.py:155-181, 207-245) ---- */
/* member mask source for sd_sample_rows */
#define SD_MEMBER_NONE 0     /* no penalty                                      */
#define SD_MEMBER_MASK 1     /* explicit uint8 mask [rows][V]                    */
#define SD_MEMBER_WINDOW 2   /* window counts, all rows (draft heads / AR)       */
#define SD_MEMBER_TREE 3     /* window counts + per-row branch splice (verify)   */
#define SD_TRUNC_NONE 0
#define SD_TRUNC_TOP_P 1
#define SD_TRUNC_MIN_P 2
#define SD_TRUNC_ETA 3
#define SD_IN_LOGITS_F32 0
#define SD_IN_LOGITS_F64 1
#define SD_IN_PROBS_F64 2
#define SD_IN_SCALED_F32 3 /* penalised scaled fp32 logits + per-tile statistics from sd_lmhead_sample_stats */

typedef struct {
  int rows, V, in_kind;
  double temperature, theta;
  int ctrl_style;
  int member_kind;
  const uint8_t* member_mask;      /* SD_MEMBER_MASK */
  const int32_t* win_count;        /* [V] */
  const int32_t* win_ring;         /* [W] ring storage */
  const int64_t* state;            /* device session state (ring head/len) */
  int window;                      /* W */
  const int32_t* tree;             /* device tree record (SD_MEMBER_TREE) */
  int depth;                       /* gamma + 1 */
  int trunc_kind;
  double trunc_value, eta_alpha;   /* eta_alpha < 0 -> sqrt(eps) */
  uint64_t seed;
  const int32_t* positions;        /* [rows] draw keys; NULL -> tree-derived (n, n+d+1) */
  int64_t n;                       /* tree-derived keys: row 0 -> n, node -> n + depth + 1 */
  double* probs_out;               /* nullable [rows][V]: penalised softmax */
  double* trunc_out;               /* nullable [rows][V]: truncated + renormalised */
  int32_t* token_out;              /* nullable [rows]: inverse-CDF draw */
  const double* stats;             /* SD_IN_SCALED_F32 only: [rows][stats_tiles][2] (max, sum exp(s - max)) per
                                      128-token tile of the penalised, scaled logits (sd_lmhead_sample_stats) */
  int stats_tiles;
} sd_sample_args;
int sd_sample_rows(const void* in, const sd_sample_args* args_host, sd_stream_t stream);

/* Verification LM head fused with the sampler's first pass (
 * replaces `logits = h0 @ embed.T` + the penalty/softmax-statistics half of
 * penalized_probs_masked, engine.py:237-245 / sampling.py:98-153, which the
 * reference computes over [T, V] in numpy). x: bf16 h0 [M][K] (M <= 128),
 * embed_tmap: sd_make_lmhead_tmap of the tied bf16 embedding [V][K] re-laid by
 * sd_tile_lmhead into contiguous 16 KB (128-token x 64-wide) boxes
 * (sd_lmhead_tiled_bytes). The
 * penalty fields of `args` (temperature, theta, ctrl_style, member_kind NONE /
 * WINDOW / TREE with its window and tree record) are applied in the epilogue;
 * writes logits [M][V] = penalised logits / temperature (fp32) and stats
 * [M][sd_lmhead_tiles(V)][2] = (max, sum exp(s - max)) per 128-token tile, for
 * the tree's live rows only. Follow with sd_sample_rows(in_kind =
 * SD_IN_SCALED_F32, stats, stats_tiles). tcgen05 + TMA, sm_100a. */
size_t sd_lmhead_tiled_bytes(int V, int K);
int sd_tile_lmhead(const void* embed, int V, int K, void* tiled, sd_stream_t stream);
int sd_make_lmhead_tmap(const void* tiled, int V, int K, void* tmap_out_host /* 128 bytes */);
int sd_lmhead_tiles(int V);
int sd_lmhead_sample_stats(const void* x, int M, int K, const void* embed_tmap_host, int V,
                           const sd_sample_args* args_host, float* logits, double* stats, sd_stream_t stream);

/* per-head top-w of the penalised draft distributions, ties to lower id
 * (engine.py:207-215). out: concatenated candidates, head k gets widths[k]. */
int sd_draft_topw(const float* logits, int heads, int V, const int32_t* win_count, double temperature,
                  double theta, int ctrl_style, const int32_t* widths_host, int32_t* out, sd_stream_t stream);

/* ---- n-gram table (ngram.py:18-66): open-addressing hash + per-first-token chains ----
 * Table memory = sd_ngram_bytes(n, cap, V) bytes, zero-initialised by sd_ngram_init. */
size_t sd_ngram_bytes(int n, int cap, int V);
int sd_ngram_init(void* table, int n, int cap, int V, sd_stream_t stream);
int sd_ngram_update(void* table, const int32_t* seq, int n_tail, int n_new, sd_stream_t stream);
/* out_grams [k][n], out_count [1] */
int sd_ngram_retrieve(const void* table, const int32_t* first, int k, int32_t* out_grams, int32_t* out_count,
                      sd_stream_t stream);
int sd_ngram_frequency(const void* table, const int32_t* grams, int count, int32_t* out, sd_stream_t stream);
int sd_ngram_size(const void* table, int32_t* out, sd_stream_t stream);

/* ---- tree (tree.py:87-175) + acceptance/commit (engine.py:247-290) ----
 * Device tree record layout: see sd_tree_layout(). */
int sd_tree_layout(int32_t* offsets_host, int n);
/* per_head: concatenated candidates; grams [n_grams][depth] (n_grams from
 * device when n_grams_dev != NULL, else n_grams_host). Writes the verify rows:
 * row 0 = pending (state) at base_pos, node i at base_pos + 1 + depth. */
int sd_tree_build(const int32_t* per_head, const int32_t* widths_host, int depth, const int32_t* grams,
                  const int32_t* n_grams_dev, int n_grams_host, const int64_t* state, int64_t base_pos,
                  int32_t* tree, sd_stream_t stream);
/* retrieve (first = per_head[0]) + build in one launch */
int sd_draft_tree(const void* ngram_table, int k, const int32_t* per_head, const int32_t* widths_host,
                  int depth, const int64_t* state, int64_t base_pos, int32_t* grams_scratch, int32_t* tree,
                  sd_stream_t stream);

/* session state (int64[16]) slots */
#define SD_ST_RING_HEAD 0
#define SD_ST_RING_LEN 1
#define SD_ST_HIST_LEN 2
#define SD_ST_PENDING 3
#define SD_ST_ERROR 4
#define SD_ST_BASE 5        /* committed length n-1 (device-maintained by sd_accept_commit) */
/* step result (int32[32]) slots */
#define SD_RES_ACCEPTED 0
#define SD_RES_BEST 1
#define SD_RES_PICK 2
#define SD_RES_ORIGIN 3
#define SD_RES_ROWS 4
#define SD_RES_PATHS 5
#define SD_RES_PENDING 6   /* int32 copy of the pending token (next draft input) */
#define SD_RES_BASE 7      /* n-1 of the step (the verify rows' cache offset) */
#define SD_RES_YS 8
#define SD_RES_KEEP 16

/* acceptance + commit: path validity vs y, uniform pick at
 * (select_seed, n), accepted count, ys, keep offsets -> result; then window
 * push, history append, n-gram update (ngram may be NULL), pending <- last ys. */
int sd_accept_commit(const int32_t* tree, const int32_t* y, uint64_t select_seed, int64_t n, int depth, int bonus,
                     int64_t* state, int32_t* win_ring, int32_t* win_count, int window, int32_t* history,
                     void* ngram_table, int32_t* result, sd_stream_t stream);
/* push tokens into the penalty window (sampling.py:98-109) */
int sd_window_push(const int32_t* tokens, int count, int64_t* state, int32_t* win_ring, int32_t* win_count,
                   int window, sd_stream_t stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif
