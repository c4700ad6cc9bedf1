/*
 * qcfuse_b200 — C ABI of the B200-native QCFuse fused-prefill kernels.
 *
 * Every entry point takes device pointers, plain sizes and a CUDA stream, never
 * allocates, never synchronises, and returns an int status (0 = QCF_OK,
 * negative = error; qcf_last_error() holds the message for the calling thread).
 * No torch types cross this boundary. The reference package is pure Python, so
 * its "FFI" is Python calling these through ctypes; each
 * function names the reference symbol (file:line under
 * /root/reference/pkg/src/qcfuse/) whose arithmetic it replaces.
 *
 * Layouts (row-major, token-major like the reference's LayerKV and .qcfk):
 *   KV table / chunk KV : [rows][Hkv][D]   one tensor per layer (layer stride given)
 *   activations x       : [M][d]           float32 residual stream
 *   weights (GEMM B)    : [N][K]           K-major (the reference's [d_in][d_out]
 *                                           transposed once at load)
 *   positions / rows    : int32
 * dtype codes: QCF_F32 (parity mode) or QCF_BF16 (speed mode).
 */
#ifndef QCFUSE_B200_H
#define QCFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* qcf_stream_t;

enum qcf_status {
  QCF_OK = 0,
  QCF_EINVAL = -1,       /* bad argument            -> ValueError */
  QCF_ESHAPE = -2,       /* inconsistent shapes     -> ValueError */
  QCF_ECUDA = -3,        /* CUDA launch/runtime     -> RuntimeError */
  QCF_EUNSUPPORTED = -4, /* shape/dtype not built   -> NotImplementedError */
  QCF_EWORKSPACE = -5    /* workspace too small     -> ValueError */
};

enum qcf_dtype { QCF_F32 = 0, QCF_BF16 = 1 };

/* GEMM B-operand (weight) layouts. TILE64 = [N/64][K/64][64][64]: every 64x64
 * tile is 8 KB contiguous, so weight streaming reads whole DRAM pages. */
enum qcf_b_layout { QCF_B_ROWMAJOR = 0, QCF_B_TILE64 = 1 };

enum qcf_epilogue {
  QCF_EPI_STORE = 0,     /* C = acc                (C in out_dtype)          */
  QCF_EPI_RELU = 1,      /* C = max(acc, 0)        (C in out_dtype)          */
  QCF_EPI_ADD_F32 = 2    /* C(f32) += acc          (residual stream update)  */
};

/* ---- library ------------------------------------------------------------ */
const char* qcf_version(void);
const char* qcf_last_error(void);
/* 1 when the sm_100a tcgen05 GEMM is usable on the current device. */
int qcf_tc_available(void);
/* Number of bf16 GEMM / attention calls that ran on the SIMT (FFMA) kernels
 * because the shape is outside the tcgen05 contract (e.g. head dim != 128).
 * A speed-mode run reports it; it must stay 0 at the benchmarked shapes. */
long long qcf_simt_fallbacks(void);
/* 1: such a bf16 call fails with QCF_EUNSUPPORTED instead of running on SIMT
 * (also env QCF_STRICT_TC=1). 0 (default): it runs on SIMT and is counted. */
int qcf_set_strict_tc(int on);

/* ---- deterministic init: model.py:35-46 (splitmix64_at), 67-69, 225-257 ----
 * Writes draws [start, start + rows*cols) of the splitmix64 stream keyed by
 * `seed`, each mapped to float32(-0.05 + 0.1*u53), as a rows x cols row-major
 * matrix; with transpose=1 the matrix is written as out[c*ld_out + r] (K-major
 * GEMM operand). out_dtype f32 or bf16 (bf16 = round-to-nearest of the f32). */
int qcf_init_uniform(uint64_t seed, uint64_t start, int64_t rows, int64_t cols,
                     int transpose, int out_dtype, void* out, int64_t ld_out,
                     qcf_stream_t stream);

/* ---- fused-context assembly: fusion.py:234-263 + model.py:271-292 ---------- */
typedef struct {
  const void* k;          /* chunk K, layer 0 row 0 ([L][n_tok][Hkv][D])       */
  const void* v;          /* chunk V                                          */
  int64_t layer_stride;   /* elements between consecutive layers              */
  int32_t n_tok;          /* chunk length S_c                                 */
  int32_t offset;         /* fused row of the chunk's first token (off_c >= 1)*/
} qcf_chunk_desc;

/* fused_k[l][off_c + i] = R(off_c) . chunk_k[l][i]   (re-rotation composes)
 * fused_v[l][off_c + i] = chunk_v[l][i]                (bit copy)
 * fused_*[l][0]         = bos_*[l]                     (BOS row, position 0)
 * `chunks` is a DEVICE array of n_chunks descriptors. cos/sin tables are float64
 * [n_pos][D/2] built on the host exactly as model.py:264-280 builds the angles.
 * fused_v may be NULL: K only (the f32 critical-layer keys of the fp32
 * scoring mode); bos_v and the descriptors' v are then not read. */
int qcf_assemble(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                 const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                 int64_t fused_layer_stride, int n_layers, int hkv, int d,
                 const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                 int dtype, qcf_stream_t stream);

/* Same with an explicit rotation delta per chunk (device int32 array, NULL =
 * the chunk's fused row offset; max_delta bounds the table lookup). Rows land at
 * desc.offset.. but K rotates by deltas[c]: used to build the probe's anchor
 * prefix [BOS | R(off_c) K_c[anchors] ...] (fusion.py:281-303) straight from
 * device-resident anchor rows when the chunk pool lives in host memory. */
/* Layers [layer0, layer0 + n_layers) only (bos_k/bos_v, fused_k/fused_v and the
 * descriptors' k/v still point at layer 0): lets the assembly of layer l run on a
 * side stream while the recompute works on earlier layers (fusion.py:234-263 per layer). */
int qcf_assemble_range(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                       const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                       int64_t fused_layer_stride, int layer0, int n_layers, int hkv, int d,
                       const double* cos_tbl, const double* sin_tbl, int64_t n_pos, int dtype,
                       qcf_stream_t stream);
/* qcf_assemble_range that leaves out the fused rows whose bit is set in skip_rows
 * (device bitmap, bit r of word r/32 = fused row r): the selected rows, which the
 * recompute rewrites in every layer (fusion.py:477-478), so their chunk K/V are
 * neither read nor written (the same final table, ~15% fewer assembly bytes). */
int qcf_assemble_range_skip(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                            const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                            int64_t fused_layer_stride, int layer0, int n_layers, int hkv, int d,
                            const double* cos_tbl, const double* sin_tbl, int64_t n_pos, int dtype,
                            const uint32_t* skip_rows, qcf_stream_t stream);
/* Bitmap of rows: for each of n_req requests, bit p of bitmap[r * words_per_req ..]
 * is set for every pos[r * stride + i] > 0, i < n_per_req (the recompute rows'
 * positions; BOS / padding entries are 0). */
int qcf_rows_bitmap(const int32_t* pos, int64_t stride, int n_req, int64_t n_per_req, uint32_t* bitmap,
                    int64_t words_per_req, qcf_stream_t stream);
int qcf_assemble_rot(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                     const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                     int64_t fused_layer_stride, int n_layers, int hkv, int d,
                     const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                     const int32_t* deltas, int max_delta, int dtype, qcf_stream_t stream);

/* dst[l][i] = src[l][rows[i]] for K and V (anchor prefix gather, fusion.py:281-303) */
int qcf_gather_rows(const void* src_k, const void* src_v, int64_t src_layer_stride,
                    const int32_t* rows, int64_t n_rows, void* dst_k, void* dst_v,
                    int64_t dst_layer_stride, int n_layers, int64_t row_elems,
                    int dtype, qcf_stream_t stream);

/* ---- per-row ops: model.py:305-308 (LN), fusion.py:464 (embedding gather) -- */
/* x[i] = emb[tokens[rows ? rows[i] - row_base : i]]  (float32 residual stream) */
int qcf_embed(const int32_t* tokens, const int32_t* rows, int32_t row_base, int64_t m,
              const float* emb, int d, float* x, qcf_stream_t stream);
/* out[i] = (x[i]-mean)/sqrt(var+eps)*g + b ; out in out_dtype */
int qcf_layernorm(const float* x, int64_t m, int d, const float* g, const float* b,
                  float eps, void* out, int out_dtype, qcf_stream_t stream);
/* x += delta (residual update, written back), then out = LN(x). delta may be
 * NULL (= qcf_layernorm). Fuses model.py:375-376's residual adds into the
 * following LayerNorm so the projections store instead of read-modify-write. */
int qcf_add_layernorm(float* x, const float* delta, int64_t m, int d, const float* g, const float* b,
                      float eps, void* out, int out_dtype, qcf_stream_t stream);
/* x[i] += delta[i] for n floats (n % 4 == 0, 16-byte aligned) */
int qcf_add_rows(float* x, const float* delta, int64_t n, qcf_stream_t stream);
/* logits[r] = LN_f(x[rows[r]]) @ emb^T  (model.py:384-385, fusion.py:540) */
int qcf_lm_head(const float* x, const int32_t* rows, int64_t n_rows, int d,
                const float* g, const float* b, float eps, const float* emb,
                int vocab, float* logits, qcf_stream_t stream);
/* Greedy decode step on the device (model.py:433-465): t = argmax(logits[0:vocab])
 * (ties -> lowest index, like np.argmax); log_tokens[*step] = t (if *step < log_cap);
 * *tok = t; *pos += 1; *step += 1. Lets a CUDA graph of one decode step replay
 * without a host round trip per token. */
int qcf_decode_advance(const float* logits, int vocab, int32_t* tok, int32_t* pos, int32_t* step,
                       int32_t* log_tokens, int log_cap, qcf_stream_t stream);
/* norms[i] = mean_h ||k[i,h,:]||_2   (store.py:339-340) */
int qcf_key_norms(const void* k, int64_t n, int hkv, int d, float* norms, int dtype,
                  qcf_stream_t stream);

/* ---- projections: model.py:361-363, 375, 341-342 ---------------------------
 * C[M,N] (op)= A[M,K] . B[N,K]^T, A/B in `dtype` (bf16 -> tcgen05 tensor cores,
 * f32 -> FFMA parity kernel), fp32 accumulation, epilogue per qcf_epilogue. */
int qcf_gemm(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb,
             void* c, int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue,
             int out_dtype, qcf_stream_t stream);
/* Same contract with a caller-owned workspace (qcf_gemm_workspace() bytes,
 * ZERO-FILLED once before first use; the kernels leave its flag words zeroed):
 *  - skinny M (<= 256, the probe's q rows) splits K across the CTAs of a thread-
 *    block cluster so the weights stream at HBM rate; the fp32 partials are summed
 *    in rank order through distributed shared memory (deterministic, no workspace
 *    needed; the older global-memory split-K with a workspace remains the fallback);
 *  - opt-in (qcf_set_gemm_plan +8) stream-K for the 2-CTA kernel: equal k-block
 *    ranges per CTA pair, split tiles fixed up through the workspace in
 *    cluster order (deterministic).
 * ws may be NULL (no split-K / stream-K). */
size_t qcf_gemm_workspace(int64_t m, int64_t n, int64_t k);
int qcf_gemm_ws(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc,
                int64_t m, int64_t n, int64_t k, int epilogue, int out_dtype, int b_layout, void* ws,
                size_t ws_bytes, qcf_stream_t stream);
/* Same contract, forced onto the SIMT path (cross-check of the tensor-core path). */
int qcf_gemm_simt(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb,
                  void* c, int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue,
                  int out_dtype, qcf_stream_t stream);

/* ---- RoPE at absolute positions + KV scatter: fusion.py:471-478 ------------
 * qkv: float32 [M][(H + 2*Hkv)*D] (Q | K | V). q_out[i] = R(pos[i]).Q[i]
 * (dtype); k_tab[dst_rows[i]] = R(pos[i]).K[i]; v_tab[dst_rows[i]] = V[i]. */
int qcf_rope_qkv_scatter(const float* qkv, int64_t m, int h, int hkv, int d,
                         const int32_t* pos, const int32_t* dst_rows,
                         const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                         void* q_out, void* k_tab, void* v_tab, int dtype,
                         qcf_stream_t stream);

/* Fused QKV projection + RoPE + KV scatter (bf16, tcgen05): the projection
 * a[M,K] . w[(H+2Hkv)D, K]^T never touches HBM in fp32; its epilogue rotates
 * Q/K at pos[i] and writes q_out[i], k_tab[dst_rows[i]], v_tab[dst_rows[i]].
 * M <= 256 (the probe's query rows): cluster split-K weight streaming with the
 * rotation + scatter applied in the distributed-shared-memory reduction; other M:
 * the 2-CTA (normal or swapped) tiles, rotation in the epilogue (bit-identical
 * across the two orientations). Returns QCF_EUNSUPPORTED when d % 32 != 0 (callers then use
 * qcf_gemm + qcf_rope_qkv_scatter). fusion.py:470-478.
 * cs_tbl: float32 [n_pos][d/2][2] = (float(cos), float(sin)) of the float64
 * angle table (the bf16 epilogue rotates in fp32; 16-byte aligned). */
int qcf_gemm_qkv_rope(const void* a, int64_t lda, const void* w, int64_t ldb, int b_layout, int64_t m, int64_t k,
                      int h, int hkv, int d, const int32_t* pos, const int32_t* dst_rows,
                      const float* cs_tbl, int64_t n_pos, void* q_out,
                      void* k_tab, void* v_tab, void* ws, size_t ws_bytes, qcf_stream_t stream);

/* ---- location-aware attention: fusion.py:194-208 -> model.py:326-338 -------
 * out[i,h] = sum_{j<=kmax[i]} softmax_j(q[i,h].k[j,h/(H/Hkv)] / float(sqrt(D))) v[j]
 * q/out [M][H][D], k/v table [n_keys][Hkv][D]; kmax inclusive, < n_keys. */
/* Arbitrary visibility (the public sparse_attention, fusion.py:194-208):
 * key j visible to row i iff j <= kmax[i] and bit (j & 31) of
 * mask[i*mask_words + j/32] is set; every row needs one visible key. SIMT
 * (FFMA) kernel, float32 softmax; q/out [M][H][D], k/v [n_keys][Hkv][D]. */
int qcf_attention_masked(int dtype, const void* q, const void* k, const void* v, const int32_t* kmax,
                         const uint32_t* mask, int64_t mask_words, int64_t m, int h, int hkv, int d,
                         int64_t n_keys, void* out, qcf_stream_t stream);
int qcf_attention(int dtype, const void* q, const void* k, const void* v,
                  const int32_t* kmax, int64_t m, int h, int hkv, int d,
                  int64_t n_keys, void* out, qcf_stream_t stream);
/* Homogeneous request batch: q/out [n_req][m][H][D], kmax [n_req][m], K/V
 * tables [n_req][n_keys][Hkv][D] (one launch, blockIdx.z = request). */
int qcf_attention_batched(int dtype, const void* q, const void* k, const void* v,
                          const int32_t* kmax, int64_t m, int n_req, int h, int hkv, int d,
                          int64_t n_keys, void* out, qcf_stream_t stream);
/* Same with a caller-owned workspace (>= qcf_attention_workspace bytes): with
 * qcf_set_attention_split(n > 1) and tile pairs that fit in one wave of CTAs,
 * every pair's key range is split into n chunks (split-KV) whose pieces a
 * second kernel combines. Off by default: slower than single tiles at the
 * one-request fused shape on B200 (tools/attn_bench.py). */
size_t qcf_attention_workspace(int64_t m, int n_req, int h, int64_t n_keys);  /* 0: no split applies */
int qcf_attention_split(int64_t m, int n_req, int h, int64_t n_keys);         /* split-KV factor (1 = none) */
int qcf_set_attention_split(int n_split);                       /* 0 = off (default), 2..16 */
int qcf_attention_batched_ws(int dtype, const void* q, const void* k, const void* v,
                             const int32_t* kmax, int64_t m, int n_req, int h, int hkv, int d,
                             int64_t n_keys, void* out, void* ws, size_t ws_bytes,
                             qcf_stream_t stream);
/* Tuning knob (process-wide): tcgen05 attention kernel 1 = one 128-row query
 * tile per CTA over 128-key tiles; 2 = two query tiles per CTA ping-ponging on
 * the tensor core (3 = the same with one thread per full row); 4 = one query
 * tile per CTA over 64-key tiles, two CTAs resident per SM; 8 = one query tile
 * per CTA, two softmax warp groups on alternate key tiles, three S buffers;
 * 0 (default) = 4 when the grid fills both CTA slots of every SM (or one slot
 * with key ranges of at most 256 keys), split-KV pairs for one-wave grids,
 * else 1. */
int qcf_set_attention_kernel(int version);
/* Tuning knob (process-wide): tcgen05 GEMM tile plan for M > 32. 0 (default) =
 * wave-quantisation model; 1 = 2-CTA 256x256; 2 = 1-CTA 128x256; 3 = 128x128;
 * 4 = 128x64; 5 = 2-CTA 128x256 (64 rows per CTA) (falls back to auto when the
 * shape does not fit the plan);
 * +8 = stream-K schedule for the 2-CTA kernel (off by default: slower here). */
int qcf_set_gemm_plan(int plan);

/* ---- critical-layer scoring: fusion.py:313-326 + 566-569 ------------------
 * scores[n] = mean_{h,t} softmax_n((q[t,h].k[n,h]) * scale), t over all nq rows
 * (agg_last=0) or the last row (agg_last=1). precise=1 accumulates in float64.
 * workspace >= qcf_score_workspace(...) bytes. */
size_t qcf_score_workspace(int64_t n_ctx, int nq, int h);
int qcf_score(int dtype, const void* q, const void* k, int64_t n_ctx, int nq, int h,
              int hkv, int d, double scale, int agg_last, int precise, float* scores,
              void* workspace, size_t ws_bytes, qcf_stream_t stream);
/* Homogeneous request batch: q [n_req*nq][H][D]; request r's context keys start
 * at k + r*k_req_stride elements (rows of Hkv*D); scores [n_req][n_ctx].
 * bf16 with precise=0 runs on the tensor cores (tcgen05 QK^T in TMEM fused with
 * the row max/sum and the per-key (h,t) mean: 4 launches for the whole batch);
 * precise=1 / f32 run the SIMT kernels per request (float64 when precise).
 * workspace >= qcf_score_batched_workspace(...) bytes. */
size_t qcf_score_batched_workspace(int64_t n_ctx, int nq, int n_req, int h, int hkv);
int qcf_score_batched(int dtype, const void* q, const void* k, int64_t k_req_stride, int64_t n_ctx,
                      int nq, int n_req, int h, int hkv, int d, double scale, int agg_last,
                      int precise, float* scores, void* workspace, size_t ws_bytes,
                      qcf_stream_t stream);

/* ---- comparison policies: CacheBlend / KVShare, fusion.py:352-392 ----
 * KV deviation of the layer-1 recompute pass: out[n] = sum_h ||new_k - old_k||_2
 * + sum_h ||new_v - old_v||_2 (float64 norms, f32 out); tables [n][Hkv][D]. */
int qcf_kv_deviation(int dtype, const void* old_k, const void* old_v, const void* new_k, const void* new_v,
                     int64_t n, int hkv, int d, float* out, qcf_stream_t stream);
/* Received attention: out[j] = mean_{h, rows t} softmax_j((q[t,h].k[j]) * scale) over
 * keys j <= row_pos[t] (model.py:326-338 weights, averaged as fusion.py:390).
 * q [n_rows][H][D], k [n_keys][Hkv][D]; float64 accumulation; rows are
 * processed in chunks that fit the caller's workspace (>= 8*(n_keys + H*n_keys + 2H) + 256 B). */
int qcf_received_attention(int dtype, const void* q, const void* k, int64_t n_keys, int n_rows, int h,
                           int hkv, int d, double scale, const int32_t* row_pos, float* out,
                           void* workspace, size_t ws_bytes, qcf_stream_t stream);

/* ---- Top-N selection: fusion.py:141-158 (stable argsort, ties -> lower index)
 * idx_out[0..n_sel) = ascending (1-based + base) positions of the n_sel largest
 * scores, in the order numpy's stable argsort of -float64(scores) gives:
 * -0.0 == +0.0 (lower index first), NaN after every number. n_sel is computed
 * by the host as ceil(ratio*n) in double. workspace >= qcf_topn_workspace(n). */
size_t qcf_topn_workspace(int64_t n);
int qcf_topn(const float* scores, int64_t n, int64_t n_sel, int32_t base,
             int32_t* idx_out, void* workspace, size_t ws_bytes, qcf_stream_t stream);
/* Batch of n_req score rows [n_req][n]: request r's indices go to
 * idx_out + r*out_stride; dst_out (optional) receives idx + r*dst_add at the
 * same slots (the request's rows in a batched fused table). One launch. */
int qcf_topn_batched(const float* scores, int64_t n, int n_req, int64_t n_sel, int32_t base,
                     int32_t* idx_out, int64_t out_stride, int32_t* dst_out, int32_t dst_add,
                     qcf_stream_t stream);

/* The same selection over float64 scores (the public select_topn ranks
 * float64, fusion.py:156): 64-bit keys, no float32 rounding of the input. */
int qcf_topn_f64(const double* scores, int64_t n, int64_t n_sel, int32_t base, int32_t* idx_out,
                 qcf_stream_t stream);

/* Small device helpers used by the request graph. */
/* out[i] = a[i] + add (int32) */
int qcf_iota_add(const int32_t* a, int64_t n, int32_t add, int32_t* out, qcf_stream_t stream);
/* out[i] = start + i */
int qcf_iota(int64_t n, int32_t start, int32_t* out, qcf_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* QCFUSE_B200_H */
