// K4: critical-layer query->context scoring (fusion.py:313-326, _softmax_last
// fusion.py:566-569): per (head, query row) a softmax over the n_ctx context
// keys of (Q_c . K) * scale, then the mean over (head, row) per key. Three
// passes: logits into the workspace, per-row max/sum, column mean. `precise`
// runs the contraction and softmax in float64 (the fp32 parity scoring mode,
// whose float32-rounded output orders exactly like the reference's scores).
#include <math.h>

#include "common.cuh"

namespace qcf {

constexpr int SC_TILE = 64;  // keys per CTA
constexpr int SC_TQ = 32;    // query rows per CTA (4 x 8 register-tiled)

// logits S[h][t][n] = (q[t,h] . k[n,h]) * scale for a 64-key x 32-row tile of one
// head; each of 128 threads owns a 4 (rows) x 4 (keys) register tile, operands
// staged transposed in shared memory so a k-step is 2 vector loads for 16 FMAs.
template <typename T, typename Acc>
__global__ void __launch_bounds__(128) score_logits_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                           int64_t n_ctx, int nq, int t0, int h,
                                                           int hkv, int d, Acc scale,
                                                           Acc* __restrict__ S,
                                                           const int32_t* __restrict__ row_pos) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smraw[];
  Acc* Qs = reinterpret_cast<Acc*>(smraw);      // [d][SC_TQ]
  Acc* Ks = Qs + (size_t)d * SC_TQ;             // [d][SC_TILE]
  const int nt = nq - t0;
  const int head = blockIdx.y, kvh = head / (h / hkv);
  const int64_t n0 = (int64_t)blockIdx.x * SC_TILE;
  const int tq0 = blockIdx.z * SC_TQ;
  for (int e = threadIdx.x; e < SC_TQ * d; e += blockDim.x) {
    const int t = e / d, c = e % d;
    Qs[c * SC_TQ + t] = (tq0 + t < nt) ? (Acc)to_f<T>(q[((int64_t)(t0 + tq0 + t) * h + head) * d + c]) : (Acc)0;
  }
  for (int e = threadIdx.x; e < SC_TILE * d; e += blockDim.x) {
    const int j = e / d, c = e % d;
    const int64_t n = n0 + j;
    Ks[c * SC_TILE + j] = n < n_ctx ? (Acc)to_f<T>(k[(n * hkv + kvh) * d + c]) : (Acc)0;
  }
  __syncthreads();
  const int tj = threadIdx.x & 15, tt = threadIdx.x >> 4;   // 16 key quads x 8 row quads
  Acc acc[4][4] = {};
  for (int c = 0; c < d; ++c) {
    Acc qv[4], kv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) qv[i] = Qs[c * SC_TQ + tt * 4 + i];
#pragma unroll
    for (int j = 0; j < 4; ++j) kv[j] = Ks[c * SC_TILE + tj * 4 + j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += qv[i] * kv[j];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = tq0 + tt * 4 + i;
    if (t >= nt) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tj * 4 + j;
      // causal variant (received attention): key n visible to row t iff n <= row_pos[t]
      const bool vis = !row_pos || n <= (int64_t)row_pos[t0 + t];
      if (n < n_ctx) S[((int64_t)head * nt + t) * n_ctx + n] = vis ? acc[i][j] * scale : (Acc)-INFINITY;
    }
  }
}

template <typename Acc>
__global__ void score_rowstats_kernel(const Acc* __restrict__ S, int64_t n_ctx, Acc* __restrict__ rmax,
                                      Acc* __restrict__ rsum) {
  pdl_wait();
  pdl_trigger();
  __shared__ Acc red[32];
  const int64_t r = blockIdx.x;
  const Acc* s = S + r * n_ctx;
  Acc mx = -INFINITY;
  for (int64_t n = threadIdx.x; n < n_ctx; n += blockDim.x) mx = s[n] > mx ? s[n] : mx;
  for (int o = 16; o > 0; o >>= 1) { Acc t = __shfl_xor_sync(0xffffffffu, mx, o); mx = t > mx ? t : mx; }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : (Acc)-INFINITY;
    for (int o = 16; o > 0; o >>= 1) { Acc t = __shfl_xor_sync(0xffffffffu, mx, o); mx = t > mx ? t : mx; }
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  Acc sum = 0;
  for (int64_t n = threadIdx.x; n < n_ctx; n += blockDim.x) sum += exp(s[n] - mx);
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    rmax[r] = mx;
    rsum[r] = t;
  }
}

// column mean: CTA = 32 columns (lanes) x 8 warps splitting the (h,t) rows
template <typename Acc>
__global__ void __launch_bounds__(256) score_colmean_kernel(const Acc* __restrict__ S, int64_t n_ctx, int rows,
                                                            const Acc* __restrict__ rmax,
                                                            const Acc* __restrict__ rsum,
                                                            float* __restrict__ scores,
                                                            Acc* __restrict__ colacc, int first,
                                                            int last, Acc inv_total) {
  pdl_wait();
  pdl_trigger();
  __shared__ Acc part[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * 32 + lane;
  Acc acc = 0;
  if (n < n_ctx) {
#pragma unroll 4
    for (int r = warp; r < rows; r += 8) acc += exp(S[(int64_t)r * n_ctx + n] - rmax[r]) / rsum[r];
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && n < n_ctx) {
    Acc t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    if (colacc) {  // row-chunked column sums (received attention): accumulate, scale at the end
      t += first ? (Acc)0 : colacc[n];
      if (last) scores[n] = (float)(t * inv_total);
      else colacc[n] = t;
    } else {
      scores[n] = (float)(t / (Acc)rows);
    }
  }
}

template <typename T, typename Acc>
static int score_impl(const void* q, const void* k, int64_t n_ctx, int nq, int h, int hkv, int d,
                      double scale, int agg_last, float* scores, void* ws, cudaStream_t s) {
  const int t0 = agg_last ? nq - 1 : 0;
  const int nt = nq - t0;
  const int rows = h * nt;
  Acc* S = reinterpret_cast<Acc*>(ws);
  Acc* rmax = S + (int64_t)rows * n_ctx;
  Acc* rsum = rmax + rows;
  const size_t smem = sizeof(Acc) * (size_t)d * (SC_TQ + SC_TILE);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(score_logits_kernel<T, Acc>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "qcf_score attr");
  }
  QCF_REQUIRE(smem <= 220 * 1024, QCF_EUNSUPPORTED, "qcf_score: head dim too large");
  dim3 g1(ceil_div(n_ctx, SC_TILE), h, ceil_div(nt, SC_TQ));
  QCF_LAUNCH("score_logits_kernel", score_logits_kernel<T, Acc>, dim3(g1), dim3(128), smem, s, (const T*)q, (const T*)k, n_ctx, nq, t0, h, hkv,
                                                    d, (Acc)scale, S, (const int32_t*)nullptr);
  QCF_LAUNCH_CHECK("qcf_score logits");
  QCF_LAUNCH("score_rowstats_kernel", score_rowstats_kernel<Acc>, dim3(rows), dim3(256), 0, s, S, n_ctx, rmax, rsum);
  QCF_LAUNCH_CHECK("qcf_score rowstats");
  QCF_LAUNCH("score_colmean_kernel", score_colmean_kernel<Acc>, dim3(ceil_div(n_ctx, 32)), dim3(256), 0, s, S, n_ctx, rows, rmax, rsum, scores,
             (Acc*)nullptr, 1, 1, (Acc)0);
  QCF_LAUNCH_CHECK("qcf_score colmean");
  return QCF_OK;
}

// Received attention (KVShare, fusion.py:388-392 with the layer-1 pass of
// 352-373): out[n] = mean over (h, rows) of softmax_n(q[t,h].k[n] * scale) with
// key n visible to row t iff n <= row_pos[t]. Rows are processed in chunks
// that fit the workspace; column sums accumulate in Acc across chunks.
template <typename T, typename Acc>
static int received_impl(const void* q, const void* k, int64_t n_keys, int n_rows, int h, int hkv, int d,
                         double scale, const int32_t* row_pos, float* out, void* ws, size_t ws_bytes,
                         cudaStream_t s) {
  const size_t per_row = sizeof(Acc) * ((size_t)h * n_keys + 2 * (size_t)h);
  const size_t fixed = sizeof(Acc) * (size_t)n_keys + 256;
  QCF_REQUIRE(ws_bytes >= fixed + per_row, QCF_EWORKSPACE, "qcf_received_attention: workspace too small");
  const int chunk = (int)std::min<size_t>((size_t)n_rows, (ws_bytes - fixed) / per_row);
  Acc* colacc = reinterpret_cast<Acc*>(ws);
  Acc* S = colacc + n_keys;
  const size_t smem = sizeof(Acc) * (size_t)d * (SC_TQ + SC_TILE);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(score_logits_kernel<T, Acc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "qcf_received_attention attr");
  }
  QCF_REQUIRE(smem <= 220 * 1024, QCF_EUNSUPPORTED, "qcf_received_attention: head dim too large");
  const size_t esz = sizeof(T);
  for (int r0 = 0; r0 < n_rows; r0 += chunk) {
    const int nr = std::min(chunk, n_rows - r0);
    const int rows = h * nr;
    Acc* rmax = S + (int64_t)rows * n_keys;
    Acc* rsum = rmax + rows;
    const void* qc = reinterpret_cast<const uint8_t*>(q) + (size_t)r0 * h * d * esz;
    dim3 g1(ceil_div(n_keys, SC_TILE), h, ceil_div(nr, SC_TQ));
    QCF_LAUNCH("score_logits_kernel", score_logits_kernel<T, Acc>, dim3(g1), dim3(128), smem, s, (const T*)qc,
               (const T*)k, n_keys, nr, 0, h, hkv, d, (Acc)scale, S, row_pos + r0);
    QCF_LAUNCH_CHECK("qcf_received_attention logits");
    QCF_LAUNCH("score_rowstats_kernel", score_rowstats_kernel<Acc>, dim3(rows), dim3(256), 0, s, S, n_keys, rmax, rsum);
    QCF_LAUNCH_CHECK("qcf_received_attention rowstats");
    QCF_LAUNCH("score_colmean_kernel", score_colmean_kernel<Acc>, dim3(ceil_div(n_keys, 32)), dim3(256), 0, s, S,
               n_keys, rows, rmax, rsum, out, colacc, r0 == 0 ? 1 : 0, r0 + nr >= n_rows ? 1 : 0,
               (Acc)(1.0 / ((double)h * n_rows)));
    QCF_LAUNCH_CHECK("qcf_received_attention colmean");
  }
  return QCF_OK;
}

}  // namespace qcf

namespace qcf {
size_t score_tc_workspace(int64_t n_ctx, int nq, int h, int hkv, int n_req);
int score_tc_launch(const void* q, const void* k, int64_t k_req_stride, int64_t n_ctx, int nq, int n_req, int h,
                    int hkv, int d, double scale, int agg_last, float* scores, void* ws, size_t ws_bytes,
                    cudaStream_t s);
bool tc_available();
}  // namespace qcf

extern "C" size_t qcf_score_workspace(int64_t n_ctx, int nq, int h) {
  const size_t rows = (size_t)h * nq;
  return sizeof(double) * (rows * (size_t)n_ctx + 2 * rows) + 256;
}

extern "C" size_t qcf_score_batched_workspace(int64_t n_ctx, int nq, int n_req, int h, int hkv) {
  return std::max(qcf_score_workspace(n_ctx, nq, h), qcf::score_tc_workspace(n_ctx, nq, h, hkv, n_req));
}

extern "C" int qcf_score_batched(int dtype, const void* q, const void* k, int64_t k_req_stride, int64_t n_ctx,
                                 int nq, int n_req, int h, int hkv, int d, double scale, int agg_last, int precise,
                                 float* scores, void* workspace, size_t ws_bytes, qcf_stream_t stream) {
  QCF_REQUIRE(q && k && scores && workspace, QCF_EINVAL, "qcf_score: null pointer");
  QCF_REQUIRE(n_ctx > 0 && nq > 0 && n_req > 0 && h > 0 && hkv > 0 && h % hkv == 0 && d > 0, QCF_EINVAL,
              "qcf_score: bad sizes");
  QCF_REQUIRE(dtype == QCF_F32 || dtype == QCF_BF16, QCF_EINVAL, "qcf_score: bad dtype");
  auto s = qcf::as_stream(stream);
  if (dtype == QCF_BF16 && !precise && qcf::tc_available()) {
    // tensor-core speed mode (score_tc.cu); shapes it does not cover use the SIMT kernels
    const int st = qcf::score_tc_launch(q, k, k_req_stride, n_ctx, nq, n_req, h, hkv, d, scale, agg_last, scores,
                                        workspace, ws_bytes, s);
    if (st != QCF_EUNSUPPORTED) return st;
  }
  QCF_REQUIRE(ws_bytes >= qcf_score_workspace(n_ctx, nq, h), QCF_EWORKSPACE, "qcf_score: workspace too small");
  const size_t esz = dtype == QCF_F32 ? 4 : 2;
  for (int r = 0; r < n_req; ++r) {
    const void* qr = reinterpret_cast<const uint8_t*>(q) + (size_t)r * nq * h * d * esz;
    const void* kr = reinterpret_cast<const uint8_t*>(k) + (size_t)r * k_req_stride * esz;
    float* sr = scores + (int64_t)r * n_ctx;
    int st;
    if (dtype == QCF_F32)
      st = precise ? qcf::score_impl<float, double>(qr, kr, n_ctx, nq, h, hkv, d, scale, agg_last, sr, workspace, s)
                   : qcf::score_impl<float, float>(qr, kr, n_ctx, nq, h, hkv, d, scale, agg_last, sr, workspace, s);
    else
      st = precise ? qcf::score_impl<__nv_bfloat16, double>(qr, kr, n_ctx, nq, h, hkv, d, scale, agg_last, sr,
                                                            workspace, s)
                   : qcf::score_impl<__nv_bfloat16, float>(qr, kr, n_ctx, nq, h, hkv, d, scale, agg_last, sr,
                                                           workspace, s);
    if (st != QCF_OK) return st;
  }
  return QCF_OK;
}

extern "C" int qcf_score(int dtype, const void* q, const void* k, int64_t n_ctx, int nq, int h,
                         int hkv, int d, double scale, int agg_last, int precise, float* scores,
                         void* workspace, size_t ws_bytes, qcf_stream_t stream) {
  return qcf_score_batched(dtype, q, k, n_ctx * hkv * d, n_ctx, nq, 1, h, hkv, d, scale, agg_last, precise, scores,
                           workspace, ws_bytes, stream);
}

extern "C" int qcf_received_attention(int dtype, const void* q, const void* k, int64_t n_keys, int n_rows, int h,
                                      int hkv, int d, double scale, const int32_t* row_pos, float* out,
                                      void* workspace, size_t ws_bytes, qcf_stream_t stream) {
  QCF_REQUIRE(q && k && row_pos && out && workspace, QCF_EINVAL, "qcf_received_attention: null pointer");
  QCF_REQUIRE(n_keys > 0 && n_rows > 0 && h > 0 && hkv > 0 && h % hkv == 0 && d > 0, QCF_EINVAL,
              "qcf_received_attention: bad sizes");
  auto s = qcf::as_stream(stream);
  if (dtype == QCF_F32)
    return qcf::received_impl<float, double>(q, k, n_keys, n_rows, h, hkv, d, scale, row_pos, out, workspace,
                                             ws_bytes, s);
  if (dtype == QCF_BF16)
    return qcf::received_impl<__nv_bfloat16, double>(q, k, n_keys, n_rows, h, hkv, d, scale, row_pos, out,
                                                     workspace, ws_bytes, s);
  QCF_REQUIRE(false, QCF_EINVAL, "qcf_received_attention: bad dtype");
}
