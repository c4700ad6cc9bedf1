// Row-wise ops of the decoder layer: embedding gather (fusion.py:464,
// model.py:350), LayerNorm (model.py:305-308), the tied lm-head on the last
// query row (model.py:384-385 / fusion.py:540), and chunk key norms
// (store.py:339-340). One warp per row; statistics accumulate in float64 so the
// float32 residual stream matches numpy's pairwise float32 sums to ~1 ulp.
#include "common.cuh"

namespace qcf {

__global__ void embed_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ rows,
                             int32_t row_base, int64_t m, const float* __restrict__ emb, int d,
                             float* __restrict__ x) {
  const int64_t i = blockIdx.x;
  if (i >= m) return;
  const int tok = rows ? tokens[rows[i] - row_base] : tokens[i];
  const float* src = emb + (int64_t)tok * d;
  float* dst = x + i * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) dst[e] = src[e];
}

__device__ __forceinline__ void row_stats(const float* __restrict__ xr, int d, int lane,
                                          double& mean, double& rstd_var) {
  double s = 0.0;
  for (int e = lane; e < d; e += 32) s += (double)xr[e];
  s = warp_sum(s);
  mean = s / d;
  double v = 0.0;
  for (int e = lane; e < d; e += 32) {
    double t = (double)xr[e] - mean;
    v += t * t;
  }
  rstd_var = warp_sum(v) / d;
}

// One CTA (128 threads) per row; the row stays in registers between the mean
// and variance passes (d <= 128 * LN_VPT), block reductions in fp32.
constexpr int LN_THREADS = 128, LN_VPT = 64;

__device__ __forceinline__ float block_sum_128(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = red[0] + red[1] + red[2] + red[3];
  __syncthreads();
  return t;
}

template <typename T>
__global__ void __launch_bounds__(LN_THREADS) layernorm_kernel(const float* __restrict__ x, int64_t m, int d,
                                                               const float* __restrict__ g,
                                                               const float* __restrict__ b, float eps,
                                                               T* __restrict__ out) {
  __shared__ float red[4];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * d;
  float v[LN_VPT];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int e = threadIdx.x + i * LN_THREADS;
    v[i] = e < d ? xr[e] : 0.f;
    s += v[i];
  }
  const float mean = block_sum_128(s, red) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int e = threadIdx.x + i * LN_THREADS;
    const float t = v[i] - mean;
    q += e < d ? t * t : 0.f;
  }
  const float var = block_sum_128(q, red) / d;
  const float sd = sqrtf(var + eps);  // numpy: (x - mean) / sqrt(var + eps) * g + b  (model.py:308)
  T* orow = out + row * d;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int e = threadIdx.x + i * LN_THREADS;
    if (e < d) orow[e] = from_f<T>(((v[i] - mean) / sd) * g[e] + b[e]);
  }
}

// One block per output row: LN_f into shared memory, then one warp per vocab id.
__global__ void lm_head_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows, int d,
                               const float* __restrict__ g, const float* __restrict__ b, float eps,
                               const float* __restrict__ emb, int vocab, float* __restrict__ logits) {
  extern __shared__ float xs[];
  __shared__ float stat[2];
  const int r = blockIdx.x;
  const float* xr = x + (int64_t)(rows ? rows[r] : r) * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (warp == 0) {
    double mean, var;
    row_stats(xr, d, lane, mean, var);
    if (lane == 0) { stat[0] = (float)mean; stat[1] = sqrtf((float)var + eps); }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d; e += blockDim.x) xs[e] = ((xr[e] - stat[0]) / stat[1]) * g[e] + b[e];
  __syncthreads();
  for (int v = warp; v < vocab; v += nw) {
    const float* er = emb + (int64_t)v * d;
    float acc = 0.f;
    for (int e = lane; e < d; e += 32) acc = fmaf(xs[e], er[e], acc);
    acc = warp_sum(acc);
    if (lane == 0) logits[(int64_t)r * vocab + v] = acc;
  }
}

template <typename T>
__global__ void key_norms_kernel(const T* __restrict__ k, int64_t n, int hkv, int d,
                                 float* __restrict__ norms) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (row >= n) return;
  double acc = 0.0;
  for (int h = 0; h < hkv; ++h) {
    const T* kr = k + (row * hkv + h) * d;
    double s = 0.0;
    for (int e = lane; e < d; e += 32) {
      double t = (double)to_f<T>(kr[e]);
      s += t * t;
    }
    s = warp_sum(s);
    acc += sqrt(s);
  }
  if (lane == 0) norms[row] = (float)(acc / hkv);
}

}  // namespace qcf

extern "C" {

int qcf_embed(const int32_t* tokens, const int32_t* rows, int32_t row_base, int64_t m,
              const float* emb, int d, float* x, qcf_stream_t stream) {
  QCF_REQUIRE(tokens && emb && x && d > 0 && m >= 0, QCF_EINVAL, "qcf_embed: bad args");
  if (m == 0) return QCF_OK;
  QCF_REQUIRE(m <= 0x7fffffff, QCF_EUNSUPPORTED, "qcf_embed: too many rows");
  qcf::embed_kernel<<<(unsigned)m, 256, 0, qcf::as_stream(stream)>>>(tokens, rows, row_base, m, emb, d, x);
  QCF_LAUNCH_CHECK("qcf_embed");
  return QCF_OK;
}

int qcf_layernorm(const float* x, int64_t m, int d, const float* g, const float* b, float eps,
                  void* out, int out_dtype, qcf_stream_t stream) {
  QCF_REQUIRE(x && g && b && out && d > 0 && m >= 0, QCF_EINVAL, "qcf_layernorm: bad args");
  if (m == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  QCF_REQUIRE(d <= qcf::LN_THREADS * qcf::LN_VPT, QCF_EUNSUPPORTED, "qcf_layernorm: d_model > %d",
              qcf::LN_THREADS * qcf::LN_VPT);
  QCF_REQUIRE(m <= 0x7fffffff, QCF_EUNSUPPORTED, "qcf_layernorm: too many rows");
  unsigned grid = (unsigned)m;
  if (out_dtype == QCF_F32)
    qcf::layernorm_kernel<float><<<grid, qcf::LN_THREADS, 0, s>>>(x, m, d, g, b, eps, (float*)out);
  else if (out_dtype == QCF_BF16)
    qcf::layernorm_kernel<__nv_bfloat16><<<grid, qcf::LN_THREADS, 0, s>>>(x, m, d, g, b, eps, (__nv_bfloat16*)out);
  else
    QCF_REQUIRE(false, QCF_EINVAL, "qcf_layernorm: bad dtype");
  QCF_LAUNCH_CHECK("qcf_layernorm");
  return QCF_OK;
}

int qcf_lm_head(const float* x, const int32_t* rows, int64_t n_rows, int d, const float* g,
                const float* b, float eps, const float* emb, int vocab, float* logits,
                qcf_stream_t stream) {
  QCF_REQUIRE(x && g && b && emb && logits && d > 0 && vocab > 0, QCF_EINVAL, "qcf_lm_head: bad args");
  QCF_REQUIRE(d * 4 <= 200 * 1024, QCF_EUNSUPPORTED, "qcf_lm_head: d_model too large");
  if (n_rows == 0) return QCF_OK;
  const size_t smem = (size_t)d * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(qcf::lm_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return qcf::cuda_status(e, "qcf_lm_head attr");
  }
  qcf::lm_head_kernel<<<(unsigned)n_rows, 512, smem, qcf::as_stream(stream)>>>(x, rows, d, g, b, eps, emb, vocab, logits);
  QCF_LAUNCH_CHECK("qcf_lm_head");
  return QCF_OK;
}

int qcf_key_norms(const void* k, int64_t n, int hkv, int d, float* norms, int dtype,
                  qcf_stream_t stream) {
  QCF_REQUIRE(k && norms && hkv > 0 && d > 0, QCF_EINVAL, "qcf_key_norms: bad args");
  if (n == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  unsigned grid = (unsigned)((n + 7) / 8);
  if (dtype == QCF_F32)
    qcf::key_norms_kernel<float><<<grid, 256, 0, s>>>((const float*)k, n, hkv, d, norms);
  else
    qcf::key_norms_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)k, n, hkv, d, norms);
  QCF_LAUNCH_CHECK("qcf_key_norms");
  return QCF_OK;
}

}  // extern "C"
