// Row-wise ops of the decoder layer: embedding gather (fusion.py:464,
// model.py:350), LayerNorm (model.py:305-308), the tied lm-head on the last
// query row (model.py:384-385 / fusion.py:540), and chunk key norms
// (store.py:339-340). LayerNorm keeps a row in registers (one CTA per row) and
// reduces in fp32; key norms accumulate in float64.
#include "common.cuh"

namespace qcf {

__global__ void embed_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ rows,
                             int32_t row_base, int64_t m, const float* __restrict__ emb, int d,
                             float* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x;
  if (i >= m) return;
  const int tok = rows ? tokens[rows[i] - row_base] : tokens[i];
  const float* src = emb + (int64_t)tok * d;
  float* dst = x + i * d;
  if ((d & 3) == 0 && !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)) {
    for (int e = threadIdx.x; e < (d >> 2); e += blockDim.x)
      reinterpret_cast<float4*>(dst)[e] = __ldg(reinterpret_cast<const float4*>(src) + e);
  } else {
    for (int e = threadIdx.x; e < d; e += blockDim.x) dst[e] = src[e];
  }
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

// One CTA (256 threads) per row. All loads (x, gain, bias) are issued up front
// as float4 into registers, so the kernel pays ~2 memory round trips; fp32
// block reductions for mean and (x-mean)^2.
constexpr int LN_THREADS = 256, LN_V4 = 8;  // d <= 256 * 4 * 8 = 8192

// block_sum_256 of R values at once (each value reduced exactly as block_sum_256 does)
template <int R>
__device__ __forceinline__ void block_sum_256_rows(float (&v)[R], float (*red)[LN_THREADS / 32]) {
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = warp_sum(v[q]);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < R; ++q) red[q][w] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < R; ++q) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < LN_THREADS / 32; ++i) t += red[q][i];
    v[q] = t;
  }
  __syncthreads();
}

__device__ __forceinline__ float block_sum_256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < LN_THREADS / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

template <typename T>
__device__ __forceinline__ void store4(T* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 u = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  *reinterpret_cast<uint2*>(p) = u;
}

// With `delta` != null the residual update x += delta (the projection output,
// model.py:375-376) is applied first and written back, fusing the residual add
// that would otherwise be a read-modify-write in the GEMM epilogue.
// V float4 per thread (d = 4*V*256 at most): x and delta are loaded up front,
// gain/bias only at the store (L1/L2 resident), so registers stay low and
// several rows per SM keep their loads in flight (the kernel is HBM-bound:
// 4+4 B read, 4+2 B written per element).
template <typename T, int V, int R>
__global__ void __launch_bounds__(LN_THREADS) layernorm_kernel(float* __restrict__ x, const float* __restrict__ delta,
                                                               int64_t m, int d, const float* __restrict__ g,
                                                               const float* __restrict__ b, float eps,
                                                               T* __restrict__ out) {
  // R rows per CTA: all R rows' loads are in flight together and the two block
  // reductions are shared by the R rows (per-row arithmetic unchanged)
  pdl_wait();
  pdl_trigger();
  __shared__ float red[R][LN_THREADS / 32];
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  const int n4 = d >> 2;
  float4 v[R][V], t[R][V];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int64_t row = (int64_t)blockIdx.x * R + q;
    const bool ok = row < m;
    const float4* xr = reinterpret_cast<const float4*>(x + row * d);
    const float4* dr = delta ? reinterpret_cast<const float4*>(delta + row * d) : nullptr;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int e = threadIdx.x + i * LN_THREADS;
      v[q][i] = (ok && e < n4) ? xr[e] : make_float4(0.f, 0.f, 0.f, 0.f);
      t[q][i] = (ok && dr && e < n4) ? __ldcs(dr + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  float s[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int64_t row = (int64_t)blockIdx.x * R + q;
    if (delta) {
      float4* xr = reinterpret_cast<float4*>(x + row * d);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int e = threadIdx.x + i * LN_THREADS;
        v[q][i].x += t[q][i].x; v[q][i].y += t[q][i].y; v[q][i].z += t[q][i].z; v[q][i].w += t[q][i].w;
        if (row < m && e < n4) xr[e] = v[q][i];
      }
    }
    s[q] = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) s[q] += (v[q][i].x + v[q][i].y) + (v[q][i].z + v[q][i].w);
  }
  float mean[R];
  block_sum_256_rows<R>(s, red);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    mean[q] = s[q] / d;
    float qs = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      if (threadIdx.x + i * LN_THREADS < n4) {
        const float a0 = v[q][i].x - mean[q], a1 = v[q][i].y - mean[q], a2 = v[q][i].z - mean[q],
                    a3 = v[q][i].w - mean[q];
        qs += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
      }
    }
    s[q] = qs;
  }
  block_sum_256_rows<R>(s, red);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int64_t row = (int64_t)blockIdx.x * R + q;
    if (row >= m) break;
    const float var = s[q] / d;
    const float sd = sqrtf(var + eps);  // numpy: (x - mean) / sqrt(var + eps) * g + b  (model.py:308)
    T* orow = out + row * d;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int e = threadIdx.x + i * LN_THREADS;
      if (e < n4) {
        const float4 gv = g4[e], bv = b4[e];
        const float mu = mean[q];
        store4<T>(orow + 4 * e, ((v[q][i].x - mu) / sd) * gv.x + bv.x, ((v[q][i].y - mu) / sd) * gv.y + bv.y,
                  ((v[q][i].z - mu) / sd) * gv.z + bv.z, ((v[q][i].w - mu) / sd) * gv.w + bv.w);
      }
    }
  }
}

// rows per CTA: 2 for one request's ~800 rows (18.4 -> 14.5 us), 1 for the probe's
// 32 / 256 rows (256: 10.2 vs 12.3 us) and the batch's 6400 (63.5 vs 65.6 us); 4 rows
// per CTA was slower everywhere (tools/ln_bench.py). QCF_LN_ROWS=1/2 forces it.
static int g_ln_rows = -1;
template <typename T, int R>
static int launch_ln_rows(float* x, const float* delta, int64_t m, int d, const float* g, const float* b, float eps,
                          T* out, cudaStream_t s) {
  const int n4 = d / 4;
  const unsigned grid = (unsigned)((m + R - 1) / R);
  if (n4 <= LN_THREADS)
    QCF_LAUNCH("layernorm_kernel", (layernorm_kernel<T, 1, R>), dim3(grid), dim3(LN_THREADS), 0, s, x, delta, m, d, g, b, eps, out);
  else if (n4 <= 2 * LN_THREADS)
    QCF_LAUNCH("layernorm_kernel", (layernorm_kernel<T, 2, R>), dim3(grid), dim3(LN_THREADS), 0, s, x, delta, m, d, g, b, eps, out);
  else if (n4 <= 4 * LN_THREADS)
    QCF_LAUNCH("layernorm_kernel", (layernorm_kernel<T, 4, R>), dim3(grid), dim3(LN_THREADS), 0, s, x, delta, m, d, g, b, eps, out);
  else
    QCF_LAUNCH("layernorm_kernel", (layernorm_kernel<T, LN_V4, 1>), dim3((unsigned)m), dim3(LN_THREADS), 0, s, x, delta, m, d, g, b, eps, out);
  return QCF_OK;
}
template <typename T>
static int launch_ln_vec(float* x, const float* delta, int64_t m, int d, const float* g, const float* b, float eps,
                         T* out, cudaStream_t s) {
  if (g_ln_rows < 0) {
    const char* e = getenv("QCF_LN_ROWS");
    g_ln_rows = e ? ((atoi(e) == 2) ? 2 : 1) : 0;  // 0 = by row count
  }
  const bool two = g_ln_rows == 2 || (g_ln_rows == 0 && m >= 512 && m <= 2048);
  if (two && d / 4 <= 4 * LN_THREADS) return launch_ln_rows<T, 2>(x, delta, m, d, g, b, eps, out, s);
  return launch_ln_rows<T, 1>(x, delta, m, d, g, b, eps, out, s);
}

// generic fallback (d % 4 != 0): one CTA per row, strided scalar loop
template <typename T>
__global__ void __launch_bounds__(LN_THREADS) layernorm_scalar_kernel(float* __restrict__ x,
                                                                      const float* __restrict__ delta, int64_t m,
                                                                      int d, const float* __restrict__ g,
                                                                      const float* __restrict__ b, float eps,
                                                                      T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[LN_THREADS / 32];
  float* xr = x + (int64_t)blockIdx.x * d;
  if (delta) {
    const float* dr = delta + (int64_t)blockIdx.x * d;
    for (int e = threadIdx.x; e < d; e += LN_THREADS) xr[e] = xr[e] + dr[e];
    __syncthreads();
  }
  float s = 0.f;
  for (int e = threadIdx.x; e < d; e += LN_THREADS) s += xr[e];
  const float mean = block_sum_256(s, red) / d;
  float q = 0.f;
  for (int e = threadIdx.x; e < d; e += LN_THREADS) { const float t = xr[e] - mean; q += t * t; }
  const float sd = sqrtf(block_sum_256(q, red) / d + eps);
  T* orow = out + (int64_t)blockIdx.x * d;
  for (int e = threadIdx.x; e < d; e += LN_THREADS) orow[e] = from_f<T>(((xr[e] - mean) / sd) * g[e] + b[e]);
}

__global__ void add_rows_kernel(float* __restrict__ x, const float* __restrict__ delta, int64_t n4) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(x)[i];
    const float4 t = reinterpret_cast<const float4*>(delta)[i];
    a.x += t.x; a.y += t.y; a.z += t.z; a.w += t.w;
    reinterpret_cast<float4*>(x)[i] = a;
  }
}

// lm-head: grid (vocab tiles of LM_VT, rows). Every CTA recomputes LN_f of its
// row into shared memory (d floats), then each warp dots one vocab row at a
// time with float4 loads, LM_UNROLL of them in flight per lane.
constexpr int LM_THREADS = 256, LM_VT = 16, LM_UNROLL = 8;

template <bool VEC>
__global__ void __launch_bounds__(LM_THREADS) lm_head_kernel(const float* __restrict__ x,
                                                             const int32_t* __restrict__ rows, int d,
                                                             const float* __restrict__ g,
                                                             const float* __restrict__ b, float eps,
                                                             const float* __restrict__ emb, int vocab,
                                                             float* __restrict__ logits) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float xs[];
  __shared__ float red[8];
  const int r = blockIdx.y;
  const float* xr = x + (int64_t)(rows ? rows[r] : r) * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float s = 0.f;
  for (int e = threadIdx.x; e < d; e += LM_THREADS) { const float v = xr[e]; xs[e] = v; s += v; }
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  float mean = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) mean += red[w];
  mean /= d;
  __syncthreads();
  float q = 0.f;
  for (int e = threadIdx.x; e < d; e += LM_THREADS) { const float t = xs[e] - mean; q += t * t; }
  q = warp_sum(q);
  if (lane == 0) red[warp] = q;
  __syncthreads();
  float var = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) var += red[w];
  const float sd = sqrtf(var / d + eps);
  for (int e = threadIdx.x; e < d; e += LM_THREADS) xs[e] = ((xs[e] - mean) / sd) * g[e] + b[e];
  __syncthreads();
  const int d4 = d >> 2;
  for (int vv = warp; vv < LM_VT; vv += 8) {
    const int v = blockIdx.x * LM_VT + vv;
    if (v >= vocab) break;
    float acc = 0.f;
    if (!VEC) {  // d % 4 != 0 (toy widths): scalar dot
      const float* er = emb + (int64_t)v * d;
      for (int e = lane; e < d; e += 32) acc = fmaf(xs[e], er[e], acc);
      acc = warp_sum(acc);
      if (lane == 0) logits[(int64_t)r * vocab + v] = acc;
      continue;
    }
    const float4* er = reinterpret_cast<const float4*>(emb + (int64_t)v * d);
    const float4* xs4 = reinterpret_cast<const float4*>(xs);
    for (int e0 = lane; e0 < d4; e0 += 32 * LM_UNROLL) {
      float4 w[LM_UNROLL];
#pragma unroll
      for (int u = 0; u < LM_UNROLL; ++u) {
        const int e = e0 + u * 32;
        w[u] = e < d4 ? __ldg(er + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < LM_UNROLL; ++u) {
        const int e = e0 + u * 32;
        if (e < d4) {
          const float4 xv = xs4[e];
          acc = fmaf(xv.x, w[u].x, acc);
          acc = fmaf(xv.y, w[u].y, acc);
          acc = fmaf(xv.z, w[u].z, acc);
          acc = fmaf(xv.w, w[u].w, acc);
        }
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) logits[(int64_t)r * vocab + v] = acc;
  }
}

template <typename T>
__global__ void key_norms_kernel(const T* __restrict__ k, int64_t n, int hkv, int d,
                                 float* __restrict__ norms) {
  pdl_wait();
  pdl_trigger();
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

// greedy decode step on the device (model.py:433-465): next = argmax(logits) with
// numpy's tie rule (lowest index among equal maxima), appended to log[*step];
// tok <- next, pos += 1, step += 1 -- so a CUDA graph of one decode step can be
// replayed max_new times without a host round trip per token
__global__ void __launch_bounds__(256) decode_advance_kernel(const float* __restrict__ logits, int vocab,
                                                             int32_t* __restrict__ tok, int32_t* __restrict__ pos,
                                                             int32_t* __restrict__ step,
                                                             int32_t* __restrict__ log_tokens, int log_cap) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[8];
  __shared__ int si[8];
  float best = -INFINITY;
  int bi = vocab;  // no valid index yet
  for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
    const float v = logits[i];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[warp] = best; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    if (bi >= vocab) bi = 0;  // all NaN: np.argmax would return the first NaN's index; 0 is the stand-in
    const int st = *step;
    if (st < log_cap) log_tokens[st] = bi;
    *tok = bi;
    *pos += 1;
    *step = st + 1;
  }
}

}  // namespace qcf

extern "C" {

int qcf_embed(const int32_t* tokens, const int32_t* rows, int32_t row_base, int64_t m,
              const float* emb, int d, float* x, qcf_stream_t stream) {
  QCF_REQUIRE(tokens && emb && x && d > 0 && m >= 0, QCF_EINVAL, "qcf_embed: bad args");
  if (m == 0) return QCF_OK;
  QCF_REQUIRE(m <= 0x7fffffff, QCF_EUNSUPPORTED, "qcf_embed: too many rows");
  QCF_LAUNCH("embed_kernel", qcf::embed_kernel, dim3((unsigned)m), dim3(256), 0, qcf::as_stream(stream), tokens, rows, row_base, m, emb, d, x);
  QCF_LAUNCH_CHECK("qcf_embed");
  return QCF_OK;
}

int qcf_add_layernorm(float* x, const float* delta, int64_t m, int d, const float* g, const float* b,
                      float eps, void* out, int out_dtype, qcf_stream_t stream);

int qcf_layernorm(const float* x, int64_t m, int d, const float* g, const float* b, float eps,
                  void* out, int out_dtype, qcf_stream_t stream) {
  return qcf_add_layernorm(const_cast<float*>(x), nullptr, m, d, g, b, eps, out, out_dtype, stream);
}

int qcf_add_rows(float* x, const float* delta, int64_t n, qcf_stream_t stream) {
  QCF_REQUIRE(x && delta && n >= 0 && n % 4 == 0, QCF_EINVAL, "qcf_add_rows: bad args");
  QCF_REQUIRE(!(((uintptr_t)x | (uintptr_t)delta) & 15), QCF_EINVAL, "qcf_add_rows: 16-byte alignment");
  if (n == 0) return QCF_OK;
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
  QCF_LAUNCH("add_rows_kernel", qcf::add_rows_kernel, dim3(grid), dim3(256), 0, qcf::as_stream(stream), x, delta, n4);
  QCF_LAUNCH_CHECK("qcf_add_rows");
  return QCF_OK;
}

int qcf_add_layernorm(float* x, const float* delta, int64_t m, int d, const float* g, const float* b,
                      float eps, void* out, int out_dtype, qcf_stream_t stream) {
  QCF_REQUIRE(x && g && b && out && d > 0 && m >= 0, QCF_EINVAL, "qcf_layernorm: bad args");
  if (m == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  QCF_REQUIRE(m <= 0x7fffffff, QCF_EUNSUPPORTED, "qcf_layernorm: too many rows");
  const unsigned grid = (unsigned)m;
  const bool vec = (d % 4 == 0) && d <= qcf::LN_THREADS * 4 * qcf::LN_V4 &&
                   !(((uintptr_t)x | (uintptr_t)g | (uintptr_t)b | (uintptr_t)out | (uintptr_t)delta) & 15) &&
                   (out_dtype == QCF_F32 || d % 8 == 0);
  if (out_dtype == QCF_F32) {
    if (vec) {
      const int st = qcf::launch_ln_vec<float>(x, delta, m, d, g, b, eps, (float*)out, s);
      if (st != QCF_OK) return st;
    } else QCF_LAUNCH("layernorm_scalar_kernel", qcf::layernorm_scalar_kernel<float>, dim3(grid), dim3(qcf::LN_THREADS), 0, s, x, delta, m, d, g, b, eps, (float*)out);
  } else if (out_dtype == QCF_BF16) {
    if (vec) {
      const int st = qcf::launch_ln_vec<__nv_bfloat16>(x, delta, m, d, g, b, eps, (__nv_bfloat16*)out, s);
      if (st != QCF_OK) return st;
    } else QCF_LAUNCH("layernorm_scalar_kernel", qcf::layernorm_scalar_kernel<__nv_bfloat16>, dim3(grid), dim3(qcf::LN_THREADS), 0, s, x, delta, m, d, g, b, eps, (__nv_bfloat16*)out);
  } else {
    QCF_REQUIRE(false, QCF_EINVAL, "qcf_layernorm: bad dtype");
  }
  QCF_LAUNCH_CHECK("qcf_layernorm");
  return QCF_OK;
}

int qcf_lm_head(const float* x, const int32_t* rows, int64_t n_rows, int d, const float* g,
                const float* b, float eps, const float* emb, int vocab, float* logits,
                qcf_stream_t stream) {
  QCF_REQUIRE(x && g && b && emb && logits && d > 0 && vocab > 0, QCF_EINVAL, "qcf_lm_head: bad args");
  QCF_REQUIRE(d * 4 <= 200 * 1024, QCF_EUNSUPPORTED, "qcf_lm_head: d_model too large");
  const bool vec = d % 4 == 0 && !(((uintptr_t)emb) & 15);
  if (n_rows == 0) return QCF_OK;
  const size_t smem = (size_t)d * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(qcf::lm_head_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(qcf::lm_head_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return qcf::cuda_status(e, "qcf_lm_head attr");
  }
  dim3 grid((unsigned)((vocab + qcf::LM_VT - 1) / qcf::LM_VT), (unsigned)n_rows);
  if (vec)
    QCF_LAUNCH("lm_head_kernel", qcf::lm_head_kernel<true>, dim3(grid), dim3(qcf::LM_THREADS), smem, qcf::as_stream(stream), x, rows, d, g, b, eps, emb, vocab, logits);
  else
    QCF_LAUNCH("lm_head_kernel", qcf::lm_head_kernel<false>, dim3(grid), dim3(qcf::LM_THREADS), smem, qcf::as_stream(stream), x, rows, d, g, b, eps, emb, vocab, logits);
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
    QCF_LAUNCH("key_norms_kernel", qcf::key_norms_kernel<float>, dim3(grid), dim3(256), 0, s, (const float*)k, n, hkv, d, norms);
  else
    QCF_LAUNCH("key_norms_kernel", qcf::key_norms_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, (const __nv_bfloat16*)k, n, hkv, d, norms);
  QCF_LAUNCH_CHECK("qcf_key_norms");
  return QCF_OK;
}

int qcf_decode_advance(const float* logits, int vocab, int32_t* tok, int32_t* pos, int32_t* step,
                       int32_t* log_tokens, int log_cap, qcf_stream_t stream) {
  QCF_REQUIRE(logits && tok && pos && step && vocab > 0 && log_cap >= 0, QCF_EINVAL, "qcf_decode_advance: bad args");
  QCF_LAUNCH("decode_advance_kernel", qcf::decode_advance_kernel, dim3(1), dim3(256), 0, qcf::as_stream(stream), logits,
             vocab, tok, pos, step, log_tokens, log_cap);
  QCF_LAUNCH_CHECK("qcf_decode_advance");
  return QCF_OK;
}

}  // extern "C"
