// Location-aware attention, SIMT flash form (parity path and cross-check):
// row i of the query tile sees table rows 0..kmax[i] (fusion.py:194-208 with
// the causal "key position <= row position" mask of fusion.py:467), scores
// divided by float32(sqrt(D)) and max-subtracted softmax as model.py:326-338.
// A CTA owns 32 query rows x one head; K/V tiles of 32 keys stream through
// shared memory and are reused by all 32 rows; online softmax in fp32.
// An optional bit mask [m][mask_words] (bit j of row i = key j visible) narrows
// the visible set further: the public sparse_attention's arbitrary `visible`
// masks (fusion.py:194-208, test_fusion.py:205-248).
#include <math.h>

#include "attention.cuh"
#include "common.cuh"

namespace qcf {

constexpr int AQ = 32, AK = 32;

template <typename T, int D>
__global__ void __launch_bounds__(128) attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                        const T* __restrict__ v,
                                                        const int32_t* __restrict__ kmax, int64_t m,
                                                        int h, int hkv, int64_t n_keys,
                                                        T* __restrict__ out,
                                                        const uint32_t* __restrict__ mask, int64_t mask_words) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];
  float* Qs = sm;                        // [AQ][D+1]
  float* Ks = Qs + AQ * (D + 1);         // [AK][D+1]
  float* Vs = Ks + AK * (D + 1);         // [AK][D]
  float* Ps = Vs + AK * D;               // [AQ][AK+1]
  __shared__ int kmax_s[AQ];
  __shared__ int kend_s;

  const int head = blockIdx.y, kvh = head / (h / hkv);
  const int64_t req = blockIdx.z;  // request: q/out/kmax [req][m], K/V [req][n_keys]
  q += req * m * h * D;
  out += req * m * h * D;
  kmax += req * m;
  k += req * n_keys * hkv * D;
  v += req * n_keys * hkv * D;
  const int64_t r0 = (int64_t)blockIdx.x * AQ;
  const int tid = threadIdx.x;
  const int row = tid >> 2, cg = tid & 3;       // 4 threads per query row
  constexpr int DC = (D + 3) / 4;                // output columns per thread
  const float inv_scale_div = sqrtf((float)D);

  if (tid < AQ) {
    int64_t r = r0 + tid;
    kmax_s[tid] = r < m ? min((int64_t)kmax[r], n_keys - 1) : -1;
  }
  for (int e = tid; e < AQ * D; e += blockDim.x) {
    int rr = e / D, c = e % D;
    int64_t r = r0 + rr;
    Qs[rr * (D + 1) + c] = r < m ? to_f<T>(q[(r * h + head) * D + c]) : 0.f;
  }
  __syncthreads();
  if (tid == 0) {
    int mx = -1;
    for (int i = 0; i < AQ; ++i) mx = max(mx, kmax_s[i]);
    kend_s = mx + 1;
  }
  __syncthreads();
  const int kend = kend_s;
  const int my_kmax = kmax_s[row];

  float o[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) o[c] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;

  for (int k0 = 0; k0 < kend; k0 += AK) {
    for (int e = tid; e < AK * D; e += blockDim.x) {
      int j = e / D, c = e % D;
      int64_t kr = k0 + j;
      float kv = 0.f, vv = 0.f;
      if (kr < kend) {
        kv = to_f<T>(k[(kr * hkv + kvh) * D + c]);
        vv = to_f<T>(v[(kr * hkv + kvh) * D + c]);
      }
      Ks[j * (D + 1) + c] = kv;
      Vs[j * D + c] = vv;
    }
    __syncthreads();
    // scores for this thread's 8 keys
    float s[AK / 4];
    float tmax = -INFINITY;
#pragma unroll
    for (int jj = 0; jj < AK / 4; ++jj) {
      const int j = cg * (AK / 4) + jj;
      float acc = 0.f;
#pragma unroll 8
      for (int c = 0; c < D; ++c) acc = fmaf(Qs[row * (D + 1) + c], Ks[j * (D + 1) + c], acc);
      acc = acc / inv_scale_div;
      if (k0 + j > my_kmax) acc = -INFINITY;
      if (mask != nullptr && r0 + row < m && k0 + j < n_keys &&
          !((mask[(req * m + r0 + row) * mask_words + ((k0 + j) >> 5)] >> ((k0 + j) & 31)) & 1u))
        acc = -INFINITY;
      s[jj] = acc;
      tmax = fmaxf(tmax, acc);
    }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float m_new = fmaxf(m_run, tmax);
    const float alpha = (m_run == -INFINITY) ? 0.f : expf(m_run - m_new);
    float psum = 0.f;
#pragma unroll
    for (int jj = 0; jj < AK / 4; ++jj) {
      float p = (s[jj] == -INFINITY) ? 0.f : expf(s[jj] - m_new);
      Ps[row * (AK + 1) + cg * (AK / 4) + jj] = p;
      psum += p;
    }
    psum += __shfl_xor_sync(0xffffffffu, psum, 1);
    psum += __shfl_xor_sync(0xffffffffu, psum, 2);
    l_run = l_run * alpha + psum;
    m_run = m_new;
    __syncwarp();
#pragma unroll
    for (int cc = 0; cc < DC; ++cc) {
      const int c = cg * DC + cc;
      float acc = o[cc] * alpha;
      if (c < D) {
#pragma unroll 8
        for (int j = 0; j < AK; ++j) acc = fmaf(Ps[row * (AK + 1) + j], Vs[j * D + c], acc);
      }
      o[cc] = acc;
    }
    __syncthreads();
  }
  const int64_t r = r0 + row;
  if (r < m) {
    const float inv = 1.f / l_run;
#pragma unroll
    for (int cc = 0; cc < DC; ++cc) {
      const int c = cg * DC + cc;
      if (c < D) out[(r * h + head) * D + c] = from_f<T>(o[cc] * inv);
    }
  }
}

template <typename T, int D>
static int launch_simt(const void* q, const void* k, const void* v, const int32_t* kmax, int64_t m,
                       int h, int hkv, int64_t n_keys, void* out, cudaStream_t s, int n_req,
                       const uint32_t* mask, int64_t mask_words) {
  const size_t smem = sizeof(float) * (AQ * (D + 1) + AK * (D + 1) + AK * D + AQ * (AK + 1));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(attn_simt_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "attn_simt attr");
  }
  dim3 grid(ceil_div(m, AQ), h, n_req);
  QCF_LAUNCH("attn_simt_kernel", attn_simt_kernel<T, D>, dim3(grid), dim3(128), smem, s, (const T*)q, (const T*)k, (const T*)v, kmax, m, h,
                                                 hkv, n_keys, (T*)out, mask, mask_words);
  QCF_LAUNCH_CHECK("qcf_attention(simt)");
  return QCF_OK;
}

template <typename T>
static int dispatch_d(int d, const void* q, const void* k, const void* v, const int32_t* kmax,
                      int64_t m, int h, int hkv, int64_t n_keys, void* out, cudaStream_t s, int n_req,
                      const uint32_t* mask, int64_t mw) {
  switch (d) {
    case 8: return launch_simt<T, 8>(q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mw);
    case 16: return launch_simt<T, 16>(q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mw);
    case 32: return launch_simt<T, 32>(q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mw);
    case 64: return launch_simt<T, 64>(q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mw);
    case 128: return launch_simt<T, 128>(q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mw);
    default: break;
  }
  set_error("qcf_attention: unsupported d_head %d (8/16/32/64/128)", d);
  return QCF_EUNSUPPORTED;
}

int attention_simt_launch(int dtype, const void* q, const void* k, const void* v,
                          const int32_t* kmax, int64_t m, int h, int hkv, int d, int64_t n_keys,
                          void* out, cudaStream_t s, int n_req, const uint32_t* mask, int64_t mask_words) {
  if (dtype == QCF_F32) return dispatch_d<float>(d, q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mask_words);
  return dispatch_d<__nv_bfloat16>(d, q, k, v, kmax, m, h, hkv, n_keys, out, s, n_req, mask, mask_words);
}

}  // namespace qcf

extern "C" int qcf_attention_masked(int dtype, const void* q, const void* k, const void* v, const int32_t* kmax,
                                    const uint32_t* mask, int64_t mask_words, int64_t m, int h, int hkv, int d,
                                    int64_t n_keys, void* out, qcf_stream_t stream) {
  QCF_REQUIRE(q && k && v && kmax && mask && out, QCF_EINVAL, "qcf_attention_masked: null pointer");
  QCF_REQUIRE(h > 0 && hkv > 0 && h % hkv == 0 && n_keys > 0 && m >= 0, QCF_EINVAL, "qcf_attention_masked: bad shape");
  QCF_REQUIRE(mask_words >= (n_keys + 31) / 32, QCF_ESHAPE, "qcf_attention_masked: mask rows too short");
  QCF_REQUIRE(dtype == QCF_F32 || dtype == QCF_BF16, QCF_EINVAL, "qcf_attention_masked: bad dtype");
  if (m == 0) return QCF_OK;
  return qcf::attention_simt_launch(dtype, q, k, v, kmax, m, h, hkv, d, n_keys, out, qcf::as_stream(stream), 1, mask,
                                    mask_words);
}
