// Comparison-policy kernels: the layer-1 KV deviation that
// ranks tokens for CacheBlend and KVShare (fusion.py:375-380):
//   dev[n] = sum_h ||k_new[n,h] - k_old[n,h]||_2 + sum_h ||v_new[n,h] - v_old[n,h]||_2
// with float64 norms (the reference casts the difference to float64), cast to f32.
// One warp per row; lanes stride the head dim.
#include "common.cuh"

namespace qcf {

template <typename T>
__global__ void kv_deviation_kernel(const T* __restrict__ ok, const T* __restrict__ ov, const T* __restrict__ nk,
                                    const T* __restrict__ nv, int64_t n, int hkv, int d, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (row >= n) return;
  double acc = 0.0;
  for (int which = 0; which < 2; ++which) {
    const T* a = which ? ov : ok;
    const T* b = which ? nv : nk;
    for (int h = 0; h < hkv; ++h) {
      const int64_t base = (row * hkv + h) * d;
      double s = 0.0;
      for (int e = lane; e < d; e += 32) {
        // float32 difference first (numpy: (new - old).astype(float64))
        const double t = (double)(to_f<T>(b[base + e]) - to_f<T>(a[base + e]));
        s += t * t;
      }
      s = warp_sum(s);
      acc += sqrt(s);
    }
  }
  if (lane == 0) out[row] = (float)acc;
}

}  // namespace qcf

extern "C" int qcf_kv_deviation(int dtype, const void* old_k, const void* old_v, const void* new_k, const void* new_v,
                                int64_t n, int hkv, int d, float* out, qcf_stream_t stream) {
  QCF_REQUIRE(old_k && old_v && new_k && new_v && out && hkv > 0 && d > 0 && n >= 0, QCF_EINVAL,
              "qcf_kv_deviation: bad args");
  if (n == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  const unsigned grid = (unsigned)((n + 7) / 8);
  if (dtype == QCF_F32)
    QCF_LAUNCH("kv_deviation_kernel", qcf::kv_deviation_kernel<float>, dim3(grid), dim3(256), 0, s,
               (const float*)old_k, (const float*)old_v, (const float*)new_k, (const float*)new_v, n, hkv, d, out);
  else if (dtype == QCF_BF16)
    QCF_LAUNCH("kv_deviation_kernel", qcf::kv_deviation_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s,
               (const __nv_bfloat16*)old_k, (const __nv_bfloat16*)old_v, (const __nv_bfloat16*)new_k,
               (const __nv_bfloat16*)new_v, n, hkv, d, out);
  else
    QCF_REQUIRE(false, QCF_EINVAL, "qcf_kv_deviation: bad dtype");
  QCF_LAUNCH_CHECK("qcf_kv_deviation");
  return QCF_OK;
}
