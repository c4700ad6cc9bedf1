// RoPE at absolute positions for the freshly projected rows plus the in-place
// scatter of their K/V into the fused table (fusion.py:471-478: the new K/V
// replace rows `sel` before attention). Q/K pairs rotate with the float64
// cos/sin table; in parity mode (f32) the rotation itself runs in float64 with
// explicit rounding, reproducing model.py:282-286 bit for bit.
#include "common.cuh"

namespace qcf {

template <typename T, bool kExact>
__global__ void rope_qkv_scatter_kernel(const float* __restrict__ qkv, int64_t m, int h, int hkv,
                                        int d, const int32_t* __restrict__ pos,
                                        const int32_t* __restrict__ dst_rows,
                                        const double* __restrict__ ctab,
                                        const double* __restrict__ stab, T* __restrict__ q_out,
                                        T* __restrict__ k_tab, T* __restrict__ v_tab) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x;
  if (i >= m) return;
  const int half = d / 2;
  const int qd = h * d, kd = hkv * d;
  const int width = qd + 2 * kd;
  const float* row = qkv + i * width;
  const int p = pos[i];
  const int64_t dst = dst_rows ? dst_rows[i] : i;
  const double* ct = ctab + (int64_t)p * half;
  const double* st = stab + (int64_t)p * half;
  // pairs of Q and K (rotated), then V elements (copied)
  const int n_pairs = (qd + kd) / 2;
  for (int t = threadIdx.x; t < n_pairs; t += blockDim.x) {
    const int e = 2 * t;
    const int j = (e % d) >> 1;
    float oe, oo;
    if (kExact) rotate_pair_exact(row[e], row[e + 1], ct[j], st[j], oe, oo);
    else rotate_pair_fast(row[e], row[e + 1], (float)ct[j], (float)st[j], oe, oo);
    if (e < qd) {
      T* q = q_out + i * qd + e;
      q[0] = from_f<T>(oe);
      q[1] = from_f<T>(oo);
    } else {
      T* k = k_tab + dst * kd + (e - qd);
      k[0] = from_f<T>(oe);
      k[1] = from_f<T>(oo);
    }
  }
  for (int e = threadIdx.x; e < kd; e += blockDim.x) v_tab[dst * kd + e] = from_f<T>(row[qd + kd + e]);
}

}  // namespace qcf

extern "C" int qcf_rope_qkv_scatter(const float* qkv, int64_t m, int h, int hkv, int d,
                                    const int32_t* pos, const int32_t* dst_rows,
                                    const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                                    void* q_out, void* k_tab, void* v_tab, int dtype,
                                    qcf_stream_t stream) {
  QCF_REQUIRE(qkv && pos && cos_tbl && sin_tbl && q_out && k_tab && v_tab, QCF_EINVAL,
              "qcf_rope_qkv_scatter: null pointer");
  QCF_REQUIRE(h > 0 && hkv > 0 && h % hkv == 0 && d % 2 == 0, QCF_EINVAL,
              "qcf_rope_qkv_scatter: bad head shape");
  (void)n_pos;  // positions are bounds-checked by the host (table covers max position)
  if (m == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  if (dtype == QCF_F32)
    QCF_LAUNCH("rope_qkv_scatter_kernel", qcf::rope_qkv_scatter_kernel<float, true>, dim3((unsigned)m), dim3(256), 0, s, qkv, m, h, hkv, d, pos,
        dst_rows, cos_tbl, sin_tbl, (float*)q_out, (float*)k_tab, (float*)v_tab);
  else if (dtype == QCF_BF16)
    QCF_LAUNCH("rope_qkv_scatter_kernel", qcf::rope_qkv_scatter_kernel<__nv_bfloat16, false>, dim3((unsigned)m), dim3(256), 0, s, qkv, m, h, hkv, d,
        pos, dst_rows, cos_tbl, sin_tbl, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_tab,
        (__nv_bfloat16*)v_tab);
  else
    QCF_REQUIRE(false, QCF_EINVAL, "qcf_rope_qkv_scatter: bad dtype");
  QCF_LAUNCH_CHECK("qcf_rope_qkv_scatter");
  return QCF_OK;
}
