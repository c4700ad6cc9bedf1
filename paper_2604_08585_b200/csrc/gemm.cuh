// Shared GEMM contract helpers (epilogues, argument checks).
#pragma once
#include "common.cuh"

namespace qcf {

__device__ __forceinline__ void epilogue_store(void* C, int64_t ldc, int64_t m, int64_t n, float v,
                                               int epi, int out_dtype) {
  if (epi == QCF_EPI_ADD_F32) {
    float* c = reinterpret_cast<float*>(C) + m * ldc + n;
    *c = *c + v;
    return;
  }
  if (epi == QCF_EPI_RELU) v = fmaxf(v, 0.f);
  if (out_dtype == QCF_F32) reinterpret_cast<float*>(C)[m * ldc + n] = v;
  else reinterpret_cast<__nv_bfloat16*>(C)[m * ldc + n] = __float2bfloat16_rn(v);
}

inline int gemm_check_args(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb,
                           void* c, int64_t ldc, int64_t m, int64_t n, int64_t k, int epi,
                           int out_dtype) {
  QCF_REQUIRE(a && b && c, QCF_EINVAL, "qcf_gemm: null pointer");
  QCF_REQUIRE(dtype == QCF_F32 || dtype == QCF_BF16, QCF_EINVAL, "qcf_gemm: bad dtype %d", dtype);
  QCF_REQUIRE(out_dtype == QCF_F32 || out_dtype == QCF_BF16, QCF_EINVAL, "qcf_gemm: bad out dtype");
  QCF_REQUIRE(epi >= QCF_EPI_STORE && epi <= QCF_EPI_ADD_F32, QCF_EINVAL, "qcf_gemm: bad epilogue");
  QCF_REQUIRE(epi != QCF_EPI_ADD_F32 || out_dtype == QCF_F32, QCF_EINVAL,
              "qcf_gemm: residual epilogue needs f32 output");
  QCF_REQUIRE(m >= 0 && n >= 0 && k > 0, QCF_ESHAPE, "qcf_gemm: bad sizes");
  QCF_REQUIRE(lda >= k && ldb >= k && ldc >= n, QCF_ESHAPE, "qcf_gemm: leading dims too small");
  return QCF_OK;
}

int gemm_simt_launch(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb, void* c,
                     int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue, int out_dtype,
                     cudaStream_t s);
// tcgen05 path; returns QCF_EUNSUPPORTED when the shape/alignment is not covered.
int gemm_tc_launch(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc,
                   int64_t m, int64_t n, int64_t k, int epilogue, int out_dtype, cudaStream_t s, int b_layout = 0,
                   void* ws = nullptr, size_t ws_bytes = 0);

size_t gemm_workspace_bytes(int64_t m, int64_t n, int64_t k);
int gemm_qkv_rope_launch(const void* a, int64_t lda, const void* w, int64_t ldb, int64_t m, int64_t k, int h,
                         int hkv, int d, const int32_t* pos, const int32_t* dst, const float* cs_tbl,
                         void* q_out, void* k_tab, void* v_tab, cudaStream_t s,
                         int b_layout, void* ws, size_t ws_bytes);
int gemm_tc_skinny(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                   int64_t n, int64_t k, int epilogue, int out_dtype, int b_layout, void* ws, size_t ws_bytes,
                   cudaStream_t s);

}  // namespace qcf
