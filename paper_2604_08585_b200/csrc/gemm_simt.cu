// FFMA (SIMT) GEMM: the float32 parity-mode projection kernel and the
// cross-check for the tcgen05 path. C[M,N] (op)= A[M,K] . B[N,K]^T with fp32
// accumulation (model.py:361-363, 375, 341-342 compute a @ W in float32).
#include "common.cuh"
#include "gemm.cuh"

namespace qcf {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename TIn>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const TIn* __restrict__ A, int64_t lda,
                                                        const TIn* __restrict__ B, int64_t ldb,
                                                        void* __restrict__ C, int64_t ldc, int64_t M,
                                                        int64_t N, int64_t K, int epi, int out_dtype) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) float As[SB_K][SB_M + 4];
  __shared__ __align__(16) float Bs[SB_K][SB_N + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * SB_M, n0 = (int64_t)blockIdx.x * SB_N;
  float acc[4][4] = {};
  // loader mapping: 64 rows x 16 k, 4 elements per thread along k
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  for (int64_t k0 = 0; k0 < K; k0 += SB_K) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t kk = k0 + lk + u;
      int64_t am = m0 + lr, bn = n0 + lr;
      As[lk + u][lr] = (am < M && kk < K) ? to_f<TIn>(A[am * lda + kk]) : 0.f;
      Bs[lk + u][lr] = (bn < N && kk < K) ? to_f<TIn>(B[bn * ldb + kk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      epilogue_store(C, ldc, m, n, acc[i][j], epi, out_dtype);
    }
  }
}

int gemm_simt_launch(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb, void* c,
                     int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue, int out_dtype,
                     cudaStream_t s) {
  dim3 grid(ceil_div(n, SB_N), ceil_div(m, SB_M));
  QCF_REQUIRE(grid.y <= 65535, QCF_EUNSUPPORTED, "gemm_simt: M too large");
  if (dtype == QCF_F32)
    QCF_LAUNCH("gemm_simt_kernel", gemm_simt_kernel<float>, dim3(grid), dim3(256), 0, s, (const float*)a, lda, (const float*)b, ldb, c, ldc,
                                                 m, n, k, epilogue, out_dtype);
  else
    QCF_LAUNCH("gemm_simt_kernel", gemm_simt_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, (const __nv_bfloat16*)a, lda,
        (const __nv_bfloat16*)b, ldb, c, ldc, m, n, k, epilogue, out_dtype);
  QCF_LAUNCH_CHECK("qcf_gemm_simt");
  return QCF_OK;
}

}  // namespace qcf

extern "C" int qcf_gemm_simt(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb,
                             void* c, int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue,
                             int out_dtype, qcf_stream_t stream) {
  int st = qcf::gemm_check_args(dtype, a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype);
  if (st != QCF_OK) return st;
  if (m == 0 || n == 0) return QCF_OK;
  return qcf::gemm_simt_launch(dtype, a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype,
                               qcf::as_stream(stream));
}
