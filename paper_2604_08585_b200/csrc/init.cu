// On-device deterministic weight init: the splitmix64 stream of model.py:35-46
// mapped as model.py:67-69 / 240-241, bit-identical to the reference's float32
// weights. Generating on the GPU avoids the reference's >= 94 GB host
// temporaries at Llama-3-8B shape (model.py:240-241 materialises every draw).
#include "common.cuh"

namespace qcf {

__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t step) {
  uint64_t z = seed + (step + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// float32(-0.05 + u53 * (0.05 - (-0.05))) with the same float64 rounding steps
__device__ __forceinline__ float draw_weight(uint64_t seed, uint64_t step) {
  const double lo = -0.05, range = 0.05 - (-0.05);
  double u = (double)(splitmix64_at(seed, step) >> 11) * 0x1.0p-53;
  return __double2float_rn(__dadd_rn(lo, __dmul_rn(u, range)));
}

template <typename T>
__global__ void init_uniform_kernel(uint64_t seed, uint64_t start, int64_t rows, int64_t cols,
                                    int transpose, T* __restrict__ out, int64_t ld) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int j = ty; j < 32; j += 8) {
    int64_t r = r0 + j, c = c0 + tx;
    float v = 0.f;
    if (r < rows && c < cols) v = draw_weight(seed, start + (uint64_t)(r * cols + c));
    if (!transpose) {
      if (r < rows && c < cols) out[r * ld + c] = from_f<T>(v);
    } else {
      tile[j][tx] = v;
    }
  }
  if (!transpose) return;
  __syncthreads();
  // out[c][r]: lanes walk r (contiguous)
  for (int j = ty; j < 32; j += 8) {
    int64_t c = c0 + j, r = r0 + tx;
    if (r < rows && c < cols) out[c * ld + r] = from_f<T>(tile[tx][j]);
  }
}

}  // namespace qcf

extern "C" int qcf_init_uniform(uint64_t seed, uint64_t start, int64_t rows, int64_t cols,
                                int transpose, int out_dtype, void* out, int64_t ld_out,
                                qcf_stream_t stream) {
  QCF_REQUIRE(out && rows >= 0 && cols >= 0, QCF_EINVAL, "qcf_init_uniform: bad args");
  QCF_REQUIRE(ld_out >= (transpose ? rows : cols), QCF_ESHAPE, "qcf_init_uniform: ld_out too small");
  if (rows == 0 || cols == 0) return QCF_OK;
  dim3 grid(qcf::ceil_div(cols, 32), qcf::ceil_div(rows, 32)), block(32, 8);
  QCF_REQUIRE(grid.y <= 65535, QCF_EUNSUPPORTED, "qcf_init_uniform: too many rows");
  auto s = qcf::as_stream(stream);
  if (out_dtype == QCF_F32)
    QCF_LAUNCH("init_uniform_kernel", qcf::init_uniform_kernel<float>, dim3(grid), dim3(block), 0, s, seed, start, rows, cols, transpose, (float*)out, ld_out);
  else if (out_dtype == QCF_BF16)
    QCF_LAUNCH("init_uniform_kernel", qcf::init_uniform_kernel<__nv_bfloat16>, dim3(grid), dim3(block), 0, s, seed, start, rows, cols, transpose, (__nv_bfloat16*)out, ld_out);
  else
    QCF_REQUIRE(false, QCF_EINVAL, "qcf_init_uniform: bad dtype %d", out_dtype);
  QCF_LAUNCH_CHECK("qcf_init_uniform");
  return QCF_OK;
}
