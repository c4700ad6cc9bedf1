// Shared helpers for the qcfuse_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>
#include <string>

#include "../../include/qcfuse_b200.h"

namespace qcf {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

#define QCF_REQUIRE(cond, code, ...)  \
  do {                                \
    if (!(cond)) {                    \
      ::qcf::set_error(__VA_ARGS__);  \
      return (code);                  \
    }                                 \
  } while (0)

#define QCF_LAUNCH_CHECK(where) \
  do { cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) return ::qcf::cuda_status(_e, where); } while (0)

inline cudaStream_t as_stream(qcf_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---- element conversion ----------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// Warp reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Exact float64 pair rotation, written with explicit round-to-nearest ops so
// nvcc cannot contract into FMA: reproduces numpy's
//   out_even = even*cos - odd*sin ; out_odd = even*sin + odd*cos
// on float64 followed by astype(float32)   (model.py:282-286).
__device__ __forceinline__ void rotate_pair_exact(float e, float o, double c, double s,
                                                  float& oe, float& oo) {
  double de = (double)e, dd = (double)o;
  oe = __double2float_rn(__dsub_rn(__dmul_rn(de, c), __dmul_rn(dd, s)));
  oo = __double2float_rn(__dadd_rn(__dmul_rn(de, s), __dmul_rn(dd, c)));
}

__device__ __forceinline__ void rotate_pair_fast(float e, float o, float c, float s,
                                                 float& oe, float& oo) {
  oe = e * c - o * s;
  oo = e * s + o * c;
}


// ---- Programmatic Dependent Launch ---------------------------------------------
// Every hot-path kernel is launched with programmatic stream serialisation: it
// may be scheduled while its predecessor drains, runs its prologue, and blocks
// in pdl_wait() (griddepcontrol.wait = predecessor complete + memory visible)
// before touching global memory; pdl_trigger() lets the next kernel launch.
// Both are no-ops when a kernel is launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define QCF_LAUNCH(where, ...)                                          \
  do {                                                                  \
    cudaError_t _e = ::qcf::launch_k(__VA_ARGS__);                     \
    if (_e != cudaSuccess) return ::qcf::cuda_status(_e, where);        \
  } while (0)
}  // namespace qcf
