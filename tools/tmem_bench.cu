// tcgen05.ld throughput on one SM: W warps (one per TMEM lane quarter, or several per
// quarter) each load 32 lanes x 32 columns (4 KB) per tcgen05.ld.32x32b.x32 in a loop;
// reports bytes per SM clock. Also with tcgen05.mma traffic (SS 128x128x16) running.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2604_08585_b200/csrc \
//        -o tools/bin/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace qcf::sm100;

__global__ void __launch_bounds__(512, 1) kern(int n_warps, int iters, int with_mma, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  __shared__ volatile int done;
  __shared__ int finished;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i & 255);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); done = 0; finished = 0; }
  if (warp == 0) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  uint32_t acc = 0;
  if (warp == 15 && with_mma) {   // keep the tensor core busy: SS 128x128x16 into columns 256..383
    const uint32_t idesc = idesc_bf16_f32(128, 128);
    const uint64_t a0 = umma_desc_k_sw128(smem), b0 = umma_desc_k_sw128(smem + 16384);
    while (!done) {
      for (int i = 0; i < 64; ++i) mma_bf16_e(tmem + 256, a0 + (uint64_t)((i & 3) * 2), b0 + (uint64_t)((i & 3) * 2), idesc, 1u);
    }
  } else if (warp < n_warps) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      tmem_ld32(base, r);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 32; ++q) acc += r[q];
    }
    long long t1 = clock64();
    if (lane == 0) {
      out[warp] = t1 - t0;
      if (atomicAdd(&finished, 1) == n_warps - 1) done = 1;
    }
  }
  if (acc == 12345) out[63] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int iters = 4096;
  for (int mma = 0; mma < 2; ++mma)
    for (int nw : {1, 4, 8, 12}) {
      cudaMemset(d, 0, 64 * 8);
      kern<<<1, 512, 70000>>>(nw, iters, mma, d);
      kern<<<1, 512, 70000>>>(nw, iters, mma, d);
      long long h[64];
      cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
      const double bytes = (double)nw * iters * 4096.0;
      printf("{\"warps\": %d, \"mma_running\": %d, \"bytes_per_clk\": %.1f, \"clk_per_ld_per_warp\": %.1f, \"err\": \"%s\"}\n",
             nw, mma, bytes / mx, (double)mx / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
