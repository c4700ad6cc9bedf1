// Microbenchmark: how fast can 148 CTAs stream a weight matrix through TMA
// into a shared-memory ring (no math)? Varies box size and ring depth.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../../paper_2604_08585_b200/csrc/sm100.cuh"
using namespace qcf::sm100;

template <int STAGES, int BOX_ROWS, int KATOMS>
__global__ void __launch_bounds__(128) stream_kernel(const __grid_constant__ CUtensorMap map, int n_rowblocks, int k_atoms, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int ATOM = BOX_ROWS * 128;
  constexpr int STAGE = ATOM * KATOMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  // work: row-block rb = blockIdx.x + i*grid, all k atoms
  const int kst = k_atoms / KATOMS;
  int total = 0;
  for (int rb = blockIdx.x; rb < n_rowblocks; rb += gridDim.x) total += kst;
  if (threadIdx.x == 0) {
    int it = 0;
    for (int rb = blockIdx.x; rb < n_rowblocks; rb += gridDim.x)
      for (int kb = 0; kb < kst; ++kb, ++it) {
        const int s = it % STAGES; const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], STAGE);
        for (int j = 0; j < KATOMS; ++j)
          tma_load_4d(smem + s * STAGE + j * ATOM, &map, &full[s], 0, 0, kb * KATOMS + j, rb * (BOX_ROWS / 64));
      }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int it = 0; it < total; ++it) {
      const int s = it % STAGES; const uint32_t ph = (it / STAGES) & 1;
      mbar_wait(&full[s], ph);
      acc += smem[s * STAGE + 5];
      mbar_arrive(&empty[s]);
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, int BOX_ROWS, int KATOMS>
void run(void* w, int64_t n, int64_t k, EncodeTiledFn enc, int grid, unsigned long long* sink, void* flush, size_t fbytes) {
  CUtensorMap map;
  cuuint64_t dims[4] = {64, 64, (cuuint64_t)(k / 64), (cuuint64_t)(n / 64)};
  cuuint64_t strides[3] = {128, 8192, (cuuint64_t)(k / 64) * 8192};
  cuuint32_t box[4] = {64, 64, 1, (cuuint32_t)(BOX_ROWS / 64)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, w, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = STAGES * BOX_ROWS * 128 * KATOMS + 1024 + 256;
  cudaFuncSetAttribute(stream_kernel<STAGES, BOX_ROWS, KATOMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemset(flush, r, fbytes);
    cudaEventRecord(e0);
    stream_kernel<STAGES, BOX_ROWS, KATOMS><<<grid, 128, smem>>>(map, (int)(n / BOX_ROWS), (int)(k / 64), sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("stages=%2d box_rows=%3d katoms=%d grid=%d: %.1f us  %.0f GB/s  (%s)\n", STAGES, BOX_ROWS, KATOMS, grid, best * 1e3,
         n * k * 2 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t n = 12288, k = 4096;
  void* w; cudaMalloc(&w, n * k * 2); cudaMemset(w, 1, n * k * 2);
  size_t fb = 512ull << 20; void* flush; cudaMalloc(&flush, fb);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)p;
  run<4, 64, 1>(w, n, k, enc, 148, sink, flush, fb);
  run<4, 64, 1>(w, n, k, enc, 296, sink, flush, fb);
  run<4, 64, 1>(w, n, k, enc, 592, sink, flush, fb);
  run<8, 64, 1>(w, n, k, enc, 296, sink, flush, fb);
  run<8, 64, 1>(w, n, k, enc, 592, sink, flush, fb);
  run<2, 64, 4>(w, n, k, enc, 296, sink, flush, fb);
  run<2, 64, 4>(w, n, k, enc, 592, sink, flush, fb);
  run<16, 64, 1>(w, n, k, enc, 296, sink, flush, fb);
  // plain memcpy reference
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  void* dst; cudaMalloc(&dst, n * k * 2);
  cudaMemset(flush, 3, fb);
  cudaEventRecord(e0); cudaMemcpy(dst, w, n * k * 2, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("memcpy D2D 100MB: %.1f us  %.0f GB/s (r+w)\n", ms * 1e3, 2 * n * k * 2 / (ms * 1e-3) / 1e9);
  return 0;
}
