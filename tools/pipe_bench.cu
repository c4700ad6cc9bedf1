// Per-SM throughput of the instructions the attention softmax issues:
// MUFU.EX2 (ex2.approx.f32), F2FP (cvt.rn.bf16x2.f32), FFMA2, FMNMX3.
// One CTA of `warps` warps per SM, 8 independent chains per thread.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void bench(float* out, int iters, long long* cyc) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {
        asm volatile("ex2.approx.f32 %0, %0;" : "+f"(x[i]));
      } else if (OP == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        acc ^= r;
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (r & 1));
      } else if (OP == 2) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*reinterpret_cast<unsigned long long*>(&x[i & 6])) :
                     "l"(*reinterpret_cast<unsigned long long*>(&x[(i + 2) & 6])),
                     "l"(*reinterpret_cast<unsigned long long*>(&x[(i + 4) & 6])));
      } else if (OP == 3) {
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(x[(i + 1) & 7]), "f"(x[(i + 2) & 7]));
      } else if (OP == 4) {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(*reinterpret_cast<uint32_t*>(&x[i])));
      } else if (OP == 5) {  // scalar FFMA, 8 independent chains
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(x[(i + 1) & 7]), "f"(x[(i + 2) & 7]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = acc;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void bench_ffma2_8(float* out, int iters, long long* cyc) {
  unsigned long long y[8];
  for (int i = 0; i < 8; ++i) {
    float a = -0.001f * (threadIdx.x + i), b = 0.5f * i;
    y[i] = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
  }
  const unsigned long long c1 = 0x3f8000003f800000ull, c2 = 0x3c23d70a3c23d70aull;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[i]) : "l"(c1), "l"(c2));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)y[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static void run_ffma2_8(int warps) {
  const int iters = 4096, blocks = 148;
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * warps * 32 * sizeof(float));
  cudaMalloc(&cyc, blocks * sizeof(long long));
  bench_ffma2_8<<<blocks, warps * 32>>>(out, iters, cyc);
  bench_ffma2_8<<<blocks, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double winst = (double)iters * 8 * warps;
  printf("{\"op\": \"fma.rn.f32x2 x8 indep (const operands)\", \"warps\": %d, \"clk_per_warp_inst_per_sm\": %.3f}\n",
         warps, avg / winst);
  cudaFree(out);
  cudaFree(cyc);
}

template <int OP>
static void run(const char* name, int warps) {
  const int iters = 4096, blocks = 148;
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * warps * 32 * sizeof(float));
  cudaMalloc(&cyc, blocks * sizeof(long long));
  bench<OP><<<blocks, warps * 32>>>(out, iters, cyc);
  bench<OP><<<blocks, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double winst = (double)iters * 8 * warps;  // warp instructions per SM
  printf("{\"op\": \"%s\", \"warps\": %d, \"clk_per_warp_inst_per_sm\": %.3f, \"thread_ops_per_clk_per_sm\": %.2f}\n",
         name, warps, avg / winst, winst * 32 / avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16, 32}) {
    run_ffma2_8(w);
    run<5>("fma.rn.f32 scalar", w);
  }
  for (int w : {4, 8, 16}) {
    run<0>("ex2.approx.f32", w);
    run<1>("cvt.rn.bf16x2.f32", w);
    run<2>("fma.rn.f32x2", w);
    run<3>("max3.f32", w);
    run<4>("ex2.approx.ftz.bf16x2", w);
  }
  return 0;
}
