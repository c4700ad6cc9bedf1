// K4 on the 5th-gen tensor cores: critical-layer query->context scoring
// (fusion.py:313-326 + _softmax_last 566-569) in the bf16 speed mode.
//
//   s[h,t,n] = (Q_c[t,h] . K_c[n,h]) * scale        softmax over the n_ctx keys
//   score[n] = mean_{h,t} softmax_n(s[h,t,:])
//
// One CTA = (128 context keys, one kv head, one request). The K tile is the
// UMMA A operand (M = 128 keys = TMEM lanes); the B operand is every query row
// of the heads sharing that kv head (N = G*nt columns, G = H/Hkv), staged by a
// 3D TMA box straight out of the [t][H][D] probe output. One elected thread
// issues D/16 tcgen05.mma into a TMEM accumulator [128 keys x N].
//
// The softmax needs global row statistics before the column reduction, so the
// contraction runs twice (K re-read, mostly from L2):
//   pass 1  per (row, key tile): tile max and sum of exp (row = (h,t) = a TMEM
//           column): each warp transposes-and-reduces its 32x32 TMEM block with
//           31 shuffles (recursive halving), 4 warps combine through smem.
//   pass 2  every thread owns one key (one TMEM lane): it folds the global
//           (max, sum) of each column into sum_c exp(s - M_c) / L_c over its G*nt
//           columns, in registers -> partial[kv head][key].
//   stats   per (h,t) row: fold the tile partials into (max, 1/sum) once.
//   final   score[n] = sum over kv heads (fixed order) / (H * nt).
// Deterministic (no atomics). Work per request: 2 x 2*n_ctx*H*nt*D flop and
// 2 x n_ctx*Hkv*D*2 bytes of K.
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

namespace qcf {

using namespace sm100;

int make_kmajor_map3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld, int box_rows,
                     int64_t batch, int64_t batch_stride);
int make_map_bf16(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                  const uint32_t* box);

constexpr int ST_BM = 128;                 // keys per CTA
constexpr int ST_MAXN = 256;               // query columns per CTA (UMMA N limit)
constexpr int ST_THREADS = 128;

__device__ __forceinline__ float st_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Recursive-halving transpose reduction: lane i ends with op over the warp's 32
// lanes of column i of the 32x32 block v[] (31 shuffles).
template <bool MAX>
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = upper ? v[i] : v[i + o];
      const float keep = upper ? v[i + o] : v[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[i] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
  return v[0];
}

template <bool PASS2>
__global__ void __launch_bounds__(ST_THREADS)
score_tc_kernel(const __grid_constant__ CUtensorMap map_k, const __grid_constant__ CUtensorMap map_q, int n_ctx,
                int nq, int t0, int nt, int H, int Hkv, int D, int n_pad, float sl2, float2* __restrict__ stats,
                float* __restrict__ partial) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int n_atoms = D / 64;
  const int q_atom = n_pad * 128;
  uint8_t* sK = smem;                                  // [D/64][128 keys][128 B]
  uint8_t* sQ = smem + n_atoms * ST_BM * 128;          // [D/64][n_pad rows][128 B]
  __shared__ uint64_t bar_full, bar_done;
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][4][32];
  __shared__ float sM[ST_MAXN], sInv[ST_MAXN];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int G = H / Hkv;
  const int N = G * nt;
  const int n_kt = gridDim.x;
  const uint32_t cols = n_pad <= 32 ? 32 : (n_pad <= 64 ? 64 : (n_pad <= 128 ? 128 : 256));

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_q);
    mbar_init(&bar_full, 1);
    mbar_init(&bar_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_slot, cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem = tmem_slot;

  if (threadIdx.x < 32) {  // warp 0: one lane loads, the converged warp issues (elected lane)
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar_full, (uint32_t)(n_atoms * (ST_BM + N) * 128));
      for (int a = 0; a < n_atoms; ++a) {
        tma_load_3d(sK + a * ST_BM * 128, &map_k, &bar_full, kvh * D + a * 64, kt * ST_BM, req);
        tma_load_3d(sQ + a * q_atom, &map_q, &bar_full, a * 64, kvh * G, req * nq + t0);
      }
    }
    __syncwarp();
    mbar_wait(&bar_full, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(ST_BM, n_pad);
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint64_t a = umma_desc_k_sw128(sK + (kk >> 2) * (ST_BM * 128)) + (uint64_t)((kk & 3) * 2);
      const uint64_t b = umma_desc_k_sw128(sQ + (kk >> 2) * q_atom) + (uint64_t)((kk & 3) * 2);
      mma_bf16_e(tmem, a, b, idesc, kk != 0);
    }
    mma_commit_e(&bar_done);
  }

  const int key = kt * ST_BM + warp * 32 + lane;
  const bool valid = key < n_ctx;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;

  if (PASS2) {
    // global (max, 1/sum) of every column, reduced once by score_tc_stats_kernel
    for (int c = threadIdx.x; c < N; c += ST_THREADS) {
      const int head = kvh * G + c % G, t = c / G;
      const float2 ms = stats[((int64_t)req * H * nt + (int64_t)head * nt + t) * n_kt];
      sM[c] = ms.x;
      sInv[c] = ms.y;
    }
    __syncthreads();
  }

  mbar_wait(&bar_done, 0);
  tc_fence_after();

  float acc = 0.f;
  for (int c0 = 0; c0 < n_pad; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + c0, r);
    tmem_ld_wait();
    if (PASS2) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int c = c0 + i;
        if (c < N) acc += st_ex2(fmaf(__uint_as_float(r[i]), sl2, -sM[c])) * sInv[c];
      }
    } else {
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = valid ? __uint_as_float(r[i]) * sl2 : -INFINITY;
      float e[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) e[i] = v[i];
      const float wmax = warp_transpose_reduce<true>(e, lane);   // column c0+lane over this warp's keys
      red[0][warp][lane] = wmax;
      __syncthreads();
      const float cmax = fmaxf(fmaxf(red[0][0][lane], red[0][1][lane]), fmaxf(red[0][2][lane], red[0][3][lane]));
#pragma unroll
      for (int i = 0; i < 32; ++i) e[i] = st_ex2(v[i] - __shfl_sync(0xffffffffu, cmax, i));
      const float wsum = warp_transpose_reduce<false>(e, lane);
      red[1][warp][lane] = wsum;
      __syncthreads();
      if (warp == 0 && c0 + lane < N) {
        const int c = c0 + lane;
        const int head = kvh * G + c % G, t = c / G;
        const float l = (red[1][0][lane] + red[1][1][lane]) + (red[1][2][lane] + red[1][3][lane]);
        stats[((int64_t)req * H * nt + (int64_t)head * nt + t) * n_kt + kt] = make_float2(cmax, l);
      }
      __syncthreads();
    }
  }
  if (PASS2 && valid) partial[((int64_t)req * Hkv + kvh) * n_ctx + key] = acc;

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, cols);
  }
}

// between the passes: per (h, t) row, fold the per-key-tile (max, sum) partials
// into (max, 1/sum), stored in the row's first slot (deterministic order)
__global__ void score_tc_stats_kernel(float2* __restrict__ stats, int64_t n_rows, int n_kt) {
  pdl_wait();
  pdl_trigger();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= n_rows) return;
  float2* p = stats + row * n_kt;
  float m = -INFINITY;
  for (int j = 0; j < n_kt; ++j) m = fmaxf(m, p[j].x);
  float l = 0.f;
  for (int j = 0; j < n_kt; ++j) l += p[j].y * st_ex2(p[j].x - m);
  p[0] = make_float2(m, 1.f / l);
}

__global__ void score_tc_final_kernel(const float* __restrict__ partial, int n_ctx, int Hkv, float inv_rows,
                                      float* __restrict__ scores) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int req = blockIdx.y;
  if (n >= n_ctx) return;
  const float* p = partial + (int64_t)req * Hkv * n_ctx + n;
  float s = 0.f;
  for (int h = 0; h < Hkv; ++h) s += p[(int64_t)h * n_ctx];
  scores[(int64_t)req * n_ctx + n] = s * inv_rows;
}

size_t score_tc_workspace(int64_t n_ctx, int nq, int h, int hkv, int n_req) {
  const int64_t n_kt = (n_ctx + ST_BM - 1) / ST_BM;
  return (size_t)n_req * ((size_t)h * nq * n_kt * sizeof(float2) + (size_t)hkv * n_ctx * sizeof(float)) + 256;
}

// q: [n_req*nq][H][D] bf16; k: request r's context keys at k + r*k_req_stride
// elements, rows of Hkv*D; scores [n_req][n_ctx].
int score_tc_launch(const void* q, const void* k, int64_t k_req_stride, int64_t n_ctx, int nq, int n_req, int h,
                    int hkv, int d, double scale, int agg_last, float* scores, void* ws, size_t ws_bytes,
                    cudaStream_t s) {
  const int t0 = agg_last ? nq - 1 : 0;
  const int nt = nq - t0;
  const int G = h / hkv;
  const int N = G * nt;
  const int n_pad = (N + 15) / 16 * 16;
  if (d % 64 != 0 || d > 256 || n_pad > ST_MAXN || G > 256 || nt > 256 || n_ctx > INT32_MAX || n_req > 65535)
    return QCF_EUNSUPPORTED;
  if (((uintptr_t)q | (uintptr_t)k) & 15) return QCF_EUNSUPPORTED;
  if ((k_req_stride * 2) % 16 != 0) return QCF_EUNSUPPORTED;
  QCF_REQUIRE(ws_bytes >= score_tc_workspace(n_ctx, nq, h, hkv, n_req), QCF_EWORKSPACE,
              "qcf_score: workspace too small");
  CUtensorMap mk, mq;
  const int64_t kw = (int64_t)hkv * d;
  int st = make_kmajor_map3(&mk, k, n_ctx, kw, kw, ST_BM, n_req, n_req > 1 ? k_req_stride : n_ctx * kw);
  if (st != QCF_OK) return st;
  const uint64_t qdims[3] = {(uint64_t)d, (uint64_t)h, (uint64_t)n_req * nq};
  const uint64_t qstr[2] = {(uint64_t)d * 2, (uint64_t)h * d * 2};
  const uint32_t qbox[3] = {64, (uint32_t)G, (uint32_t)nt};
  st = make_map_bf16(&mq, q, 3, qdims, qstr, qbox);
  if (st != QCF_OK) return st;
  const int n_kt = (int)((n_ctx + ST_BM - 1) / ST_BM);
  float2* stats = reinterpret_cast<float2*>(ws);
  float* partial = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) +
                                            (size_t)n_req * h * nq * n_kt * sizeof(float2));
  const size_t smem = 1024 + (size_t)(d / 64) * (ST_BM + n_pad) * 128;
  static bool attr = false;
  if (!attr) {
    for (auto fn : {score_tc_kernel<false>, score_tc_kernel<true>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(1024 + 4 * (ST_BM + ST_MAXN) * 128));
      if (e != cudaSuccess) return cuda_status(e, "score_tc attr");
    }
    attr = true;
  }
  const float sl2 = (float)scale * 1.4426950408889634f;
  const dim3 grid((unsigned)n_kt, (unsigned)hkv, (unsigned)n_req);
  QCF_LAUNCH("score_tc_kernel<1>", score_tc_kernel<false>, grid, dim3(ST_THREADS), smem, s, mk, mq, (int)n_ctx, nq,
             t0, nt, h, hkv, d, n_pad, sl2, stats, partial);
  QCF_LAUNCH_CHECK("qcf_score(tcgen05) pass 1");
  const int64_t n_rows = (int64_t)n_req * h * nt;
  QCF_LAUNCH("score_tc_stats_kernel", score_tc_stats_kernel, dim3(ceil_div(n_rows, 128)), dim3(128), 0, s, stats, n_rows,
             n_kt);
  QCF_LAUNCH_CHECK("qcf_score(tcgen05) stats");
  QCF_LAUNCH("score_tc_kernel<2>", score_tc_kernel<true>, grid, dim3(ST_THREADS), smem, s, mk, mq, (int)n_ctx, nq,
             t0, nt, h, hkv, d, n_pad, sl2, stats, partial);
  QCF_LAUNCH_CHECK("qcf_score(tcgen05) pass 2");
  QCF_LAUNCH("score_tc_final_kernel", score_tc_final_kernel, dim3(ceil_div(n_ctx, 256), n_req), dim3(256), 0, s,
             (const float*)partial, (int)n_ctx, hkv, 1.f / (float)(h * nt), scores);
  QCF_LAUNCH_CHECK("qcf_score(tcgen05) final");
  return QCF_OK;
}

}  // namespace qcf
