// tcgen05 GEMM for the projections of the probe, the selective recompute and
// full prefill (model.py:361-363, 375, 341-342):  C[M,N] (op)= A[M,K] . B[N,K]^T
// with bf16 operands and fp32 accumulation in tensor memory.
//
// Persistent, warp-specialised CTA (one per SM):
//   warp 0      TMA producer  : A/B K-slabs (64 elements = one 128 B swizzle atom)
//                               into a STAGES-deep shared-memory ring
//   warp 1      MMA issuer    : one elected thread issues tcgen05.mma 128xBNx16
//                               into one of two TMEM accumulators
//   warps 2..5  epilogue      : tcgen05.ld -> fused epilogue (store / ReLU /
//                               residual add) -> global; overlaps the next
//                               tile's main loop (double-buffered TMEM)
// Tiles run m-fastest so consecutive CTAs share the weight (B) tile in L2.
#include <cuda.h>

#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "gemm.cuh"
#include "sm100.cuh"

namespace qcf {

using namespace sm100;

constexpr int TC_BM = 128, TC_BK = 64;
constexpr int TC_THREADS = 192;


// fused epilogue for 32 consecutive columns of one output row
__device__ __forceinline__ void epilogue_row32(void* __restrict__ C, int64_t ldc, int row, int col0, int N,
                                               const uint32_t (&r)[32], int epi, int out_dtype) {
  if (out_dtype == QCF_F32) {
    float* crow = reinterpret_cast<float*>(C) + (int64_t)row * ldc + col0;
    if (col0 + 32 <= N) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                               __uint_as_float(r[j + 3]));
        if (epi == QCF_EPI_ADD_F32) {
          float4 o = *reinterpret_cast<const float4*>(crow + j);
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        } else if (epi == QCF_EPI_RELU) {
          v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
        }
        *reinterpret_cast<float4*>(crow + j) = v;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < N; ++j) {
        float v = __uint_as_float(r[j]);
        if (epi == QCF_EPI_ADD_F32) v += crow[j];
        else if (epi == QCF_EPI_RELU) v = fmaxf(v, 0.f);
        crow[j] = v;
      }
    }
  } else {
    __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)row * ldc + col0;
    if (col0 + 32 <= N) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 pk;
        __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float x = __uint_as_float(r[j + 2 * u]), y = __uint_as_float(r[j + 2 * u + 1]);
          if (epi == QCF_EPI_RELU) { x = fmaxf(x, 0.f); y = fmaxf(y, 0.f); }
          p2[u] = __floats2bfloat162_rn(x, y);
        }
        *reinterpret_cast<uint4*>(crow + j) = pk;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < N; ++j) {
        float v = __uint_as_float(r[j]);
        if (epi == QCF_EPI_RELU) v = fmaxf(v, 0.f);
        crow[j] = __float2bfloat16_rn(v);
      }
    }
  }
}

template <int BN>
struct TcCfg {
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulators
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               void* __restrict__ C, int64_t ldc, int M, int N, int K, int epi, int out_dtype) {
  using Cfg = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;   // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (M + TC_BM - 1) / TC_BM;
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_tiles * n_tiles;
  const int k_blocks = (K + TC_BK - 1) / TC_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < Cfg::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      uint32_t it = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int mb = w % m_tiles, nb = w / m_tiles;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
          tma_load_2d(sA + s * Cfg::A_BYTES, &map_a, &full[s], kb * TC_BK, mb * TC_BM);
          tma_load_2d(sB + s * Cfg::B_BYTES, &map_b, &full[s], kb * TC_BK, nb * BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(TC_BM, BN);
      uint32_t it = 0, t = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a0 = umma_desc_k_sw128(sA + s * Cfg::A_BYTES);
          const uint64_t b0 = umma_desc_k_sw128(sB + s * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk)  // +32 B per K=16 step inside the swizzle atom
            mma_bf16(d_tmem, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5
    const int g = warp & 3;  // TMEM lane quarter this warp may access
    uint32_t t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      const int mb = w % m_tiles, nb = w / m_tiles;
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const int row = mb * TC_BM + g * 32 + lane;
      const bool row_ok = row < M;
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * BN + cc * 32 + ((uint32_t)(g * 32) << 16), r);
        tmem_ld_wait();
        const int col0 = nb * BN + cc * 32;
        if (!row_ok || col0 >= N) continue;
        epilogue_row32(C, ldc, row, col0, N, r, epi, out_dtype);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- 2-CTA variant
// A CTA pair (cluster of 2) computes a 256 x BN tile with tcgen05.mma.cta_group::2:
// CTA r holds A rows [128r, 128r+128) and B rows [r*BN/2, (r+1)*BN/2) of the tile,
// the leader (rank 0) issues the MMAs, each CTA's TMEM holds its 128 output rows.
// Per SM this halves the B bytes per MMA cycle, doubling the TMA lookahead.
template <int BN>
struct Tc2Cfg {
  static constexpr int STAGES = 6;
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;          // 16 KB (this CTA's 128 rows)
  static constexpr int B_BYTES = (BN / 2) * TC_BK * 2;       // this CTA's half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                void* __restrict__ C, int64_t ldc, int M, int N, int K, int epi, int out_dtype) {
  using Cfg = Tc2Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;   // [2]
  uint64_t* tempty = tfull + 2;            // [2] (leader's copy is the one used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int m_pairs = (M + 2 * TC_BM - 1) / (2 * TC_BM);
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_pairs * n_tiles;
  const int k_blocks = (K + TC_BK - 1) / TC_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < Cfg::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * 128); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      uint32_t it = 0;
      for (int w = cluster; w < n_work; w += n_clusters) {
        const int mp = w % m_pairs, nb = w / m_pairs;
        const int arow = mp * 2 * TC_BM + rank * TC_BM;
        const int brow = nb * BN + rank * (BN / 2);
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
          tma_load_2d_pair(sA + s * Cfg::A_BYTES, &map_a, &full[s], kb * TC_BK, arow);
          tma_load_2d_pair(sB + s * Cfg::B_BYTES, &map_b, &full[s], kb * TC_BK, brow);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (leader only)
      constexpr uint32_t idesc = idesc_bf16_f32(2 * TC_BM, BN);
      uint32_t it = 0, t = 0;
      for (int w = cluster; w < n_work; w += n_clusters, ++t) {
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a0 = umma_desc_k_sw128(sA + s * Cfg::A_BYTES);
          const uint64_t b0 = umma_desc_k_sw128(sB + s * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk)
            mma_bf16_pair(d_tmem, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          mma_commit_pair(&empty[s]);
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5 (both CTAs, own 128 rows)
    const int g = warp & 3;
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
    uint32_t t = 0;
    for (int w = cluster; w < n_work; w += n_clusters, ++t) {
      const int mp = w % m_pairs, nb = w / m_pairs;
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const int row = mp * 2 * TC_BM + rank * TC_BM + g * 32 + lane;
      const bool row_ok = row < M;
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * BN + cc * 32 + ((uint32_t)(g * 32) << 16), r);
        tmem_ld_wait();
        const int col0 = nb * BN + cc * 32;
        if (!row_ok || col0 >= N) continue;
        epilogue_row32(C, ldc, row, col0, N, r, epi, out_dtype);
      }
      tc_fence_before();
      mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2D bf16 K-major operand [rows][k] with leading dimension ld, box {64, box_rows}, SW128
int make_kmajor_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld, int box_rows) {
  EncodeTiledFn enc = get_encode();
  QCF_REQUIRE(enc, QCF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QCF_REQUIRE(r == CUDA_SUCCESS, QCF_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return QCF_OK;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN>
static int launch_bn(const CUtensorMap& ma, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                     int64_t n, int64_t k, int epi, int out_dtype, cudaStream_t s) {
  CUtensorMap mb;
  int st = make_kmajor_map(&mb, b, n, k, ldb, BN);
  if (st != QCF_OK) return st;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TcCfg<BN>::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc attr");
    attr_set = true;
  }
  const int64_t work = ((m + TC_BM - 1) / TC_BM) * ((n + BN - 1) / BN);
  const int grid = (int)std::min<int64_t>(work, sm_count());
  gemm_tc_kernel<BN><<<grid, TC_THREADS, TcCfg<BN>::SMEM, s>>>(ma, mb, c, ldc, (int)m, (int)n, (int)k, epi,
                                                               out_dtype);
  QCF_LAUNCH_CHECK("qcf_gemm(tcgen05)");
  return QCF_OK;
}

template <int BN>
static int launch_pair(const CUtensorMap& ma, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                       int64_t n, int64_t k, int epi, int out_dtype, cudaStream_t s) {
  CUtensorMap mb;
  int st = make_kmajor_map(&mb, b, n, k, ldb, BN / 2);
  if (st != QCF_OK) return st;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Tc2Cfg<BN>::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc2 attr");
    attr_set = true;
  }
  const int64_t work = ((m + 2 * TC_BM - 1) / (2 * TC_BM)) * ((n + BN - 1) / BN);
  const int clusters = (int)std::min<int64_t>(work, sm_count() / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Tc2Cfg<BN>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<BN>, ma, mb, c, ldc, (int)m, (int)n, (int)k, epi,
                                     out_dtype);
  if (e != cudaSuccess) return cuda_status(e, "qcf_gemm(tcgen05 pair)");
  QCF_LAUNCH_CHECK("qcf_gemm(tcgen05 pair)");
  return QCF_OK;
}

static int g_pair_mode = -1;  // QCF_GEMM_PAIR env: 0 off, 1 on (default on)

int gemm_tc_launch(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                   int64_t n, int64_t k, int epilogue, int out_dtype, cudaStream_t s) {
  // TMA: 16-byte aligned bases and row strides; vector epilogue alignment
  if ((k % 8) || (lda % 8) || (ldb % 8) || ((uintptr_t)a & 15) || ((uintptr_t)b & 15)) return QCF_EUNSUPPORTED;
  if (out_dtype == QCF_F32 && ((ldc % 4) || ((uintptr_t)c & 15))) return QCF_EUNSUPPORTED;
  if (out_dtype == QCF_BF16 && ((ldc % 8) || ((uintptr_t)c & 15))) return QCF_EUNSUPPORTED;
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return QCF_EUNSUPPORTED;
  CUtensorMap ma;
  int st = make_kmajor_map(&ma, a, m, k, lda, TC_BM);
  if (st != QCF_OK) return st;
  if (g_pair_mode < 0) {
    const char* e = getenv("QCF_GEMM_PAIR");
    g_pair_mode = (e && e[0] == '0') ? 0 : 1;
  }
  const int sms = sm_count();
  const int64_t mt = (m + TC_BM - 1) / TC_BM;
  // 2-CTA 256-row tiles vs 1-CTA 128-row tiles: estimate each one's useful
  // fraction (wave quantisation x row padding; 1-CTA pays ~15% for its
  // shallower TMA lookahead) and take the better one
  if (g_pair_mode && m >= 192 && n >= 256) {
    const int64_t mps = (m + 255) / 256, units = mps * ((n + 255) / 256), clusters = sms / 2;
    const double e_pair = (double)units / (double)(((units + clusters - 1) / clusters) * clusters) *
                          (double)m / (double)(mps * 256);
    const int64_t t1 = mt * ((n + 255) / 256);
    const double e_one = 0.85 * (double)t1 / (double)(((t1 + sms - 1) / sms) * sms) * (double)m / (double)(mt * 128);
    if (units >= clusters / 2 && e_pair >= e_one)
      return launch_pair<256>(ma, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s);
  }
  // tile width: enough tiles to cover the SMs, widest tile otherwise
  if (n >= 256 && mt * ((n + 255) / 256) >= sms) return launch_bn<256>(ma, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s);
  if (n >= 128 && mt * ((n + 127) / 128) >= sms) return launch_bn<128>(ma, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s);
  return launch_bn<64>(ma, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s);
}

}  // namespace qcf
