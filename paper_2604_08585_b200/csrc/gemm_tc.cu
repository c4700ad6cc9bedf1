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

constexpr int QCF_EPI_ROPE_QKV = 3;
// Stream-K for the 2-CTA kernel: OFF by default. Measured on B200 (tools/gemm_plans.py):
// the contiguous per-cluster k-ranges lose the L2 sharing of weight k-slices that
// the data-parallel schedule gets from clusters running the same n-tile in
// lockstep, and the owner's fix-up waits for clusters that finish last; at the
// fused-path shapes it was 5-60% slower. qcf_set_gemm_plan(+8) turns it on.
static int g_streamk = 0;
static int g_group_m = -1;  // raster group (m pairs) of the 2-CTA kernel; QCF_GEMM_GROUP env  // internal: RoPE + KV scatter epilogue of the QKV GEMM

struct EpiArgs {
  int kind, out_dtype;
  int b_tiled;  // B stored tile-major (64x64 tiles, 8 KB contiguous) -> 4D TMA boxes
  const int32_t* pos;
  const int32_t* dst;
  const float* cs_tbl;  // RoPE (cos, sin) pairs, float32 [n_pos][d/2][2]
  void* q_out;
  void* k_tab;
  void* v_tab;
  int h, hkv, d;
  int preload_w = 0;   // cluster split-K kernel: request the first weight k-blocks before the PDL wait
};

// fused epilogue for 32 consecutive columns of one output row
__device__ __forceinline__ void epilogue_row32(void* __restrict__ C, int64_t ldc, int row, int col0, int N,
                                               const uint32_t (&r)[32], const EpiArgs& ea) {
  const int epi = ea.kind, out_dtype = ea.out_dtype;
  if (epi == QCF_EPI_ROPE_QKV) {
    // C columns = [Q | K | V] of `h`/`hkv` heads x d; rotate Q and K pairs at
    // pos[row] (fusion.py:471-475), scatter K/V into table row dst[row] (477-478)
    const int qd = ea.h * ea.d, kd = ea.hkv * ea.d;
    int base;
    __nv_bfloat16* out;
    bool rot = true;
    if (col0 < qd) {
      base = col0;
      out = reinterpret_cast<__nv_bfloat16*>(ea.q_out) + (int64_t)row * qd + base;
    } else {
      const int64_t drow = ea.dst[row];
      if (col0 < qd + kd) {
        base = col0 - qd;
        out = reinterpret_cast<__nv_bfloat16*>(ea.k_tab) + drow * kd + base;
      } else {
        base = col0 - qd - kd;
        out = reinterpret_cast<__nv_bfloat16*>(ea.v_tab) + drow * kd + base;
        rot = false;
      }
    }
    const int half = ea.d >> 1;
    const int64_t t0 = (int64_t)ea.pos[row] * half + ((base % ea.d) >> 1);
    // 16 (cos, sin) pairs = 128 contiguous bytes: 8 vector loads, all issued up front
    float4 cs[8];
    if (rot) {
      const float4* src = reinterpret_cast<const float4*>(ea.cs_tbl + 2 * t0);
#pragma unroll
      for (int i = 0; i < 8; ++i) cs[i] = __ldg(src + i);
    }
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float e = __uint_as_float(r[2 * i]), o = __uint_as_float(r[2 * i + 1]);
      if (rot) {
        const float c = (i & 1) ? cs[i >> 1].z : cs[i >> 1].x, sn = (i & 1) ? cs[i >> 1].w : cs[i >> 1].y;
        const float oe = e * c - o * sn, oo = e * sn + o * c;
        e = oe;
        o = oo;
      }
      __nv_bfloat162 b2 = __floats2bfloat162_rn(e, o);
      pk[i] = *reinterpret_cast<uint32_t*>(&b2);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      reinterpret_cast<uint4*>(out)[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    return;
  }
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

// SKINNY (M <= 32): the A slab holds only 32 rows (4 KB) so the ring can be 16
// deep; the MMA still reads 128 A rows, the extra 96 are stale smem feeding
// output rows >= M that the epilogue never stores.
// SKINNY also moves 4 swizzle atoms (K=256) per stage, amortising the per-stage
// mbarrier round trips of the producer/MMA threads over 4x more weight bytes.

template <int BN, bool SKINNY = false>
struct TcCfg {
  static constexpr int KATOMS = SKINNY ? 4 : 1;   // 64-element K atoms per stage
  static constexpr int STAGES = SKINNY ? 4 : (BN == 256 ? 4 : (BN == 128 ? 6 : 8));
  static constexpr int A_ATOM = (SKINNY ? 32 : TC_BM) * TC_BK * 2;
  static constexpr int B_ATOM = BN * TC_BK * 2;
  static constexpr int A_BYTES = KATOMS * A_ATOM;
  static constexpr int B_BYTES = KATOMS * B_ATOM;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulators
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, bool SKINNY = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               void* __restrict__ C, int64_t ldc, int M, int N, int K, const EpiArgs ea, int splits,
               int a_box_rows, float* __restrict__ partial) {
  using Cfg = TcCfg<BN, SKINNY>;
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
  const int n_work = m_tiles * n_tiles * splits;
  constexpr int KSTAGE = TC_BK * Cfg::KATOMS;                 // K elements per stage
  const int k_blocks = (K + KSTAGE - 1) / KSTAGE;
  const int kb_per = (k_blocks + splits - 1) / splits;
  const uint32_t stage_tx = (uint32_t)Cfg::KATOMS * ((uint32_t)a_box_rows * TC_BK * 2 + Cfg::B_ATOM);
  // work unit w -> (m tile fastest, then split, then n tile); split sp covers
  // k blocks [sp*kb_per, min(k_blocks, (sp+1)*kb_per))
  auto unit = [&](int w, int& mb, int& nb, int& kb0, int& kb1) {
    mb = w % m_tiles;
    const int r = w / m_tiles;
    const int sp = r % splits;
    nb = r / splits;
    kb0 = sp * kb_per;
    kb1 = min(k_blocks, kb0 + kb_per);
  };

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
  pdl_wait();  // prologue above overlaps the previous kernel's tail
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      uint32_t it = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        int mb, nb, kb0, kb1;
        unit(w, mb, nb, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], stage_tx);
#pragma unroll
          for (int j = 0; j < Cfg::KATOMS; ++j) {
            tma_load_2d(sA + s * Cfg::A_BYTES + j * Cfg::A_ATOM, &map_a, &full[s], kb * KSTAGE + j * TC_BK, mb * TC_BM);
            if (ea.b_tiled)
              tma_load_4d(sB + s * Cfg::B_BYTES + j * Cfg::B_ATOM, &map_b, &full[s], 0, 0, kb * Cfg::KATOMS + j,
                          nb * (BN / 64));
            else
              tma_load_2d(sB + s * Cfg::B_BYTES + j * Cfg::B_ATOM, &map_b, &full[s], kb * KSTAGE + j * TC_BK, nb * BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (converged warp, elected lane)
      constexpr uint32_t idesc = idesc_bf16_f32(TC_BM, BN);
      uint32_t it = 0, t = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
        int mb, nb, kb0, kb1;
        unit(w, mb, nb, kb0, kb1);
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
#pragma unroll
          for (int j = 0; j < Cfg::KATOMS; ++j) {
            const uint64_t a0 = umma_desc_k_sw128(sA + s * Cfg::A_BYTES + j * Cfg::A_ATOM);
            const uint64_t b0 = umma_desc_k_sw128(sB + s * Cfg::B_BYTES + j * Cfg::B_ATOM);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 16; ++kk)  // +32 B per K=16 step inside the swizzle atom
              mma_bf16_e(d_tmem, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc,
                       (kb > kb0 || j || kk) ? 1u : 0u);
          }
          mma_commit_e(&empty[s]);
        }
        mma_commit_e(&tfull[acc]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5
    const int g = warp & 3;  // TMEM lane quarter this warp may access
    uint32_t t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      int mb, nb, kb0, kb1;
      unit(w, mb, nb, kb0, kb1);
      const int sp = (w / m_tiles) % splits;
      const int acc = t & 1;
      const int row = mb * TC_BM + g * 32 + lane;
      const bool row_ok = row < M;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * BN + cc * 32 + ((uint32_t)(g * 32) << 16), r);
        tmem_ld_wait();
        const int col0 = nb * BN + cc * 32;
        if (!row_ok || col0 >= N) continue;
        if (splits > 1)  // raw fp32 partial; qcf reduce applies the epilogue in a fixed order
          epilogue_row32(partial + (int64_t)sp * M * N, N, row, col0, N, r, EpiArgs{QCF_EPI_STORE, QCF_F32});
        else
          epilogue_row32(C, ldc, row, col0, N, r, ea);
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
// PM = the pair's M: 256 (each CTA 128 rows, one TMEM lane per row) or 128
// (each CTA 64 rows; the accumulator uses the "2x2" TMEM layout: lanes 0-63 hold
// columns [0, BN/2) of rows 0-63, lanes 64-127 columns [BN/2, BN) of the same
// rows -- BN/2 TMEM columns per accumulator). PM = 128 halves the row padding
// and doubles the unit count of small-M GEMMs (one request: M = 800).
template <int BN, int PM = 256>
struct Tc2Cfg {
  static constexpr int ROWS = PM / 2;                         // A rows per CTA
  static constexpr int STAGES = (PM == 256 && BN == 256) ? 6 : 8;
  static constexpr int A_BYTES = ROWS * TC_BK * 2;            // this CTA's rows
  static constexpr int B_BYTES = (BN / 2) * TC_BK * 2;        // this CTA's half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC_COLS = PM == 256 ? BN : BN / 2;    // TMEM columns per accumulator
  static constexpr int TMEM_COLS = 2 * ACC_COLS;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

// Stream-K (sk = 1): the pair's work is the contiguous range of global k-block
// iterations [c*T/P, (c+1)*T/P) over all (unit, k-block) pairs (T = units x
// k-blocks, P = clusters), so every cluster does the same number of MMAs and no
// wave is partially idle. A unit split across clusters is finished by the
// cluster that computed its FIRST k-blocks (it reaches them last, at the end of
// its range): later clusters spill their fp32 pieces to `sk_part` (one slot per
// CTA; a cluster spills at most its first segment) and raise a flag; the owner
// waits for the flags, adds the pieces in cluster order (deterministic), applies
// the epilogue and clears the flags for the next launch.
struct SegIter {
  int64_t g, g1;        // stream-K: global iteration range
  int u, u_stride, n_units, kb_units;
  bool sk;
  __device__ __forceinline__ bool next(int& unit, int& kb0, int& kb1) {
    if (sk) {
      if (g >= g1) return false;
      unit = (int)(g / kb_units);
      kb0 = (int)(g - (int64_t)unit * kb_units);
      { const int64_t e = (int64_t)kb0 + (g1 - g); kb1 = e < kb_units ? (int)e : kb_units; }
      g += kb1 - kb0;
      return true;
    }
    if (u >= n_units) return false;
    unit = u;
    kb0 = 0;
    kb1 = kb_units;
    u += u_stride;
    return true;
  }
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int BN, int PM = 256>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                void* __restrict__ C, int64_t ldc, int M, int N, int K, const EpiArgs ea, int sk,
                int* __restrict__ sk_flags, float* __restrict__ sk_part, int group_m) {
  using Cfg = Tc2Cfg<BN, PM>;
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
  const int m_pairs = (M + PM - 1) / PM;
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_pairs * n_tiles;
  const int k_blocks = (K + TC_BK - 1) / TC_BK;
  const int64_t T = (int64_t)n_work * k_blocks;
  // unit -> (m pair, n tile): m fastest inside groups of `group_m` m pairs, so a
  // wave of clusters covers a compact (group_m x ~clusters/group_m) block of the
  // output: both its A rows and its weight columns stay L2-resident
  const int gsz = min(group_m, m_pairs);
  auto coords = [&](int w, int& mp, int& nb) {
    const int grp = w / (gsz * n_tiles);
    const int first = grp * gsz;
    const int gm = min(gsz, m_pairs - first);
    const int idx = w - grp * gsz * n_tiles;
    mp = first + idx % gm;
    nb = idx / gm;
  };
  auto sk_start = [&](int c) -> int64_t { return (int64_t)c * T / n_clusters; };
  auto segs = [&]() {
    SegIter it;
    it.g = sk_start(cluster);
    it.g1 = sk_start(cluster + 1);
    it.u = cluster;
    it.u_stride = n_clusters;
    it.n_units = n_work;
    it.kb_units = k_blocks;
    it.sk = sk != 0;
    return it;
  };

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
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      uint32_t it = 0;
      SegIter sg = segs();
      int w, kbs, kbe;
      while (sg.next(w, kbs, kbe)) {
        int mp, nb;
        coords(w, mp, nb);
        const int arow = mp * PM + rank * Cfg::ROWS;
        const int brow = nb * BN + rank * (BN / 2);
        for (int kb = kbs; kb < kbe; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
          tma_load_2d_pair(sA + s * Cfg::A_BYTES, &map_a, &full[s], kb * TC_BK, arow);
          if (ea.b_tiled)
            tma_load_4d_pair(sB + s * Cfg::B_BYTES, &map_b, &full[s], 0, 0, kb, brow / 64);
          else
            tma_load_2d_pair(sB + s * Cfg::B_BYTES, &map_b, &full[s], kb * TC_BK, brow);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ---------------- MMA issuer (leader only; converged warp, elected lane)
      constexpr uint32_t idesc = idesc_bf16_f32(PM, BN);
      uint32_t it = 0, t = 0;
      SegIter sg = segs();
      int w, kbs, kbe;
      for (; sg.next(w, kbs, kbe); ++t) {
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * Cfg::ACC_COLS;
        for (int kb = kbs; kb < kbe; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (it / Cfg::STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a0 = umma_desc_k_sw128(sA + s * Cfg::A_BYTES);
          const uint64_t b0 = umma_desc_k_sw128(sB + s * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk)
            mma_bf16_pair_e(d_tmem, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc,
                          (kb > kbs || kk) ? 1u : 0u);
          mma_commit_pair_e(&empty[s]);
        }
        mma_commit_pair_e(&tfull[acc]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5 (both CTAs, own 128 rows)
    const int g = warp & 3;
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
    uint32_t t = 0;
    SegIter sg = segs();
    int w, kbs, kbe;
    const int et = threadIdx.x - 64;  // 0..127 within the epilogue warps
    for (; sg.next(w, kbs, kbe); ++t) {
      int mp, nb;
      coords(w, mp, nb);
      const int acc = t & 1;
      // row within this CTA's rows and first output column of this warp's TMEM half
      const int rt = PM == 256 ? g * 32 + lane : (g & 1) * 32 + lane;
      const int cbase = PM == 256 ? 0 : (g >> 1) * (BN / 2);
      const int row = mp * PM + rank * Cfg::ROWS + rt;
      const bool row_ok = row < M;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      if (kbs != 0) {
        // ---- a later piece of a split unit: spill the fp32 partial, raise the flag
        float* dst = sk_part + ((int64_t)(cluster * 2 + rank) * TC_BM + rt) * BN + cbase;
#pragma unroll 1
        for (int cc = 0; cc < Cfg::ACC_COLS / 32; ++cc) {
          uint32_t r[32];
          tmem_ld32(tmem_base + acc * Cfg::ACC_COLS + cc * 32 + ((uint32_t)(g * 32) << 16), r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg(reinterpret_cast<float4*>(dst + cc * 32 + j),
                   make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                               __uint_as_float(r[j + 3])));
        }
        tc_fence_before();
        mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) st_release(&sk_flags[cluster * 2 + rank], 1);
        continue;
      }
      // ---- owner (or whole unit): gather the later pieces of this unit, if any
      int c_last = cluster;
      if (kbe != k_blocks) {
        const int64_t unit_end = (int64_t)(w + 1) * k_blocks;
        while (c_last + 1 < n_clusters && sk_start(c_last + 1) < unit_end) ++c_last;
        if (et == 0)
          for (int c2 = cluster + 1; c2 <= c_last; ++c2)
            while (ld_acquire(&sk_flags[c2 * 2 + rank]) == 0) {}
        named_bar_sync(1, 128);
      }
#pragma unroll 1
      for (int cc = 0; cc < Cfg::ACC_COLS / 32; ++cc) {
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * Cfg::ACC_COLS + cc * 32 + ((uint32_t)(g * 32) << 16), r);
        tmem_ld_wait();
        for (int c2 = cluster + 1; c2 <= c_last; ++c2) {
          const float* src = sk_part + ((int64_t)(c2 * 2 + rank) * TC_BM + rt) * BN + cbase + cc * 32;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 p4 = __ldcg(reinterpret_cast<const float4*>(src + j));
            r[j] = __float_as_uint(__uint_as_float(r[j]) + p4.x);
            r[j + 1] = __float_as_uint(__uint_as_float(r[j + 1]) + p4.y);
            r[j + 2] = __float_as_uint(__uint_as_float(r[j + 2]) + p4.z);
            r[j + 3] = __float_as_uint(__uint_as_float(r[j + 3]) + p4.w);
          }
        }
        const int col0 = nb * BN + cbase + cc * 32;
        if (!row_ok || col0 >= N) continue;
        epilogue_row32(C, ldc, row, col0, N, r, ea);
      }
      tc_fence_before();
      mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      if (c_last > cluster) {  // every thread is done with the pieces: re-arm the flags
        named_bar_sync(1, 128);
        if (et == 0)
          for (int c2 = cluster + 1; c2 <= c_last; ++c2) sk_flags[c2 * 2 + rank] = 0;
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Swapped 2-CTA GEMM for mid-size M (the single request's ~800 recompute rows):
// the WEIGHT rows are the MMA's M side (256 per CTA pair, 128 per CTA) and the
// activation rows its N side, a runtime width BNA (multiple of 16, <= 256) chosen
// so the activation rows split into near-equal tiles: M = 800 runs as 4 x 208
// (4% padding) instead of 4 x 256 rows (28%). TMEM lanes = output columns, TMEM
// columns = activation rows, so the epilogue thread of lane n writes column n
// of 32 consecutive rows per tcgen05.ld (warp-coalesced along the row).
// Unit u -> (weight pair, activation tile) in bands of `gw` weight pairs: inside
// a band the weight pair runs fastest, so one wave of clusters covers a compact
// gw x (clusters / gw) block and every operand tile it reads is shared by the
// clusters of that wave through L2. gw = 1 is the plain order (activation tile
// fastest: each wave re-reads the WHOLE activation matrix from DRAM -- at the
// batch shape M = 6400, K = 14336 that is 183 MB per wave, 3.4x the
// algorithmic bytes, profiles/gemm_traffic.json).
__device__ __forceinline__ void swap_unit(int u, int n_wp, int n_act, int gw, int& wt, int& at) {
  const int per_band = gw * n_act;
  const int band = u / per_band, rem = u - band * per_band;
  const int bw = min(gw, n_wp - band * gw);   // the last band may be narrower
  wt = band * gw + rem % bw;
  at = rem / bw;
}

constexpr int SW_STAGES = 6;
constexpr int SW_A_BYTES = 128 * TC_BK * 2;  // this CTA's 128 weight rows
constexpr int SW_B_BYTES = 128 * TC_BK * 2;  // up to 128 activation rows (BNA / 2)
constexpr int SW_STAGE = SW_A_BYTES + SW_B_BYTES;
constexpr int SW_SMEM = SW_STAGES * SW_STAGE + 1024 + 256 + 4 * 32 * 33 * 4;  // + epilogue staging

__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc2s_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                 void* __restrict__ C, int64_t ldc, int M, int N, int K, const EpiArgs ea, int bna, int n_act,
                 int gw) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                // weights [stage]
  uint8_t* sB = smem + SW_STAGES * SW_A_BYTES;       // activations [stage]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SW_STAGES * SW_STAGE);
  uint64_t* empty = full + SW_STAGES;
  uint64_t* tfull = empty + SW_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2] (leader's copy is the one used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int n_wp = (N + 255) / 256;
  const int n_units = n_wp * n_act;
  const int k_blocks = (K + TC_BK - 1) / TC_BK;
  const int xrows = bna >> 1;  // activation rows per CTA

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < SW_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * 128); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const uint32_t stage_tx = 2 * (SW_A_BYTES + (uint32_t)xrows * 128);
      uint32_t it = 0;
      for (int u = cluster; u < n_units; u += n_clusters) {
        int wt, at;
        swap_unit(u, n_wp, n_act, gw, wt, at);
        const int wrow = wt * 256 + rank * 128;
        const int xrow = at * bna + rank * xrows;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % SW_STAGES;
          const uint32_t ph = (it / SW_STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], stage_tx);
          if (ea.b_tiled)
            tma_load_4d_pair(sA + s * SW_A_BYTES, &map_w, &full[s], 0, 0, kb, wrow / 64);
          else
            tma_load_2d_pair(sA + s * SW_A_BYTES, &map_w, &full[s], kb * TC_BK, wrow);
          tma_load_2d_pair(sB + s * SW_B_BYTES, &map_x, &full[s], kb * TC_BK, xrow);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ---------------- MMA issuer (leader only; converged warp, elected lane)
      const uint32_t idesc = idesc_bf16_f32(256, bna);
      uint32_t it = 0, t = 0;
      for (int u = cluster; u < n_units; u += n_clusters, ++t) {
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % SW_STAGES;
          const uint32_t ph = (it / SW_STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a0 = umma_desc_k_sw128(sA + s * SW_A_BYTES);
          const uint64_t b0 = umma_desc_k_sw128(sB + s * SW_B_BYTES);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk)
            mma_bf16_pair_e(d_tmem, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc, (kb | kk) ? 1u : 0u);
          mma_commit_pair_e(&empty[s]);
        }
        mma_commit_pair_e(&tfull[acc]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5: lane = output column -> transposed via smem
    // each tcgen05.ld gives lane n = column n of 32 consecutive rows; a padded 32 x 33
    // staging tile per warp turns that into lane = row with 32 contiguous columns, so
    // the row-per-thread epilogue (vector stores, in-register RoPE pairs) is reused
    // and the results are bit-identical to the normal orientation's
    const int g = warp & 3;
    float* stage = reinterpret_cast<float*>(smem + SW_STAGES * SW_STAGE + 256) + g * (32 * 33);  // after the barriers
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
    uint32_t t = 0;
    for (int u = cluster; u < n_units; u += n_clusters, ++t) {
      const int acc = t & 1;
      int wt, at;
      swap_unit(u, n_wp, n_act, gw, wt, at);
      const int col0 = wt * 256 + rank * 128 + g * 32;
      const int row0 = at * bna;
      const int rows = min(bna, M - row0);
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < rows; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * 256 + c0 + ((uint32_t)(g * 32) << 16), r);
        tmem_ld_wait();
        if (ea.kind != QCF_EPI_ROPE_QKV) {
          // store / ReLU / residual add: lane n holds column col0 + n of 32 consecutive
          // rows, so the warp writes each row's 32 columns in one coalesced access --
          // no shared-memory transpose (same per-element arithmetic: bit-identical)
          const int col = col0 + lane, nr = min(32, rows - c0);
          if (col < N) {
            if (ea.out_dtype == QCF_F32) {
              float* cp = reinterpret_cast<float*>(C) + (int64_t)(row0 + c0) * ldc + col;
              if (ea.kind == QCF_EPI_ADD_F32) {
                // all 32 residual loads first: interleaved with the stores they would be
                // serialised (the compiler cannot rule out ldc == 0 aliasing), one L2
                // round trip per row -- measured 119 us for W_o at M = 800 (ncu, 10% tensor)
                float res[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) res[j] = j < nr ? cp[(int64_t)j * ldc] : 0.f;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (j < nr) cp[(int64_t)j * ldc] = __uint_as_float(r[j]) + res[j];
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  if (j < nr) {
                    float v = __uint_as_float(r[j]);
                    if (ea.kind == QCF_EPI_RELU) v = fmaxf(v, 0.f);
                    cp[(int64_t)j * ldc] = v;
                  }
                }
              }
            } else {
              __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)(row0 + c0) * ldc + col;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (j < nr) {
                  float v = __uint_as_float(r[j]);
                  if (ea.kind == QCF_EPI_RELU) v = fmaxf(v, 0.f);
                  cp[(int64_t)j * ldc] = __float2bfloat16_rn(v);
                }
              }
            }
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) stage[j * 33 + lane] = __uint_as_float(r[j]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(stage[lane * 33 + j]);
        __syncwarp();
        if (lane < rows - c0 && col0 < N) epilogue_row32(C, ldc, row0 + c0 + lane, col0, N, r, ea);
      }
      tc_fence_before();
      mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
}

// epilogue of 4 consecutive columns [col, col+4) of one row from fp32 sums
// (split-K reductions): store / ReLU / residual add, or the QKV RoPE + scatter
// (4 columns = 2 interleaved pairs of one head)
__device__ __forceinline__ void epi_store4(void* __restrict__ C, int64_t ldc, int row, int col, float4 acc,
                                           const EpiArgs& ea) {
  const int epi = ea.kind, out_dtype = ea.out_dtype;
  if (epi == QCF_EPI_ROPE_QKV) {
    // columns [Q | K | V] (h / hkv heads x d); 4 columns = 2 interleaved pairs of one head
    const int qd = ea.h * ea.d, kd = ea.hkv * ea.d;
    __nv_bfloat16* out;
    int base;
    bool rot = true;
    if (col < qd) {
      base = col;
      out = reinterpret_cast<__nv_bfloat16*>(ea.q_out) + (int64_t)row * qd + base;
    } else {
      const int64_t drow = ea.dst[row];
      if (col < qd + kd) {
        base = col - qd;
        out = reinterpret_cast<__nv_bfloat16*>(ea.k_tab) + drow * kd + base;
      } else {
        base = col - qd - kd;
        out = reinterpret_cast<__nv_bfloat16*>(ea.v_tab) + drow * kd + base;
        rot = false;
      }
    }
    if (rot) {
      const int64_t t0 = (int64_t)ea.pos[row] * (ea.d >> 1) + ((base % ea.d) >> 1);
      const float4 cs = __ldg(reinterpret_cast<const float4*>(ea.cs_tbl + 2 * t0));
      const float c0 = cs.x, s0 = cs.y, c1 = cs.z, s1 = cs.w;
      const float x = acc.x * c0 - acc.y * s0, y = acc.x * s0 + acc.y * c0;
      const float z = acc.z * c1 - acc.w * s1, w = acc.z * s1 + acc.w * c1;
      acc = make_float4(x, y, z, w);
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
    *reinterpret_cast<uint2*>(out) = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    return;
  }
  if (out_dtype == QCF_F32) {
    float4* c = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + (int64_t)row * ldc + col);
    if (epi == QCF_EPI_ADD_F32) {
      const float4 o = *c;
      acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
    } else if (epi == QCF_EPI_RELU) {
      acc.x = fmaxf(acc.x, 0.f); acc.y = fmaxf(acc.y, 0.f); acc.z = fmaxf(acc.z, 0.f); acc.w = fmaxf(acc.w, 0.f);
    }
    *c = acc;
  } else {
    if (epi == QCF_EPI_RELU) {
      acc.x = fmaxf(acc.x, 0.f); acc.y = fmaxf(acc.y, 0.f); acc.z = fmaxf(acc.z, 0.f); acc.w = fmaxf(acc.w, 0.f);
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)row * ldc + col) =
        make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

// deterministic split-K reduction: C = epi(sum_s partial[s]) in split order.
// Epilogues: store / ReLU / residual add (f32 or bf16 C) and the fused QKV
// RoPE + KV scatter (the global-memory split-K fallback of the probe's projection: the rotation happens here,
// no separate rope kernel).
__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int splits, int M, int N,
                                     void* __restrict__ C, int64_t ldc, const EpiArgs ea) {
  pdl_wait();
  pdl_trigger();
  const int64_t total4 = (int64_t)M * N / 4;
  const int64_t mn = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = 4 * i;
    float4 acc = *reinterpret_cast<const float4*>(partial + e);
    for (int sp = 1; sp < splits; ++sp) {
      const float4 v = *reinterpret_cast<const float4*>(partial + sp * mn + e);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const int row = (int)(e / N), col = (int)(e - (int64_t)row * N);
    epi_store4(C, ldc, row, col, acc, ea);
  }
}

// ---------------------------------------------------------------------------
// Skinny GEMM (M <= 256: the probe's query rows, one request or a batch) as a
// weight stream with the split-K reduction inside a thread-block cluster. CTA
// (tile, split) of a cluster of S CTAs: 128 weight rows (the MMA's M side) x
// one of S equal k-ranges, the activation rows on the MMA's N side (NM = 32,
// 64, 128 or 256). Each CTA parks its fp32 partial [m][128] in its own shared
// memory (the drained stage ring); after a cluster barrier, CTA r sums slice r
// of the tile over the S partials in rank order through distributed shared
// memory (deterministic) and applies the epilogue -- no fp32 partials in HBM
// and no second kernel.
constexpr int SKC_A = 128 * TC_BK * 2;   // weight rows per stage
template <int NM>
struct SkcCfg {
  static constexpr int B = NM * TC_BK * 2;                    // activation rows per stage
  static constexpr int STAGES = NM <= 64 ? 4 : (NM == 128 ? 3 : 4);  // (5 at NM = 32: no gain)
  static constexpr int STAGE = SKC_A + B;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int OCC = NM <= 128 ? 2 : 1;               // CTAs per SM
  static_assert(NM * 128 * 4 <= STAGES * STAGE, "partial must fit in the ring");
};

__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

template <int NM>
__global__ void __launch_bounds__(TC_THREADS, SkcCfg<NM>::OCC)
gemm_skc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                void* __restrict__ C, int64_t ldc, int M, int N, int K, const EpiArgs ea) {
  using Cfg = SkcCfg<NM>;
  constexpr int SKC_STAGES = Cfg::STAGES, SKC_B = Cfg::B;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + SKC_STAGES * SKC_A;
  float* part = reinterpret_cast<float*>(smem);  // [NM][128], after the ring has drained
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SKC_STAGES * Cfg::STAGE);
  uint64_t* empty = full + SKC_STAGES;
  uint64_t* done = empty + SKC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank(), S = cluster_nctarank();
  const int tile = blockIdx.x / S;
  const int kbt = (K + TC_BK - 1) / TC_BK;
  const int kb0 = (int)(rank * kbt / S), kb1 = (int)((rank + 1) * kbt / S);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < SKC_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, NM);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the weights do not depend on the previous kernel: the first ring's worth of weight
  // k-blocks is requested before the PDL wait (only the activation rows wait for it)
  const int npre = ea.preload_w ? min(SKC_STAGES, kb1 - kb0) : 0;
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < npre; ++it) {
      const int kb = kb0 + it;
      mbar_expect_tx(&full[it], SKC_A + NM * 128);
      if (ea.b_tiled)
        tma_load_4d(sA + it * SKC_A, &map_w, &full[it], 0, 0, kb, tile * 2);
      else
        tma_load_2d(sA + it * SKC_A, &map_w, &full[it], kb * TC_BK, tile * 128);
    }
  }
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      for (int kb = kb0; kb < kb1; ++kb) {
        const int it = kb - kb0, s = it % SKC_STAGES;
        if (it >= npre) {
          mbar_wait(&empty[s], ((it / SKC_STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], SKC_A + NM * 128);
          if (ea.b_tiled)
            tma_load_4d(sA + s * SKC_A, &map_w, &full[s], 0, 0, kb, tile * 2);
          else
            tma_load_2d(sA + s * SKC_A, &map_w, &full[s], kb * TC_BK, tile * 128);
        }
        tma_load_2d(sB + s * SKC_B, &map_x, &full[s], kb * TC_BK, 0);
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (converged warp, elected lane)
      constexpr uint32_t idesc = idesc_bf16_f32(128, NM);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int it = kb - kb0, s = it % SKC_STAGES;
        mbar_wait(&full[s], (it / SKC_STAGES) & 1);
        tc_fence_after();
        const uint64_t a0 = umma_desc_k_sw128(sA + s * SKC_A);
        const uint64_t b0 = umma_desc_k_sw128(sB + s * SKC_B);
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)
          mma_bf16_e(tmem, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc, (kb > kb0 || kk) ? 1u : 0u);
        mma_commit_e(&empty[s]);
      }
      mma_commit_e(done);  // also fires when this split has no k-blocks
    }
  } else {  // ---------------- warps 2..5: TMEM partial -> shared memory [m][n]
    const int g = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < NM; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + c0 + ((uint32_t)(g * 32) << 16), r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) part[(c0 + j) * 128 + g * 32 + lane] = kb1 > kb0 ? __uint_as_float(r[j]) : 0.f;
    }
  }
  tc_fence_before();
  cluster_sync();  // every partial of the tile is in its CTA's shared memory
  // ---------------- CTA r: slice r of the tile's float4 groups, summed in rank order
  const int G = M * 32;  // float4 groups: M rows x 128 columns / 4
  const int g0 = (int)(rank * G / S), g1 = (int)((rank + 1) * G / S);
  for (int gi = g0 + (int)threadIdx.x; gi < g1; gi += blockDim.x) {
    const int m = gi >> 5, n4 = (gi & 31) * 4;
    const uint32_t off = smem_u32(part + m * 128 + n4);
    float4 acc = ld_dsmem_f4(map_to_rank_addr(off, 0));
    for (uint32_t s2 = 1; s2 < S; ++s2) {
      const float4 v = ld_dsmem_f4(map_to_rank_addr(off, s2));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const int col = tile * 128 + n4;
    if (col < N) epi_store4(C, ldc, m, col, acc, ea);
  }
  cluster_sync();  // the peers are done reading this CTA's partial
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, NM);
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

// B operand map: row-major [n][k] (2D) or tile-major [n/64][k/64][64][64] (4D),
// box of `box_rows` rows x 64 k
static int make_b_map(CUtensorMap* map, const void* ptr, int64_t n, int64_t k, int64_t ld, int box_rows,
                      int tiled) {
  if (!tiled) return make_kmajor_map(map, ptr, n, k, ld, box_rows);
  EncodeTiledFn enc = get_encode();
  QCF_REQUIRE(enc, QCF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  QCF_REQUIRE(n % 64 == 0 && k % 64 == 0 && box_rows % 64 == 0, QCF_EUNSUPPORTED, "tiled B needs n, k % 64 == 0");
  cuuint64_t dims[4] = {64, 64, (cuuint64_t)(k / 64), (cuuint64_t)(n / 64)};
  cuuint64_t strides[3] = {128, 8192, (cuuint64_t)(k / 64) * 8192};
  cuuint32_t box[4] = {64, 64, 1, (cuuint32_t)(box_rows / 64)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QCF_REQUIRE(r == CUDA_SUCCESS, QCF_ECUDA, "cuTensorMapEncodeTiled(4D) failed (%d)", (int)r);
  return QCF_OK;
}

// batched variant: [batch][rows][k] with a batch stride (elements), box {64, box_rows, 1}
int make_kmajor_map3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld, int box_rows,
                     int64_t batch, int64_t batch_stride) {
  EncodeTiledFn enc = get_encode();
  QCF_REQUIRE(enc, QCF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)k, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(batch_stride * 2)};
  cuuint32_t box[3] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QCF_REQUIRE(r == CUDA_SUCCESS, QCF_ECUDA, "cuTensorMapEncodeTiled(3D) failed (%d)", (int)r);
  return QCF_OK;
}

// generic bf16 map, SWIZZLE_128B, rank 2..5 (strides in bytes for dims 1..rank-1)
int make_map_bf16(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                  const uint32_t* box) {
  EncodeTiledFn enc = get_encode();
  QCF_REQUIRE(enc, QCF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  QCF_REQUIRE(rank >= 2 && rank <= 5, QCF_EINVAL, "make_map_bf16: bad rank");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], estr[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    estr[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank, const_cast<void*>(ptr), d, st, b, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QCF_REQUIRE(r == CUDA_SUCCESS, QCF_ECUDA, "cuTensorMapEncodeTiled(rank %d) failed (%d)", rank, (int)r);
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

template <int BN, bool SKINNY = false>
static int launch_bn(const CUtensorMap& ma, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                     int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s, int splits = 1,
                     int a_box_rows = TC_BM, float* partial = nullptr) {
  using Cfg = TcCfg<BN, SKINNY>;
  CUtensorMap mb;
  int st = make_b_map(&mb, b, n, k, ldb, BN, ea.b_tiled);
  if (st != QCF_OK) return st;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, SKINNY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc attr");
    attr_set = true;
  }
  const int64_t work = ((m + TC_BM - 1) / TC_BM) * ((n + BN - 1) / BN) * splits;
  const int grid = (int)std::min<int64_t>(work, sm_count());
  QCF_LAUNCH("gemm_tc_kernel", gemm_tc_kernel<BN, SKINNY>, dim3(grid), dim3(TC_THREADS), Cfg::SMEM, s, ma, mb, c, ldc, (int)m, (int)n, (int)k, ea,
                                                                 splits, a_box_rows, partial);
  QCF_LAUNCH_CHECK("qcf_gemm(tcgen05)");
  if (splits > 1) {
    const int64_t total4 = m * n / 4;
    const int rg = (int)std::min<int64_t>((total4 + 255) / 256, 4 * sm_count());
    QCF_LAUNCH("splitk_reduce_kernel", splitk_reduce_kernel, dim3(rg), dim3(256), 0, s, partial, splits, (int)m, (int)n, c, ldc, ea);
    QCF_LAUNCH_CHECK("qcf_gemm(split-k reduce)");
  }
  return QCF_OK;
}

// stream-K workspace: [flags: 4 KB][fp32 partial 128x256 per CTA of the grid]
static size_t sk_bytes() { return 4096 + (size_t)(sm_count() & ~1) * TC_BM * 256 * sizeof(float); }

template <int BN, int PM = 256>
static int launch_pair(const CUtensorMap& ma, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                       int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s, void* ws = nullptr,
                       size_t ws_bytes = 0) {
  CUtensorMap mb;
  int st = make_b_map(&mb, b, n, k, ldb, BN / 2, ea.b_tiled);
  if (st != QCF_OK) return st;
  // the caller's A map has a box of Tc2Cfg<BN, PM>::ROWS rows (this CTA's rows of the tile)
  const CUtensorMap& ma_pair = ma;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2_kernel<BN, PM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Tc2Cfg<BN, PM>::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc2 attr");
    attr_set = true;
  }
  if (g_group_m < 0) {
    const char* e = getenv("QCF_GEMM_GROUP");
    g_group_m = e ? atoi(e) : 0;
  }
  const int64_t work = ((m + PM - 1) / PM) * ((n + BN - 1) / BN);
  const int64_t iters = work * ((k + TC_BK - 1) / TC_BK);
  // stream-K when the caller's workspace holds the flags + partials and the unit
  // count does not fill whole waves of clusters
  const int sk = (ws && ws_bytes >= sk_bytes() && g_streamk && (work % (sm_count() / 2)) != 0 &&
                  iters >= 8 * (sm_count() / 2)) ? 1 : 0;
  const int clusters = sk ? sm_count() / 2 : (int)std::min<int64_t>(work, sm_count() / 2);
  int* sk_flags = sk ? reinterpret_cast<int*>(ws) : nullptr;
  float* sk_part = sk ? reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + 4096) : nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Tc2Cfg<BN, PM>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  // raster band of m pairs (QCF_GEMM_GROUP overrides): the fewest equal bands whose A
  // rows (PM x K bf16 per pair) stay under 32 MB, so a band's activations remain in L2
  // while every weight tile streams past them once per band -- the batch QKV / W1 (25
  // pairs, K = 4096) run as 13 + 12: DRAM reads 518 -> 291 MB and 493 -> 312 MB per
  // launch, 453 -> 436 and 509 -> 492 us (ncu, profiles/r2s3_gemm_group_ab.txt). With
  // all 25 pairs in one band the 157-183 MB of outputs pushed the 52 MB of A out of
  // L2 between waves.
  const int64_t m_pairs = (m + PM - 1) / PM;
  const int64_t max_g = std::max<int64_t>(1, (int64_t)(32e6 / ((double)PM * (double)k * 2.0)));
  const int64_t bands = (m_pairs + max_g - 1) / max_g;
  const int group_m = g_group_m > 0 ? g_group_m : (int)((m_pairs + bands - 1) / bands);
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<BN, PM>, ma_pair, mb, c, ldc, (int)m, (int)n, (int)k, ea, sk, sk_flags,
                                     sk_part, group_m);
  if (e != cudaSuccess) return cuda_status(e, "qcf_gemm(tcgen05 pair)");
  QCF_LAUNCH_CHECK("qcf_gemm(tcgen05 pair)");
  return QCF_OK;
}

// swapped 2-CTA kernel: activation tile width (multiple of 16, <= 256) and count
// minimising waves x (width + 256), the shared-memory traffic of a k-block in
// 128-byte rows: per CTA the TMA writes and the MMA reads the 128 weight rows and
// width/2 activation rows, 2 x (128 + width/2) rows against the SM's ~128 B/clk,
// which exceeds the MMA's own 2 x width cycles for every width < 256 (ncu, M = 800:
// the tensor pipe ~66% active; tools/mma_bench.cu). Same units as pair_cost.
// (The former waves x (width + 24) model picked 6 x 144 rows for the M = 800 QKV
// instead of 4 x 208.)
// (tiles narrower than 128 activation rows stream too many weight bytes per flop:
// at M = 256 the 64-wide plan measured slower than 1-CTA 128 x 64 tiles)
static double swap_overhead() {   // QCF_SWAP_OVH: the model's per-k-block constant (measurement)
  static int ovh = -1;
  if (ovh < 0) {
    const char* e = getenv("QCF_SWAP_OVH");
    ovh = e ? std::max(0, atoi(e)) : 256;
  }
  return (double)ovh;
}
static double swap_plan(int64_t m, int64_t n, int& bna, int& n_act, int min_w = 128) {
  const int64_t clusters = sm_count() / 2, wp = (n + 255) / 256;
  static int force_na = -1;   // QCF_SWAP_NA: force the activation tile count (measurement)
  if (force_na < 0) {
    const char* e = getenv("QCF_SWAP_NA");
    force_na = e ? std::max(0, atoi(e)) : 0;
  }
  if (force_na > 0) {
    const int64_t w = ((m + force_na - 1) / force_na + 15) / 16 * 16;
    if (w <= 256) {
      bna = (int)w;
      n_act = force_na;
      return 0.0;
    }
  }
  double best = 1e30;
  for (int64_t na = (m + 255) / 256; na <= (m + 255) / 256 + 8; ++na) {
    const int64_t w = ((m + na - 1) / na + 15) / 16 * 16;
    if (w > 256 || w < std::min<int64_t>(min_w, (m + 15) / 16 * 16)) continue;
    const int64_t units = wp * na;
    const double cost = (double)((units + clusters - 1) / clusters) * (double)(w + swap_overhead());
    if (cost < best - 1e-9) {
      best = cost;
      bna = (int)w;
      n_act = (int)na;
    }
  }
  return best;
}
static double pair_cost(int64_t m, int64_t n) {
  const int64_t clusters = sm_count() / 2, units = ((m + 255) / 256) * ((n + 255) / 256);
  return (double)((units + clusters - 1) / clusters) * (256.0 + swap_overhead());
}

static int launch_swap(const void* a, int64_t lda, const void* w, int64_t ldb, void* c, int64_t ldc, int64_t m,
                       int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s, int bna, int n_act) {
  CUtensorMap mw, mx;
  int st = make_b_map(&mw, w, n, k, ldb, 128, ea.b_tiled);
  if (st != QCF_OK) return st;
  st = make_kmajor_map(&mx, a, m, k, lda, bna / 2);
  if (st != QCF_OK) return st;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SW_SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc2s attr");
    attr_set = true;
  }
  const int64_t units = ((n + 255) / 256) * n_act;
  const int clusters = (int)std::min<int64_t>(units, sm_count() / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = SW_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  // band width: about sqrt(clusters) weight pairs (8 on 74 clusters); QCF_SWAP_GROUP overrides (1 = plain order)
  static int g_swap_group = -1;
  if (g_swap_group < 0) {
    const char* env = getenv("QCF_SWAP_GROUP");
    g_swap_group = env ? std::max(1, atoi(env)) : 0;
  }
  const int n_wp = (int)((n + 255) / 256);
  // activations that fit in L2 with room to spare (one request's ~800 rows) keep the plain
  // order: every wave then shares the whole activation matrix from L2 (banding measured
  // +1% TTFT there); the batch's 6400-row operands are banded
  const bool big = (double)m * (double)k * 2.0 > 48e6;
  // all weight pairs in one band when the whole weight matrix fits in L2 beside the wave's
  // activation slabs (the batch W_o, 4096 x 4096: DRAM 253 -> 223 MB per launch, ncu)
  const bool w_fits = (double)n * (double)k * 2.0 <= 40e6;
  int gw = g_swap_group > 0 ? g_swap_group
                            : (big ? (w_fits ? n_wp : (int)std::lround(std::sqrt((double)clusters))) : 1);
  gw = std::max(1, std::min(gw, n_wp));
  // (L2 priority hints -- evict_last on the band's weights, evict_first on the
  // activations -- were measured WORSE: 1909 vs 1047 MB at W2, since the wave's
  // clusters share each activation k-slab through L2; tools/gemm_hint_ab.sh)
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc2s_kernel, mw, mx, c, ldc, (int)m, (int)n, (int)k, ea, bna, n_act,
                                     gw);
  if (e != cudaSuccess) return cuda_status(e, "qcf_gemm(tcgen05 swapped pair)");
  QCF_LAUNCH_CHECK("qcf_gemm(tcgen05 swapped pair)");
  return QCF_OK;
}

static int g_swap_mode = -1;  // QCF_GEMM_SWAP env: 0 off, 1 on (default on)
static int g_pair_mode = -1;  // QCF_GEMM_PAIR env: 0 off, 1 on (default on)
static int g_gemm_plan = 0;   // qcf_set_gemm_plan: 0 auto, 1 pair/256, 2 one/256, 3 one/128, 4 one/64, 5 pair-128-rows,
                              // 6 pair/128 (256 x 128 tiles, measured slower), 7 swapped pair

void set_gemm_plan(int p) {
  g_streamk = (p & 8) ? 1 : 0;  // +8: stream-K on (measurement)
  p &= 7;
  g_gemm_plan = (p >= 0 && p <= 7) ? p : 0;
}

// Skinny-M (probe) plan: BN=64 tiles, split K until ~2 waves of CTAs stream the
// weights; A box trimmed to the live rows. Returns splits (1 = no workspace).
// Split count: the one whose unit count (tiles x splits) fills whole waves of
// SMs best (each unit streams >= 2 stages of weights); ties -> fewer splits.
// (An in-kernel "last split reduces" variant measured slower than the separate
// deterministic reduce kernel: the last CTA's serial partial reads stall its
// epilogue warps.)
static int skinny_splits(int64_t m, int64_t n, int64_t k) {
  if (m > 32) return 1;
  const int64_t tiles = (n + 63) / 64, kb = (k + 4 * TC_BK - 1) / (4 * TC_BK);
  const int64_t sms = sm_count();
  int best = 1;
  double best_eff = -1.0;
  for (int sp = 1; sp <= 16; ++sp) {
    const int64_t kb_per = (kb + sp - 1) / sp;
    if (kb_per < 2 || (sp - 1) * kb_per >= kb) continue;  // every split gets >= 1 k block
    const int64_t units = tiles * sp;
    const double eff = (double)units / (double)(((units + sms - 1) / sms) * sms);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = sp;
    }
  }
  return best;
}

// [stream-K flags + partials][skinny split-K partials]
size_t gemm_workspace_bytes(int64_t m, int64_t n, int64_t k) {
  const int sp = skinny_splits(m, n, k);
  return sk_bytes() + (sp > 1 ? (size_t)sp * m * n * sizeof(float) : 0);
}

static int gemm_tc_skinny_ea(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                             int64_t n, int64_t k, const EpiArgs& ea, void* ws, size_t ws_bytes, cudaStream_t s);

int gemm_tc_skinny(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                   int64_t n, int64_t k, int epilogue, int out_dtype, int b_layout, void* ws, size_t ws_bytes,
                   cudaStream_t s) {
  return gemm_tc_skinny_ea(a, lda, b, ldb, c, ldc, m, n, k, EpiArgs{epilogue, out_dtype, b_layout}, ws, ws_bytes, s);
}

// cluster split-K skinny launch (M <= 256): S CTAs per 128 weight rows (<= 8, the
// portable cluster size). S from a cold-L2 sweep at M = 32 (tools/gemm_plans.py,
// QCF_SKC_S): ~1.5 CTAs per SM is best (QKV 96 tiles: S = 2 28 us vs S = 3 36 us;
// the o / down projections' 32 tiles: S = 6-8); a cluster's CTAs never share an
// SM, which caps the co-resident clusters well below 2 CTAs/SM worth.
static int g_skinny_cl = -1;  // QCF_SKINNY_CL env: 0 -> the global-memory split-K path (M <= 32)
static int g_skc_max_m = 256;
static int g_skc_splits = 0;  // QCF_SKC_S: forced cluster size (measurement)
template <int NM>
static int launch_skc_nm(const CUtensorMap& mw, const void* a, int64_t lda, void* c, int64_t ldc, int64_t m,
                         int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s) {
  using Cfg = SkcCfg<NM>;
  const int64_t tiles = (n + 127) / 128, kbt = (k + TC_BK - 1) / TC_BK;
  // CTAs in flight: ~1.5 per SM at 2 CTAs/SM; just under one wave at 1 CTA/SM (M = 256:
  // the down projection's 32 tiles x 4 = 128 CTAs, 63 -> 40 us cold)
  const int64_t target = Cfg::OCC == 2 ? sm_count() * 3 / 2 : sm_count() * 7 / 8;
  int S = (int)std::max<int64_t>(1, std::min<int64_t>(8, (target + tiles / 2) / tiles));
  if (g_skc_splits > 0) S = g_skc_splits;
  S = (int)std::max<int64_t>(1, std::min<int64_t>(S, kbt));
  CUtensorMap mx;
  int st = make_kmajor_map(&mx, a, m, k, lda, NM);
  if (st != QCF_OK) return st;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_skc_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm_skc attr");
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles * S));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  static int preload = -1;   // QCF_SKC_PRELOAD=0: no weight loads before the PDL wait
  if (preload < 0) {
    const char* e = getenv("QCF_SKC_PRELOAD");
    preload = e ? atoi(e) : 1;
  }
  EpiArgs ep = ea;
  ep.preload_w = preload;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_skc_kernel<NM>, mw, mx, c, ldc, (int)m, (int)n, (int)k, ep);
  if (e != cudaSuccess) return cuda_status(e, "qcf_gemm(tcgen05 cluster split-K)");
  QCF_LAUNCH_CHECK("qcf_gemm(tcgen05 cluster split-K)");
  return QCF_OK;
}

static int launch_skc(const void* a, int64_t lda, const void* w, int64_t ldb, void* c, int64_t ldc, int64_t m,
                      int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s) {
  if (m > g_skc_max_m || (n % 4) || (k % 8) || (lda % 8) || (ldb % 8) || ((uintptr_t)a & 15) || ((uintptr_t)w & 15))
    return QCF_EUNSUPPORTED;
  // M > 64: every 128-row weight tile re-reads all M activation rows (2x the weight
  // bytes at M = 256) through L2 into one CTA per SM; that only pays off when the
  // tiles x splits fit one wave (N <= 4096: the down projection 63 -> 40 us cold,
  // QKV / up measured 1.4-1.9x slower than the 2-CTA / 1-CTA tiles)
  if (m > 64 && n > 4096) return QCF_EUNSUPPORTED;
  if (ea.kind != QCF_EPI_ROPE_QKV && ((ldc % 4) || ((uintptr_t)c & 15))) return QCF_EUNSUPPORTED;
  CUtensorMap mw;
  int st = make_b_map(&mw, w, n, k, ldb, 128, ea.b_tiled);
  if (st != QCF_OK) return st;
  if (m <= 32) return launch_skc_nm<32>(mw, a, lda, c, ldc, m, n, k, ea, s);
  if (m <= 64) return launch_skc_nm<64>(mw, a, lda, c, ldc, m, n, k, ea, s);
  if (m <= 128) return launch_skc_nm<128>(mw, a, lda, c, ldc, m, n, k, ea, s);
  return launch_skc_nm<256>(mw, a, lda, c, ldc, m, n, k, ea, s);
}

static int gemm_tc_skinny_ea(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                             int64_t n, int64_t k, const EpiArgs& ea, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (g_skinny_cl < 0) {
    const char* e = getenv("QCF_SKINNY_CL");
    g_skinny_cl = (e && e[0] == '0') ? 0 : 1;
    const char* mm = getenv("QCF_SKC_MAX_M");  // measurement knob: largest M on the cluster path
    if (mm) g_skc_max_m = atoi(mm);
    const char* ss = getenv("QCF_SKC_S");
    if (ss) g_skc_splits = atoi(ss);
  }
  if (g_skinny_cl) {
    const int st = launch_skc(a, lda, b, ldb, c, ldc, m, n, k, ea, s);
    if (st != QCF_EUNSUPPORTED) return st;
  }
  const int sp = skinny_splits(m, n, k);
  if (sp <= 1 || ws_bytes < gemm_workspace_bytes(m, n, k) || (n % 4) || ((uintptr_t)ws & 15)) return QCF_EUNSUPPORTED;
  if ((k % 8) || (lda % 8) || (ldb % 8) || ((uintptr_t)a & 15) || ((uintptr_t)b & 15)) return QCF_EUNSUPPORTED;
  if (ea.kind != QCF_EPI_ROPE_QKV && ((ldc % 4) || ((uintptr_t)c & 15))) return QCF_EUNSUPPORTED;
  const int box = (int)((m + 15) / 16 * 16);
  CUtensorMap ma;
  int st = make_kmajor_map(&ma, a, m, k, lda, box);
  if (st != QCF_OK) return st;
  return launch_bn<64, true>(ma, b, ldb, c, ldc, m, n, k, ea, s, sp, box,
                             reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + sk_bytes()));
}

static int gemm_tc_launch_ea(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc,
                             int64_t m, int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s, void* ws,
                             size_t ws_bytes);

int gemm_tc_launch(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int64_t m,
                   int64_t n, int64_t k, int epilogue, int out_dtype, cudaStream_t s, int b_layout, void* ws,
                   size_t ws_bytes) {
  return gemm_tc_launch_ea(a, lda, b, ldb, c, ldc, m, n, k, EpiArgs{epilogue, out_dtype, b_layout}, s, ws, ws_bytes);
}

int gemm_qkv_rope_launch(const void* a, int64_t lda, const void* w, int64_t ldb, int64_t m, int64_t k, int h,
                         int hkv, int d, const int32_t* pos, const int32_t* dst, const float* cs_tbl,
                         void* q_out, void* k_tab, void* v_tab, cudaStream_t s,
                         int b_layout, void* ws, size_t ws_bytes) {
  if (d % 32) return QCF_EUNSUPPORTED;  // 32-column epilogue chunks must stay inside a head
  if (((uintptr_t)q_out | (uintptr_t)k_tab | (uintptr_t)v_tab | (uintptr_t)cs_tbl) & 15) return QCF_EUNSUPPORTED;
  EpiArgs ea{QCF_EPI_ROPE_QKV, QCF_BF16, b_layout, pos, dst, cs_tbl, q_out, k_tab, v_tab, h, hkv, d};
  const int64_t n = (int64_t)(h + 2 * hkv) * d;
  void* dummy_c = q_out;  // C is not written by this epilogue
  if (m <= 256) {  // the probe's q rows: split-K weight streaming, RoPE + scatter applied in the reduction
    const int st = gemm_tc_skinny_ea(a, lda, w, ldb, dummy_c, n, m, n, k, ea, ws, ws_bytes, s);
    if (st != QCF_EUNSUPPORTED) return st;
  }
  return gemm_tc_launch_ea(a, lda, w, ldb, dummy_c, n, m, n, k, ea, s, ws, ws_bytes);
}

static int gemm_tc_launch_ea(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc,
                             int64_t m, int64_t n, int64_t k, const EpiArgs& ea, cudaStream_t s, void* ws,
                             size_t ws_bytes) {
  const int out_dtype = ea.out_dtype;
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
  switch (g_gemm_plan) {  // forced plan (tuning / measurement)
    case 1: if (m >= 192 && n >= 256) return launch_pair<256>(ma, b, ldb, c, ldc, m, n, k, ea, s, ws, ws_bytes); break;
    case 2: if (n >= 256) return launch_bn<256>(ma, b, ldb, c, ldc, m, n, k, ea, s); break;
    case 3: if (n >= 128) return launch_bn<128>(ma, b, ldb, c, ldc, m, n, k, ea, s); break;
    case 4: return launch_bn<64>(ma, b, ldb, c, ldc, m, n, k, ea, s);
    case 5:
      if (m >= 96 && n >= 256) {
        CUtensorMap ma64;
        st = make_kmajor_map(&ma64, a, m, k, lda, 64);
        if (st != QCF_OK) return st;
        return launch_pair<256, 128>(ma64, b, ldb, c, ldc, m, n, k, ea, s, ws, ws_bytes);
      }
      break;
    case 6: if (m >= 192 && n >= 128) return launch_pair<128>(ma, b, ldb, c, ldc, m, n, k, ea, s, ws, ws_bytes); break;
    case 7:
      if (n >= 256) {
        int bna = 0, na = 0;
        swap_plan(m, n, bna, na, 16);
        if (bna) return launch_swap(a, lda, b, ldb, c, ldc, m, n, k, ea, s, bna, na);
      }
      break;
    default: break;
  }
  if (g_swap_mode < 0) {
    const char* e = getenv("QCF_GEMM_SWAP");
    g_swap_mode = (e && e[0] == '0') ? 0 : 1;
  }
  // swapped pairs when the activation rows pad badly into 256-row pairs (M ~ 800:
  // 4 x 208 vs 4 x 256 rows) or their tiles fill the waves better. The epilogue is
  // the row-per-thread one behind a shared-memory transpose, so every epilogue
  // (RoPE included) is bit-identical to the normal orientation (same MMA k order,
  // same rounding): the plan choice never changes a result.
  if (g_swap_mode && g_pair_mode && m >= 64 && n >= 256 && n % 32 == 0) {
    int bna = 0, na = 0;
    const double cs = swap_plan(m, n, bna, na);
    if (bna && cs < 0.97 * pair_cost(m, n) && (n + 255) / 256 * na >= sms / 4)
      return launch_swap(a, lda, b, ldb, c, ldc, m, n, k, ea, s, bna, na);
  }
  // 2-CTA 256-row tiles vs 1-CTA 128-row tiles: estimate each one's useful
  // fraction (wave quantisation x row padding; 1-CTA pays ~15% for its
  // shallower TMA lookahead) and take the better one
  // (2-CTA pairs of 128 rows -- plan 5 -- halve the row padding of small M and double
  // the unit count, but each SM then streams 1.5x the operand bytes per flop: measured
  // 10-20% slower than the 256-row pairs at M = 800 (tools/gemm_plans.py), so the
  // automatic choice is between 256-row pairs and 1-CTA tiles)
  if (g_pair_mode && m >= 192 && n >= 256) {
    const int64_t clusters = sms / 2, nt = (n + 255) / 256;
    auto eff = [&](int64_t units, int64_t rows_padded) {
      return (double)units / (double)(((units + clusters - 1) / clusters) * clusters) * (double)m /
             (double)rows_padded;
    };
    const int64_t mps = (m + 255) / 256;
    const double e_pair = eff(mps * nt, mps * 256);
    const int64_t t1 = mt * nt;
    const double e_one = 0.85 * (double)t1 / (double)(((t1 + sms - 1) / sms) * sms) * (double)m / (double)(mt * 128);
    if (mps * nt >= clusters / 2 && e_pair >= e_one)
      return launch_pair<256>(ma, b, ldb, c, ldc, m, n, k, ea, s, ws, ws_bytes);
  }
  // tile width: enough tiles to cover the SMs, widest tile otherwise
  if (n >= 256 && mt * ((n + 255) / 256) >= sms) return launch_bn<256>(ma, b, ldb, c, ldc, m, n, k, ea, s);
  if (n >= 128 && mt * ((n + 127) / 128) >= sms) return launch_bn<128>(ma, b, ldb, c, ldc, m, n, k, ea, s);
  return launch_bn<64>(ma, b, ldb, c, ldc, m, n, k, ea, s);
}

}  // namespace qcf
