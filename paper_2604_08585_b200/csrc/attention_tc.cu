// Location-aware attention on the 5th-gen tensor cores (fusion.py:194-208 /
// model.py:326-338 with the "key position <= row position" mask of
// fusion.py:467): row i of a 128-row query tile sees table rows 0..kmax[i].
//
// One CTA = (128 query rows, one head). Warp roles:
//   warp 0      TMA producer: Q tile once, then K/V tiles of 128 keys (2-stage ring)
//   warp 1      MMA issuer:   S_j = Q.K_j^T into a double-buffered TMEM S, then
//                             O += P_{j-1}.V_{j-1} (V read MN-major straight from
//                             the token-major table: no transpose pass)
//   warps 2..17 softmax:      16 warps = 4 TMEM lane quarters (rows) x 4 column
//                             groups of 32 keys; each thread owns 32 scores of one
//                             row (one tcgen05.ld), row max combined through smem,
//                             ex2 with a lazily-updated reference max (O in TMEM is
//                             rescaled only when the running max grows by > 2^8),
//                             P -> SW128 smem, final O / l per 32-column slice.
// Query rows arrive sorted by position (selection is ascending), so a tile's
// key range is [0, max kmax] and only its tail tiles are partially masked.
#include <cuda.h>
#include <stdlib.h>

#include "attention.cuh"
#include "sm100.cuh"

namespace qcf {

using namespace sm100;

int make_kmajor_map3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld, int box_rows,
                     int64_t batch, int64_t batch_stride);

constexpr int AT_BM = 128, AT_BN = 128, AT_D = 128;
constexpr int AT_THREADS = 576;  // 2 control warps + 16 softmax warps
constexpr int AT_TILE_BYTES = AT_BM * AT_D * 2;  // 32 KB: two 16 KB SW128 atoms
// K / V ring depths of the single-tile kernel (Q + 5 tiles fit the 227 KB budget).
// Traced (tools/attn_trace.py): with a 2-deep K ring the tensor pipe idled ~900
// cycles per key tile waiting for K_{j+2}'s TMA (a K tile is 128 rows x 256 B
// strided by the table row, ~1.5 us from HBM); separate producer lanes for K and V
// keep a V wait from delaying the next K load
constexpr int AT_KS = 3;
constexpr int AT_VS = 2;
constexpr int AT_ONES_BYTES = 16 * AT_BN * 2;  // bf16 ones, 16 x 128 K-major: B operand of the row-sum MMA
constexpr int AT_SMEM = AT_TILE_BYTES * (1 + AT_KS + AT_VS) + AT_ONES_BYTES + 1024 + 256;  // Q, K, V, ones

// MN-major SW128 descriptor (B = V: N = head dim contiguous, K = keys):
// 8-key groups 1024 B apart (SBO), 64-column atoms 16 KB apart (LBO).
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(const void* smem_tile) {
  const uint32_t a = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)(16384 >> 4) << 16;  // LBO: next 64-wide MN atom
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: next 8-row K group
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#ifndef A2_EMU16
#define A2_EMU16 7  // of every 16 column pairs, this many take the FMA-pipe exp2 (balances MUFU vs FMA)
#endif
// which column pairs take the FMA-pipe exp2: spread through the loop (pair p with
// (9p mod 16) < A2_EMU16) so the MUFU and FMA pipes are fed interleaved, not in runs
#define A2_EMU(p) ((((p) * 9) & 15) < A2_EMU16)
// the single-tile kernel, with its row sums on the tensor core, has less FMA-pipe work:
// 5 of 16 measured best there (3..5 within 1%, 7 +1.2%, 9 +2.6%)
#ifndef A1_EMU16
#define A1_EMU16 5
#endif
#define A1_EMU(p) ((((p) * 9) & 15) < A1_EMU16)
// ---- softmax arithmetic helpers (packed f32x2 FFMA2/FADD2, 3-input max, exp2
// emulated on the FMA pipe for part of the columns: B200's MUFU ex2 rate (16/clk/SM)
// would otherwise bound the softmax below the tensor core's rate)
__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_split(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// 2^x for two lanes on the FMA pipe: x = n + f, n = rint(x) via the 1.5*2^23
// magic add, 2^f on [-0.5, 0.5] by a cubic (rel. err 7.5e-5, far below bf16's
// 3.9e-3 rounding of P), exponent bits added back. Inputs clamped to >= -127.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float a, b;
  f2_split(x2, a, b);
  x2 = f2(fmaxf(a, -127.f), fmaxf(b, -127.f));
  const uint64_t magic = f2(12582912.f, 12582912.f), nmagic = f2(-12582912.f, -12582912.f);
  const uint64_t t = fadd2(x2, magic);
  float ra0, rb0;
  f2_split(fadd2(t, nmagic), ra0, rb0);                // rint(x)
  const uint64_t fr = fadd2(x2, f2(-ra0, -rb0));       // x - rint(x) in [-0.5, 0.5]
  uint64_t p = ffma2(fr, f2(0.05517095f, 0.05517095f), f2(0.24260963f, 0.24260963f));
  p = ffma2(p, fr, f2(0.69326096f, 0.69326096f));
  p = ffma2(p, fr, f2(0.99992817f, 0.99992817f));
  float pa, pb, ta, tb;
  f2_split(p, pa, pb);
  f2_split(t, ta, tb);
  const float ra = __int_as_float(__float_as_int(pa) + (__float_as_int(ta) << 23));
  const float rb = __int_as_float(__float_as_int(pb) + (__float_as_int(tb) << 23));
  return f2(ra, rb);
}
__device__ __forceinline__ uint32_t bf16x2_bits(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void mma_bf16_ts_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&o)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]),
      "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]), "r"(o[16]),
      "r"(o[17]), "r"(o[18]), "r"(o[19]), "r"(o[20]), "r"(o[21]), "r"(o[22]), "r"(o[23]), "r"(o[24]),
      "r"(o[25]), "r"(o[26]), "r"(o[27]), "r"(o[28]), "r"(o[29]), "r"(o[30]), "r"(o[31]));
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return r;
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&o)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]),
      "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]));
}

#ifdef QCF_ATTN_TRACE
// measurement build only (tools/attn_trace.py): per-CTA globaltimer stamps
__device__ unsigned long long* g_attn_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long* g_attn_trace2 = nullptr;  // [64 key tiles][8] clock64 stamps, CTA (0, 0, 0)
#define QCF_TRACE2(j, k)                                                                                  \
  do {                                                                                                    \
    if (g_attn_trace2 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64)               \
      g_attn_trace2[(j) * 8 + (k)] = clock64();                                                           \
  } while (0)
#define QCF_TRACE(slot, val)                                                                              \
  do {                                                                                                    \
    if (g_attn_trace) {                                                                                   \
      const int64_t cta = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z); \
      g_attn_trace[cta * 8 + (slot)] = (val);                                                             \
    }                                                                                                     \
  } while (0)
#else
#define QCF_TRACE(slot, val) do {} while (0)
#define QCF_TRACE2(j, k) do {} while (0)
#endif

__global__ void __launch_bounds__(AT_THREADS, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
               const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ kmax, int M, int H,
               int Hkv, int n_keys, float scale_log2, __nv_bfloat16* __restrict__ out, int rshift) {
  // request (batch) index: q/out/kmax are [req][M]..., the K/V tables [req][n_keys]...
  // rshift: query tiles start at row t*128 - rshift (virtual rows < 0 are masked), so
  // the partial tile is the FIRST one (fewest keys), not the last (longest key range)
  const int req = blockIdx.z;
  kmax += (int64_t)req * M;
  out += (int64_t)req * M * H * AT_D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + AT_TILE_BYTES;                  // [AT_KS]
  uint8_t* sV = smem + (1 + AT_KS) * AT_TILE_BYTES;    // [AT_VS]
  uint8_t* sOnes = smem + (1 + AT_KS + AT_VS) * AT_TILE_BYTES;  // 16 x 128 bf16 ones (K-major, any swizzle)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOnes + AT_ONES_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* s_full = bars + 1;     // [2]
  uint64_t* s_free = bars + 3;     // [2]
  uint64_t* p_full = bars + 5;     // [2]  per TMEM P buffer (one phase per use: no parity aliasing)
  uint64_t* pv_done = bars + 7;    // [2]
  uint64_t* k_full = bars + 9;     // [AT_KS]  K ring: freed as soon as S_j is computed
  uint64_t* k_empty = k_full + AT_KS;
  uint64_t* v_full = k_empty + AT_KS;  // [AT_VS]  V ring: freed when P_j.V_j is done
  uint64_t* v_empty = v_full + AT_VS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + AT_VS);
  __shared__ float red[2][4][AT_BM];   // per-tile partial row max (double-buffered by tile parity)
  __shared__ int s_kend;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (M + AT_BM - 1) / AT_BM;
  const int qt = n_qt - 1 - blockIdx.y;  // longest tiles (largest positions) launch first
  const int head = blockIdx.x;
  const int kvh = head / (H / Hkv);
  const int m0 = qt * AT_BM - rshift;
  constexpr int N_SOFT_WARPS = AT_THREADS / 32 - 2;  // 16 softmax warps (one arrive each)

#ifdef QCF_ATTN_TRACE
  if (threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    QCF_TRACE(0, sm);
    QCF_TRACE(1, gtimer());
  }
#endif
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < AT_KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], N_SOFT_WARPS);
      mbar_init(&p_full[s], N_SOFT_WARPS);
      mbar_init(&pv_done[s], 1);
    }
    for (int s = 0; s < AT_VS; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
    s_kend = 0;
  }
  if (threadIdx.x < AT_ONES_BYTES / 16)   // ones for the row-sum MMA, then visible to the tensor core
    reinterpret_cast<uint4*>(sOnes)[threadIdx.x] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  __syncthreads();
  pdl_wait();  // barrier init + TMEM alloc overlap the previous kernel's tail
  pdl_trigger();
  if (threadIdx.x == 0) {  // Q and the first K tile (every tile has >= 1 key tile) in flight
    mbar_expect_tx(q_full, AT_TILE_BYTES);    // while the key range is being scanned
    tma_load_3d(sQ, &map_q, q_full, head * AT_D, m0, req);
    tma_load_3d(sQ + AT_TILE_BYTES / 2, &map_q, q_full, head * AT_D + 64, m0, req);
    mbar_expect_tx(&k_full[0], AT_TILE_BYTES);
    tma_load_3d(sK, &map_k, &k_full[0], kvh * AT_D, 0, req);
    tma_load_3d(sK + AT_TILE_BYTES / 2, &map_k, &k_full[0], kvh * AT_D + 64, 0, req);
  }
  // key range of this tile = 1 + max kmax over its rows (rows are normally
  // sorted by position, but the kernel does not rely on it)
  if (threadIdx.x < AT_BM) {
    const int rr = m0 + (int)threadIdx.x;
    int v = (rr >= 0 && rr < M) ? kmax[rr] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s_kend, max(1, min(v + 1, n_keys)));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_tiles = (s_kend + AT_BN - 1) / AT_BN;
  // S[2] | O | row sums: P_j is written over its own S buffer (each softmax warp over the
  // S columns it alone read), and P_j . 1 (16 equal columns at tOS) gives the row sums on
  // the tensor core instead of 16 FADD2 per thread and key tile (traced: -170 cycles/tile)
  const uint32_t tS0 = tmem, tO = tmem + 256, tOS = tmem + 384;
#ifdef QCF_ATTN_TRACE
  if (threadIdx.x == 0) { QCF_TRACE(2, gtimer()); QCF_TRACE(7, n_tiles); }
#endif

  if (warp == 0) {
    // ---------------- TMA producers: lane 0 streams K (K_0 was issued above), lane 1
    // streams V; K_j is consumed by S_j (early), V_j by P_j.V_j (a key tile later)
    if (lane == 0) {
      for (int j = 1; j < n_tiles; ++j) {
        const int st = j % AT_KS;
        mbar_wait(&k_empty[st], ((j / AT_KS) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], AT_TILE_BYTES);
        uint8_t* k = sK + st * AT_TILE_BYTES;
        tma_load_3d(k, &map_k, &k_full[st], kvh * AT_D, j * AT_BN, req);
        tma_load_3d(k + AT_TILE_BYTES / 2, &map_k, &k_full[st], kvh * AT_D + 64, j * AT_BN, req);
      }
    } else if (lane == 1) {
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % AT_VS;
        mbar_wait(&v_empty[st], ((j / AT_VS) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], AT_TILE_BYTES);
        uint8_t* v = sV + st * AT_TILE_BYTES;
        tma_load_3d(v, &map_v, &v_full[st], kvh * AT_D, j * AT_BN, req);
        tma_load_3d(v + AT_TILE_BYTES / 2, &map_v, &v_full[st], kvh * AT_D + 64, j * AT_BN, req);
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (whole warp converged; one elected lane issues)
      constexpr uint32_t idesc_s = idesc_bf16_f32(AT_BM, AT_BN);                  // K-major A, K-major B
      constexpr uint32_t idesc_o = idesc_bf16_f32(AT_BM, AT_D) | (1u << 16);      // B (V) MN-major
      constexpr uint32_t idesc_l = idesc_bf16_f32(AT_BM, 16);                     // B = ones, K-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_pv = [&](int jj) {
        const int st = jj & 1;
        mbar_wait(&p_full[st], (jj >> 1) & 1);
#ifdef QCF_ATTN_TRACE
        QCF_TRACE2(jj, 7);
#endif
        const int vs = jj % AT_VS;
        mbar_wait(&v_full[vs], (jj / AT_VS) & 1);
#ifdef QCF_ATTN_TRACE
        QCF_TRACE2(jj, 1);
#endif
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_BN / 16; ++kk) {   // A = P_jj straight from TMEM (packed bf16)
          // keys 16kk..16kk+15 were written by softmax warp cg = kk/2 at the start of its S columns
          const uint32_t pa = tS0 + st * 128 + (kk >> 1) * 32 + (kk & 1) * 8;
          const uint64_t b = umma_desc_mn_sw128(sV + vs * AT_TILE_BYTES + kk * 16 * 128);
          mma_bf16_ts_e(tO, pa, b, idesc_o, (jj | kk) != 0);
          const uint64_t bl = umma_desc_k_sw128(sOnes + (kk >> 2) * (AT_ONES_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
          mma_bf16_ts_e(tOS, pa, bl, idesc_l, (jj | kk) != 0);
        }
#ifdef QCF_ATTN_TRACE
        QCF_TRACE2(jj, 2);
#endif
        mma_commit_e(&v_empty[vs]);
        mma_commit_e(&pv_done[st]);
#ifdef QCF_ATTN_TRACE
        QCF_TRACE2(jj, 6);
#endif
      };
      // (issuing S_{j+2} ahead of P_j.V_j measured 4% slower, with either K ring depth:
      //  the traced period is set by the softmax of one tile, ~1850 cycles, plus its wait
      //  for S_{j+1}; removing all V traffic did not change it either)
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % AT_KS, sb = j & 1;
        mbar_wait(&k_full[st], (j / AT_KS) & 1);
        mbar_wait(&s_free[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {
          const uint64_t a = umma_desc_k_sw128(sQ + (kk >> 2) * (AT_TILE_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
          const uint64_t b = umma_desc_k_sw128(sK + st * AT_TILE_BYTES + (kk >> 2) * (AT_TILE_BYTES / 2)) +
                             (uint64_t)((kk & 3) * 2);
          mma_bf16_e(tS0 + sb * 128, a, b, idesc_s, kk != 0);
        }
        mma_commit_e(&s_full[sb]);
        mma_commit_e(&k_empty[st]);
#ifdef QCF_ATTN_TRACE
        QCF_TRACE2(j, 5);
#endif
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {  // ---------------- softmax / correction / epilogue (warps 2..17)
    const int g = warp & 3;               // TMEM lane quarter -> rows 32g..32g+31
    const int cg = (warp - 2) >> 2;       // column group: S keys / O dims 32cg..32cg+31
    const int r = g * 32 + lane;          // row within the tile == TMEM lane
    const int row = m0 + r;
    const int my_kmax = (row >= 0 && row < M) ? kmax[row] : -1;
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const int bar_id = 1 + g;             // named barrier of the 4 warps sharing these rows
    float m_ref = -INFINITY;
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
#ifdef QCF_ATTN_TRACE
      if (j == 0 && threadIdx.x == 64) QCF_TRACE(3, gtimer());
      if (threadIdx.x == 64) QCF_TRACE2(j, 0);
#endif
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tS0 + sb * 128 + cg * 32 + lane_off, v);
      tmem_ld_wait();

      const int lim = my_kmax - j * AT_BN - cg * 32;  // columns <= lim are visible
      const bool all_vis = __all_sync(0xffffffffu, lim >= 31);
      const bool none_vis = __all_sync(0xffffffffu, lim < 0);
      float pmax = -INFINITY;
      if (all_vis) {
        {  // two independent max chains (shorter dependency chain)
          float pm1 = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            pmax = fmax3(pmax, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            pm1 = fmax3(pm1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
          }
          pmax = fmaxf(pmax, pm1);
        }
      } else if (!none_vis) {
#pragma unroll
        for (int i = 0; i < 32; ++i) pmax = fmaxf(pmax, i <= lim ? __uint_as_float(v[i]) : -INFINITY);
      }
      red[sb][cg][r] = pmax * scale_log2;
      named_bar(bar_id, 128);

      const float tmax = fmaxf(fmaxf(red[sb][0][r], red[sb][1][r]), fmaxf(red[sb][2][r], red[sb][3][r]));
      const bool need = tmax > m_ref + 8.f;  // lazily move the reference max
      float alpha = 1.f;
      if (need) {
        alpha = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - tmax);
        m_ref = tmax;
      }
      // P buffer j&1 was read by P_{j-2}.V_{j-2}; the O rescale needs P_{j-1}.V_{j-1}
      if (j >= 2) {
        mbar_wait(&pv_done[j & 1], ((j >> 1) - 1) & 1);
        tc_fence_after();
      }
      const bool rescale = j > 0 && __any_sync(0xffffffffu, need);
      if (rescale) {
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
      }
      if (rescale) {  // rescale this warp's O slice in TMEM
        uint32_t o[32];
        tmem_ld32(tO + cg * 32 + lane_off, o);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
            "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tO + cg * 32 + lane_off),
            "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]),
            "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]), "r"(o[16]),
            "r"(o[17]), "r"(o[18]), "r"(o[19]), "r"(o[20]), "r"(o[21]), "r"(o[22]), "r"(o[23]), "r"(o[24]),
            "r"(o[25]), "r"(o[26]), "r"(o[27]), "r"(o[28]), "r"(o[29]), "r"(o[30]), "r"(o[31]));
        if (cg == 0) {  // the row sums (16 equal columns) scale with O
          uint32_t ls[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(ls[0]), "=r"(ls[1]), "=r"(ls[2]), "=r"(ls[3]), "=r"(ls[4]), "=r"(ls[5]), "=r"(ls[6]),
                "=r"(ls[7]), "=r"(ls[8]), "=r"(ls[9]), "=r"(ls[10]), "=r"(ls[11]), "=r"(ls[12]), "=r"(ls[13]),
                "=r"(ls[14]), "=r"(ls[15])
              : "r"(tOS + lane_off));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) ls[i] = __float_as_uint(__uint_as_float(ls[i]) * alpha);
          tmem_st16(tOS + lane_off, ls);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      // P = exp2(s*scale - m_ref) -> packed bf16 for keys 32cg..32cg+31 (TMEM P buffer j&1)
      uint32_t pk[16];
      if (none_vis) {
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0u;
      } else {
        if (all_vis) {  // packed f32x2 math, part of the exp2 on the FMA pipe
          const uint64_t sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m_ref, -m_ref);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t x2 = ffma2(f2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sc2, nm2);
            uint64_t p2;
            if (A1_EMU(i >> 1)) {
              p2 = exp2_poly2(x2);
            } else {
              float a, b;
              f2_split(x2, a, b);
              p2 = f2(ex2_approx(a), ex2_approx(b));
            }
            float p0, p1;
            f2_split(p2, p0, p1);
            pk[i >> 1] = bf16x2_bits(p0, p1);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float p0 = ex2_approx(fmaf(__uint_as_float(v[i]), scale_log2, -m_ref));
            float p1 = ex2_approx(fmaf(__uint_as_float(v[i + 1]), scale_log2, -m_ref));
            p0 = (i <= lim) ? p0 : 0.f;
            p1 = (i + 1 <= lim) ? p1 : 0.f;
            pk[i >> 1] = bf16x2_bits(p0, p1);
          }
        }
      }
#ifdef QCF_ATTN_TRACE
      if (threadIdx.x == 64) QCF_TRACE2(j, 3);
#endif
      tmem_st16(tS0 + sb * 128 + cg * 32 + lane_off, pk);  // keys 32cg.. -> the first 16 of this warp's S cols
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // one arrive per warp: 512 per-thread arrives cost ~1000 cycles per key tile
        mbar_arrive(&s_free[sb]);
        mbar_arrive(&p_full[j & 1]);
      }
#ifdef QCF_ATTN_TRACE
      if (threadIdx.x == 64) QCF_TRACE2(j, 4);
#endif
    }
    // epilogue: combine the 4 partial row sums, then O / l for this warp's 32 columns
#ifdef QCF_ATTN_TRACE
    if (threadIdx.x == 64) QCF_TRACE(4, gtimer());
#endif
    mbar_wait(&pv_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
    tc_fence_after();
    const float lt = __uint_as_float(tmem_ld1(tOS + lane_off));   // row sum = (P . 1)
    tmem_ld_wait();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    uint32_t o[32];
    tmem_ld32(tO + cg * 32 + lane_off, o);
    tmem_ld_wait();
#ifdef QCF_ATTN_TRACE
    if (threadIdx.x == 64) QCF_TRACE(5, gtimer());
#endif
    if (row >= 0 && row < M) {
      __nv_bfloat16* dst = out + ((int64_t)row * H + head) * AT_D + cg * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 pk4;
        __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk4);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          p2[u] = __floats2bfloat162_rn(__uint_as_float(o[i + 2 * u]) * inv, __uint_as_float(o[i + 2 * u + 1]) * inv);
        *reinterpret_cast<uint4*>(dst + i) = pk4;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
#ifdef QCF_ATTN_TRACE
    if (lane == 0) QCF_TRACE(6, gtimer());
#endif
  }
}

// ---------------------------------------------------------------------------
// v4: two CTAs per SM, 64-key tiles. The single-tile kernel's per key tile period
// (~2100 cycles traced) is one softmax latency chain with every softmax warp in the
// same phase, plus ~5 us of per-CTA setup / epilogue with the tensor core idle.
// Here one CTA (128 query rows, one head) needs only 256 TMEM columns
// (S double-buffered at 64 keys + O) and ~97 KB of shared memory, so two CTAs
// share an SM: one CTA's softmax, setup and epilogue run while the other's MMAs
// keep the tensor core busy (the hardware interleaves them; no ping-pong code).
//   warp 0      TMA: lane 0 streams Q then K tiles (2-stage ring), lane 1 V tiles
//   warp 1      MMA: S_0, S_1, then per key tile j: P_j.V_j, S_{j+2} into P_j's
//               buffer (tcgen05 ops of one thread execute in order: S_{j+2} cannot
//               overwrite P_j before P_j.V_j has read it)
//   warps 2..   softmax: SW = 4 -> one full 64-key row per thread (no cross-warp
//               max exchange); SW = 8 -> half rows, max exchanged through smem.
//               Row sums in registers (FADD2), lazy reference max (rescale O only
//               when the running max grows by > 2^8), epilogue O / l.
// ---------------------------------------------------------------------------
constexpr int A4_BN = 64;
constexpr int A4_KT = A4_BN * AT_D * 2;  // 16 KB: one 64-key K or V tile (two 8 KB SW128 atoms)
constexpr int A4_KS = 2, A4_VS = 2;
constexpr int A4_SMEM = AT_TILE_BYTES + A4_KT * (A4_KS + A4_VS) + 1024 + 256;

// MN-major SW128 descriptor for a 64-key V tile: 8-key groups 1024 B apart (SBO),
// the two 64-dim atoms 8 KB apart (LBO)
__device__ __forceinline__ uint64_t umma_desc_mn_sw128_k64(const void* smem_tile) {
  const uint32_t a = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int SW, int EMU16>
__global__ void __launch_bounds__(64 + SW * 32, 2)
attn_tc4_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ kmax, int M, int H,
                int Hkv, int n_keys, float scale_log2, __nv_bfloat16* __restrict__ out, int rshift) {
  constexpr int NCH = SW / 4;          // warps sharing one row (column chunks)
  constexpr int CW = A4_BN / NCH;      // S columns (keys) per softmax thread: 64 or 32
  constexpr int OW = AT_D / NCH;       // output dims per softmax thread: 128 or 64
  const int req = blockIdx.z;
  kmax += (int64_t)req * M;
  out += (int64_t)req * M * H * AT_D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + AT_TILE_BYTES;               // [A4_KS]
  uint8_t* sV = sK + A4_KS * A4_KT;                 // [A4_VS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + A4_VS * A4_KT);
  uint64_t* q_full = bars + 0;
  uint64_t* s_full = bars + 1;     // [2] S buffer b holds S_j, j = b mod 2
  uint64_t* p_full = bars + 3;     // [2] P_j stored over S_j (SW arrives)
  uint64_t* pv_done = bars + 5;    // [2] P_j.V_j complete
  uint64_t* k_full = bars + 7;     // [A4_KS]
  uint64_t* k_empty = k_full + A4_KS;
  uint64_t* v_full = k_empty + A4_KS;   // [A4_VS]
  uint64_t* v_empty = v_full + A4_VS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + A4_VS);
  __shared__ float red[2][NCH][AT_BM];
  __shared__ float red_l[NCH][AT_BM];
  __shared__ int s_kend;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (M + AT_BM - 1) / AT_BM;
  const int qt = n_qt - 1 - blockIdx.y;   // longest tiles first
  const int head = blockIdx.x;
  const int kvh = head / (H / Hkv);
  const int m0 = qt * AT_BM - rshift;
#ifdef QCF_ATTN_TRACE
  if (threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    QCF_TRACE(0, sm);
    QCF_TRACE(1, gtimer());
  }
#endif

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], SW);
      mbar_init(&pv_done[s], 1);
    }
    for (int s = 0; s < A4_KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < A4_VS; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
    s_kend = 0;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {  // Q and K_0 in flight while the key range is scanned
    mbar_expect_tx(q_full, AT_TILE_BYTES);
    tma_load_3d(sQ, &map_q, q_full, head * AT_D, m0, req);
    tma_load_3d(sQ + AT_TILE_BYTES / 2, &map_q, q_full, head * AT_D + 64, m0, req);
    mbar_expect_tx(&k_full[0], A4_KT);
    tma_load_3d(sK, &map_k, &k_full[0], kvh * AT_D, 0, req);
    tma_load_3d(sK + A4_KT / 2, &map_k, &k_full[0], kvh * AT_D + 64, 0, req);
  }
  if (threadIdx.x < AT_BM) {
    const int rr = m0 + (int)threadIdx.x;
    int v = (rr >= 0 && rr < M) ? kmax[rr] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMax(&s_kend, max(1, min(v + 1, n_keys)));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_tiles = (s_kend + A4_BN - 1) / A4_BN;
  const uint32_t tS = tmem, tO = tmem + 128;   // S[2] (64 columns each) | O (128)
#ifdef QCF_ATTN_TRACE
  if (threadIdx.x == 0) { QCF_TRACE(2, gtimer()); QCF_TRACE(7, n_tiles); }
#endif

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 1; j < n_tiles; ++j) {
        const int st = j % A4_KS;
        mbar_wait(&k_empty[st], ((j / A4_KS) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], A4_KT);
        uint8_t* k = sK + st * A4_KT;
        tma_load_3d(k, &map_k, &k_full[st], kvh * AT_D, j * A4_BN, req);
        tma_load_3d(k + A4_KT / 2, &map_k, &k_full[st], kvh * AT_D + 64, j * A4_BN, req);
      }
    } else if (lane == 1) {
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % A4_VS;
        mbar_wait(&v_empty[st], ((j / A4_VS) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], A4_KT);
        uint8_t* v = sV + st * A4_KT;
        tma_load_3d(v, &map_v, &v_full[st], kvh * AT_D, j * A4_BN, req);
        tma_load_3d(v + A4_KT / 2, &map_v, &v_full[st], kvh * AT_D + 64, j * A4_BN, req);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = idesc_bf16_f32(AT_BM, A4_BN);
    constexpr uint32_t idesc_o = idesc_bf16_f32(AT_BM, AT_D) | (1u << 16);  // B (V) MN-major
    mbar_wait(q_full, 0);
    tc_fence_after();
    auto issue_s = [&](int j) {
      const int st = j % A4_KS, sb = j & 1;
      mbar_wait(&k_full[st], (j / A4_KS) & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT_D / 16; ++kk) {
        const uint64_t a = umma_desc_k_sw128(sQ + (kk >> 2) * (AT_TILE_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
        const uint64_t b = umma_desc_k_sw128(sK + st * A4_KT + (kk >> 2) * (A4_KT / 2)) + (uint64_t)((kk & 3) * 2);
        mma_bf16_e(tS + sb * 64, a, b, idesc_s, kk != 0);
      }
      mma_commit_e(&s_full[sb]);
      mma_commit_e(&k_empty[st]);
      QCF_TRACE2(j, 5);
    };
    issue_s(0);
    if (n_tiles > 1) issue_s(1);
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1, vs = j % A4_VS;
      mbar_wait(&p_full[sb], (j >> 1) & 1);
      QCF_TRACE2(j, 7);
      mbar_wait(&v_full[vs], (j / A4_VS) & 1);
      QCF_TRACE2(j, 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < A4_BN / 16; ++kk) {
        // keys 16kk..16kk+15 = packed columns at the start of their owner's S columns
        const uint32_t pa = tS + sb * 64 + (kk * 16 / CW) * CW + ((kk * 16) % CW) / 2;
        const uint64_t b = umma_desc_mn_sw128_k64(sV + vs * A4_KT + kk * 16 * 128);
        mma_bf16_ts_e(tO, pa, b, idesc_o, (j | kk) != 0);
      }
      QCF_TRACE2(j, 2);
      mma_commit_e(&v_empty[vs]);
      mma_commit_e(&pv_done[sb]);
      QCF_TRACE2(j, 6);
      if (j + 2 < n_tiles) issue_s(j + 2);
    }
  } else {
    const int sw = warp - 2;
    const int g = warp & 3;               // TMEM lane quarter -> rows 32g..32g+31
    const int ch = sw >> 2;               // column chunk (SW = 8: keys / dims half)
    const int r = g * 32 + lane;
    const int row = m0 + r;
    const int my_kmax = (row >= 0 && row < M) ? kmax[row] : -1;
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const uint64_t sc2 = f2(scale_log2, scale_log2);
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
#ifdef QCF_ATTN_TRACE
      if (j == 0 && threadIdx.x == 64) QCF_TRACE(3, gtimer());
      if (threadIdx.x == 64) QCF_TRACE2(j, 0);
#endif
      tc_fence_after();
      uint32_t v[CW];
      tmem_ld32(tS + sb * 64 + ch * CW + lane_off, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
      if constexpr (CW == 64) tmem_ld32(tS + sb * 64 + 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
      tmem_ld_wait();
      const int lim = my_kmax - j * A4_BN - ch * CW;  // columns <= lim are visible
      const bool all_vis = __all_sync(0xffffffffu, lim >= CW - 1);
      const bool none_vis = __all_sync(0xffffffffu, lim < 0);
      float pmax = -INFINITY;
      if (all_vis) {
        float pm1 = -INFINITY;
#pragma unroll
        for (int i = 0; i < CW; i += 4) {
          pmax = fmax3(pmax, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          pm1 = fmax3(pm1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        }
        pmax = fmaxf(pmax, pm1);
      } else if (!none_vis) {
#pragma unroll
        for (int i = 0; i < CW; ++i) pmax = fmaxf(pmax, i <= lim ? __uint_as_float(v[i]) : -INFINITY);
      }
      float tmax = pmax * scale_log2;
      if constexpr (NCH > 1) {
        red[sb][ch][r] = tmax;
        named_bar(1 + g, 64);
        tmax = fmaxf(red[sb][0][r], red[sb][1][r]);
      }
      const bool need = tmax > m_ref + 8.f;  // lazily move the reference max
      float alpha = 1.f;
      if (need) {
        alpha = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - tmax);
        m_ref = tmax;
        l *= alpha;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {  // rescale O after P_{j-1}.V_{j-1}
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < OW / 32; ++hh) {
          uint32_t o[32];
          tmem_ld32(tO + ch * OW + hh * 32 + lane_off, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tO + ch * OW + hh * 32 + lane_off, o);
        }
      }
      uint32_t pk[CW / 2];
      if (none_vis) {
#pragma unroll
        for (int i = 0; i < CW / 2; ++i) pk[i] = 0u;
      } else if (all_vis) {
        const uint64_t nm2 = f2(-m_ref, -m_ref);
        uint64_t l2 = f2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < CW; i += 2) {
          const uint64_t x2 = ffma2(f2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sc2, nm2);
          uint64_t p2;
          if (((((i >> 1) & 15) * 9) & 15) < EMU16) {
            p2 = exp2_poly2(x2);
          } else {
            float a, b;
            f2_split(x2, a, b);
            p2 = f2(ex2_approx(a), ex2_approx(b));
          }
          l2 = fadd2(l2, p2);
          float p0, p1;
          f2_split(p2, p0, p1);
          pk[i >> 1] = bf16x2_bits(p0, p1);
        }
        float la, lb;
        f2_split(l2, la, lb);
        l += la + lb;
      } else {
#pragma unroll
        for (int i = 0; i < CW; i += 2) {
          float p0 = ex2_approx(fmaf(__uint_as_float(v[i]), scale_log2, -m_ref));
          float p1 = ex2_approx(fmaf(__uint_as_float(v[i + 1]), scale_log2, -m_ref));
          p0 = (i <= lim) ? p0 : 0.f;
          p1 = (i + 1 <= lim) ? p1 : 0.f;
          l += p0 + p1;
          pk[i >> 1] = bf16x2_bits(p0, p1);
        }
      }
#ifdef QCF_ATTN_TRACE
      if (threadIdx.x == 64) QCF_TRACE2(j, 3);
#endif
      if constexpr (CW == 64) tmem_st32(tS + sb * 64 + lane_off, pk);
      else tmem_st16(tS + sb * 64 + ch * CW + lane_off, pk);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
#ifdef QCF_ATTN_TRACE
      if (threadIdx.x == 64) QCF_TRACE2(j, 4);
#endif
    }
#ifdef QCF_ATTN_TRACE
    if (threadIdx.x == 64) QCF_TRACE(4, gtimer());
#endif
    // epilogue: O / l
    float lt = l;
    if constexpr (NCH > 1) {
      red_l[ch][r] = l;
      named_bar(1 + g, 64);
      lt = red_l[0][r] + red_l[1][r];
    }
    mbar_wait(&pv_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
    tc_fence_after();
#ifdef QCF_ATTN_TRACE
    if (threadIdx.x == 64) QCF_TRACE(5, gtimer());
#endif
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
    for (int hh = 0; hh < OW / 32; ++hh) {
      uint32_t o[32];
      tmem_ld32(tO + ch * OW + hh * 32 + lane_off, o);
      tmem_ld_wait();
      if (row >= 0 && row < M) {
        __nv_bfloat16* dst = out + ((int64_t)row * H + head) * AT_D + ch * OW + hh * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 pk4;
          __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk4);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            p2[u] = __floats2bfloat162_rn(__uint_as_float(o[i + 2 * u]) * inv, __uint_as_float(o[i + 2 * u + 1]) * inv);
          *reinterpret_cast<uint4*>(dst + i) = pk4;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
#ifdef QCF_ATTN_TRACE
    if (lane == 0) QCF_TRACE(6, gtimer());
#endif
  }
}

// ---------------------------------------------------------------------------
// v8: one 128-row query tile per CTA over 128-key tiles, with two softmax warp
// groups taking alternate key tiles (group j & 1) and THREE S buffers. In v1 all
// 16 softmax warps step through the same latency chain per tile; here one group
// exponentiates tile j while the other already works on tile j+1, and S_{j+3}
// goes into P_j's buffer right after P_j.V_j, so a group's next S is ready when it
// finishes a tile. The groups share only the lazy reference max: the owner of
// tile j publishes its per-row reference in shared memory (mref_ready[j & 1]) and
// the owner of tile j+1 starts from it. TMEM: S[3] (128 each) | O (128) = 512
// columns, so the row sums live in registers (each thread sums its 64 keys; the
// four partials of a row -- 2 groups x 2 halves, each relative to its group's
// last reference max -- are combined in the epilogue).
// Measured (tools/attn_bench.py, tools/attn_trace.py knob 8): ~1780 cycles per key
// tile vs ~2100 for v1; one request's 224 tiles 44 vs 48 us. The tile period is
// now set by shared-memory bandwidth: per key and 128-row query tile the K and V
// rows are written by TMA (512 B) and read by the MMAs (K + Q slab and V), about
// 1 KB per 8 tensor-core cycles -- the SM's ~128 B/clk. (A variant with Q in TMEM
// and two S buffers -- TS S-MMAs, 32 KB less smem traffic per tile -- measured
// ~1820 cycles per tile: the MMA round trip P_j -> P_j.V_j -> S_{j+2} then sat on
// each group's chain.)
//   warp 0      TMA: lane 0 Q then the K ring, lane 1 the V ring
//   warp 1      MMA: S_0 S_1 S_2, then per key tile j: P_j.V_j, S_{j+3} into
//               P_j's buffer (j mod 3)
//   warps 2..9  softmax group 0 (even tiles), 10..17 group 1 (odd tiles)
// ---------------------------------------------------------------------------
constexpr int A8_KS = 2, A8_VS = 3;
constexpr int A8_THREADS = 576;
constexpr int A8_SMEM = AT_TILE_BYTES * (1 + A8_KS + A8_VS) + 1024 + 256;

__global__ void __launch_bounds__(A8_THREADS, 1)
attn_tc8_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ kmax, int M, int H,
                int Hkv, int n_keys, float scale_log2, __nv_bfloat16* __restrict__ out, int rshift) {
  const int req = blockIdx.z;
  kmax += (int64_t)req * M;
  out += (int64_t)req * M * H * AT_D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + AT_TILE_BYTES;                   // [A8_KS]
  uint8_t* sV = sK + A8_KS * AT_TILE_BYTES;             // [A8_VS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + A8_VS * AT_TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* o_full = bars + 1;      // every P.V done
  uint64_t* s_full = bars + 2;      // [3]
  uint64_t* p_full = bars + 5;      // [3] (the 8 warps of the owning group)
  uint64_t* pv_done = bars + 8;     // [3]
  uint64_t* mref_ready = bars + 11; // [2] reference max after tile j published (4 warps)
  uint64_t* k_full = bars + 13;     // [A8_KS]
  uint64_t* k_empty = k_full + A8_KS;
  uint64_t* v_full = k_empty + A8_KS;  // [A8_VS]
  uint64_t* v_empty = v_full + A8_VS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + A8_VS);
  __shared__ float red[2][2][2][AT_BM]; // [group][group-tile parity][column half][row] partial row max
  __shared__ float mref_buf[2][AT_BM];  // [tile parity][row] reference max after that tile
  __shared__ float lsum[2][2][AT_BM];   // [group][half][row] row-sum partials (epilogue)
  __shared__ float lref[2][AT_BM];      // [group][row] the reference those partials are relative to
  __shared__ int s_kend;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (M + AT_BM - 1) / AT_BM;
  const int qt = n_qt - 1 - blockIdx.y;  // longest tiles first
  const int head = blockIdx.x;
  const int kvh = head / (H / Hkv);
  const int m0 = qt * AT_BM - rshift;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_v);
    mbar_init(q_full, 1);
    mbar_init(o_full, 1);
    for (int s = 0; s < 3; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 8);
      mbar_init(&pv_done[s], 1);
    }
    for (int s = 0; s < 2; ++s) mbar_init(&mref_ready[s], 4);
    for (int s = 0; s < A8_KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < A8_VS; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
    s_kend = 0;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {  // Q and K_0 in flight while the key range is scanned
    mbar_expect_tx(q_full, AT_TILE_BYTES);
    tma_load_3d(sQ, &map_q, q_full, head * AT_D, m0, req);
    tma_load_3d(sQ + AT_TILE_BYTES / 2, &map_q, q_full, head * AT_D + 64, m0, req);
    mbar_expect_tx(&k_full[0], AT_TILE_BYTES);
    tma_load_3d(sK, &map_k, &k_full[0], kvh * AT_D, 0, req);
    tma_load_3d(sK + AT_TILE_BYTES / 2, &map_k, &k_full[0], kvh * AT_D + 64, 0, req);
  }
  if (threadIdx.x < AT_BM) {
    const int rr = m0 + (int)threadIdx.x;
    int v = (rr >= 0 && rr < M) ? kmax[rr] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMax(&s_kend, max(1, min(v + 1, n_keys)));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_tiles = (s_kend + AT_BN - 1) / AT_BN;
  const uint32_t tS0 = tmem, tO = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 1; j < n_tiles; ++j) {
        const int st = j % A8_KS;
        mbar_wait(&k_empty[st], ((j / A8_KS) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], AT_TILE_BYTES);
        uint8_t* k = sK + st * AT_TILE_BYTES;
        tma_load_3d(k, &map_k, &k_full[st], kvh * AT_D, j * AT_BN, req);
        tma_load_3d(k + AT_TILE_BYTES / 2, &map_k, &k_full[st], kvh * AT_D + 64, j * AT_BN, req);
      }
    } else if (lane == 1) {
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % A8_VS;
        mbar_wait(&v_empty[st], ((j / A8_VS) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], AT_TILE_BYTES);
        uint8_t* v = sV + st * AT_TILE_BYTES;
        tma_load_3d(v, &map_v, &v_full[st], kvh * AT_D, j * AT_BN, req);
        tma_load_3d(v + AT_TILE_BYTES / 2, &map_v, &v_full[st], kvh * AT_D + 64, j * AT_BN, req);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = idesc_bf16_f32(AT_BM, AT_BN);                  // K-major A (Q) and B (K)
    constexpr uint32_t idesc_o = idesc_bf16_f32(AT_BM, AT_D) | (1u << 16);      // B (V) MN-major
    mbar_wait(q_full, 0);
    tc_fence_after();
    auto issue_s = [&](int j) {
      const int st = j % A8_KS;
      mbar_wait(&k_full[st], (j / A8_KS) & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT_D / 16; ++kk) {
        const uint64_t a = umma_desc_k_sw128(sQ + (kk >> 2) * (AT_TILE_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
        const uint64_t b = umma_desc_k_sw128(sK + st * AT_TILE_BYTES + (kk >> 2) * (AT_TILE_BYTES / 2)) +
                           (uint64_t)((kk & 3) * 2);
        mma_bf16_e(tS0 + (j % 3) * 128, a, b, idesc_s, kk != 0);
      }
      mma_commit_e(&s_full[j % 3]);
      mma_commit_e(&k_empty[st]);
      QCF_TRACE2(j, 5);
    };
    for (int j = 0; j < 3 && j < n_tiles; ++j) issue_s(j);
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j % 3, vs = j % A8_VS;
      mbar_wait(&p_full[sb], (j / 3) & 1);
      QCF_TRACE2(j, 7);
      mbar_wait(&v_full[vs], (j / A8_VS) & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT_BN / 16; ++kk) {   // keys 16kk.. : half kk/4, packed at 64*(kk/4) + 8*(kk%4)
        const uint32_t pa = tS0 + sb * 128 + (kk >> 2) * 64 + (kk & 3) * 8;
        const uint64_t b = umma_desc_mn_sw128(sV + vs * AT_TILE_BYTES + kk * 16 * 128);
        mma_bf16_ts_e(tO, pa, b, idesc_o, (j | kk) != 0);
      }
      QCF_TRACE2(j, 2);
      mma_commit_e(&v_empty[vs]);
      mma_commit_e(&pv_done[sb]);
      QCF_TRACE2(j, 6);
      if (j + 3 < n_tiles) issue_s(j + 3);
    }
    mma_commit_e(o_full);
  } else {
    const int sw = warp - 2;
    const int grp = sw >> 3;              // softmax group: tiles j with j & 1 == grp
    const int h = (sw >> 2) & 1;          // column half: keys 64h..64h+63 of a tile
    const int g = warp & 3;               // TMEM lane quarter -> rows 32g..32g+31
    const int r = g * 32 + lane;
    const int row = m0 + r;
    const int my_kmax = (row >= 0 && row < M) ? kmax[row] : -1;
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const uint64_t sc2 = f2(scale_log2, scale_log2);
    float l = 0.f, m_mine = -INFINITY;   // this thread's row-sum partial, relative to m_mine
    for (int j = grp; j < n_tiles; j += 2) {
      const int sb = j % 3;
      mbar_wait(&s_full[sb], (j / 3) & 1);
#ifdef QCF_ATTN_TRACE
      if (lane == 0 && (sw & 7) == 0) QCF_TRACE2(j, 0);
#endif
      tc_fence_after();
      const int lim = my_kmax - j * AT_BN - 64 * h;  // columns <= lim are visible
      const bool all_vis = __all_sync(0xffffffffu, lim >= 63);
      const bool none_vis = __all_sync(0xffffffffu, lim < 0);
      // pass 1: row max over this half's 64 columns, 32 at a time
      float pmax = -INFINITY;
      if (!none_vis) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[32];
          tmem_ld32(tS0 + sb * 128 + 64 * h + 32 * c + lane_off, v);
          tmem_ld_wait();
          if (all_vis) {
            float pm1 = -INFINITY;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              pmax = fmax3(pmax, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
              pm1 = fmax3(pm1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            }
            pmax = fmaxf(pmax, pm1);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) pmax = fmaxf(pmax, 32 * c + i <= lim ? __uint_as_float(v[i]) : -INFINITY);
          }
        }
      }
      const int rp = (j >> 1) & 1;      // a group's consecutive tiles alternate buffers
      red[grp][rp][h][r] = pmax * scale_log2;
      named_bar(1 + grp * 4 + g, 64);   // the two halves of these rows in this group
      const float tmax = fmaxf(red[grp][rp][0][r], red[grp][rp][1][r]);
      float m_prev = -INFINITY;         // reference max after tile j-1 (the other group's)
      if (j > 0) {
        mbar_wait(&mref_ready[(j - 1) & 1], ((j - 1) >> 1) & 1);
        m_prev = mref_buf[(j - 1) & 1][r];
      }
#ifdef QCF_ATTN_TRACE
      if (lane == 0 && (sw & 7) == 0) QCF_TRACE2(j, 1);   // (slot 1 = reference max handed over)
#endif
      const bool need = tmax > m_prev + 8.f;  // lazily move the reference max
      const float m_ref = need ? tmax : m_prev;
      if (h == 0) {
        mref_buf[j & 1][r] = m_ref;
        __syncwarp();
        if (lane == 0) mbar_arrive(&mref_ready[j & 1]);
      }
      if (m_ref > m_mine) {   // this thread's partial sum follows the reference (it only grows)
        l = (m_mine == -INFINITY) ? 0.f : l * ex2_approx(m_mine - m_ref);
        m_mine = m_ref;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {  // rescale O after P_{j-1}.V_{j-1}
        const float alpha = (m_prev == -INFINITY) ? 0.f : ex2_approx(m_prev - m_ref);
        mbar_wait(&pv_done[(j - 1) % 3], ((j - 1) / 3) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int hh = 0; hh < 4; ++hh) {   // 16 columns at a time (register budget)
          uint32_t o[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7]),
                "=r"(o[8]), "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]), "=r"(o[13]), "=r"(o[14]), "=r"(o[15])
              : "r"(tO + 64 * h + 16 * hh + lane_off));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tO + 64 * h + 16 * hh + lane_off, o);
        }
      }
      // pass 2: P = exp2(s*scale - m_ref), packed bf16, 32 keys (16 columns) at a time
      // over the first 32 of this half's 64 S columns; row-sum partial in registers
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
        uint32_t v[32];
        if (!none_vis) {
          tmem_ld32(tS0 + sb * 128 + 64 * h + 32 * c + lane_off, v);
          tmem_ld_wait();
        }
        if (none_vis) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = 0u;
        } else if (all_vis) {
          const uint64_t nm2 = f2(-m_ref, -m_ref);
          uint64_t l2 = f2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t x2 = ffma2(f2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sc2, nm2);
            uint64_t p2;
            if (A2_EMU(i >> 1)) {
              p2 = exp2_poly2(x2);
            } else {
              float a, b;
              f2_split(x2, a, b);
              p2 = f2(ex2_approx(a), ex2_approx(b));
            }
            l2 = fadd2(l2, p2);
            float p0, p1;
            f2_split(p2, p0, p1);
            pk[i >> 1] = bf16x2_bits(p0, p1);
          }
          float la, lb;
          f2_split(l2, la, lb);
          l += la + lb;
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const int e = 32 * c + i;
            float p0 = ex2_approx(fmaf(__uint_as_float(v[i]), scale_log2, -m_ref));
            float p1 = ex2_approx(fmaf(__uint_as_float(v[i + 1]), scale_log2, -m_ref));
            p0 = (e <= lim) ? p0 : 0.f;
            p1 = (e + 1 <= lim) ? p1 : 0.f;
            l += p0 + p1;
            pk[i >> 1] = bf16x2_bits(p0, p1);
          }
        }
#ifdef QCF_ATTN_TRACE
        if (c == 1 && lane == 0 && (sw & 7) == 0) QCF_TRACE2(j, 3);
#endif
        tmem_st16(tS0 + sb * 128 + 64 * h + 16 * c + lane_off, pk);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
#ifdef QCF_ATTN_TRACE
      if (lane == 0 && (sw & 7) == 0) QCF_TRACE2(j, 4);
#endif
    }
    // epilogue: combine the four row-sum partials (2 groups x 2 halves) at the final
    // reference (the largest: references only grow), then O / l for 32 dims per warp
    lsum[grp][h][r] = l;
    if (h == 0) lref[grp][r] = m_mine;
    named_bar(9, 512);                  // the 16 softmax warps
    float lt = 0.f;
    {
      const float ma = lref[0][r], mb = lref[1][r];
      const float mf = fmaxf(ma, mb);
      if (mf != -INFINITY) {
        if (ma != -INFINITY) lt += (lsum[0][0][r] + lsum[0][1][r]) * ex2_approx(ma - mf);
        if (mb != -INFINITY) lt += (lsum[1][0][r] + lsum[1][1][r]) * ex2_approx(mb - mf);
      }
    }
    const int cq = sw >> 2;   // dims 32cq..32cq+31
    mbar_wait(o_full, 0);
    tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    uint32_t o[32];
    tmem_ld32(tO + cq * 32 + lane_off, o);
    tmem_ld_wait();
    if (row >= 0 && row < M) {
      __nv_bfloat16* dst = out + ((int64_t)row * H + head) * AT_D + cq * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 pk4;
        __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk4);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          p2[u] = __floats2bfloat162_rn(__uint_as_float(o[i + 2 * u]) * inv, __uint_as_float(o[i + 2 * u + 1]) * inv);
        *reinterpret_cast<uint4*>(dst + i) = pk4;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// v2: two query tiles per CTA (ping-pong) with P kept in tensor memory.
//
// One CTA = (two 128-row query tiles, one head). TMEM: S_t / P_t (cols 128t..)
// and O_t (cols 256+128t..) for t = 0, 1. Per key tile j the MMA thread issues,
// in order,  PV(0,j-1)? .. : S(0,j) S(1,j) PV(0,j) S(0,j+1) PV(1,j) S(1,j+1) ...
// so the tensor core computes one tile's QK^T / PV while the other tile's
// softmax warps run. P_t,j is written as packed bf16 over the first 64 columns
// of S_t,j (tcgen05.st) and consumed straight from TMEM as the A operand of
// O_t += P_t,j . V_j (the .kind::f16 [a-tmem] form) -- no shared-memory round
// trip. tcgen05 ops of one thread complete in order, so S_t,j+1 (issued after
// PV_t,j) cannot overwrite P_t,j early, and "S_t,j+1 complete" also means
// "PV_t,j complete": the lazy O rescale needs no extra barrier.
// Softmax: 8 warps per tile = 4 TMEM lane quarters x 2 column halves (64 keys /
// 64 output dims each); the two halves of a row exchange their max via smem.
// Pairing of query tiles: adjacent (2p, 2p+1) when the grid spans several
// waves, mirrored (p, n-1-p) -- equal work per CTA -- when it fits in one.
// ---------------------------------------------------------------------------
// SPLIT = warps sharing one row (1: a thread owns a full 128-key row -- no
// cross-warp max exchange; 2: half rows, 8 softmax warps per tile)
template <int SPLIT>
struct A2Cfg {
  static constexpr int THREADS = 64 + 2 * 4 * SPLIT * 32;
  static constexpr int W = 128 / SPLIT;  // keys / output dims per softmax thread
};
constexpr int A2_SMEM = AT_TILE_BYTES * 6 + 1024 + 256;  // Q[2], K[2], V[2]


template <int SPLIT>
__global__ void __launch_bounds__(A2Cfg<SPLIT>::THREADS, 1)
attn_tc2_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ kmax, int M, int H,
                int Hkv, int n_keys, float scale_log2, __nv_bfloat16* __restrict__ out, int mirrored,
                int n_split, float* __restrict__ ws_o, float2* __restrict__ ws_ml, int rshift) {
  // split-KV (n_split > 1, one-wave grids): CTA (pair, chunk) covers key tiles
  // [chunk*n/n_split, (chunk+1)*n/n_split) of the pair's range and leaves an
  // unnormalised fp32 O + (max, sum) per row for attn_combine_kernel
  const int req = blockIdx.z;
  const int pair_y = (int)blockIdx.y / n_split, chunk = (int)blockIdx.y % n_split;
  kmax += (int64_t)req * M;
  out += (int64_t)req * M * H * AT_D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                          // [2 tiles]
  uint8_t* sK = smem + 2 * AT_TILE_BYTES;      // [2 stages]
  uint8_t* sV = smem + 4 * AT_TILE_BYTES;      // [2 stages]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * AT_TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* k_empty = bars + 3;   // [2]
  uint64_t* v_full = bars + 5;    // [2]
  uint64_t* v_empty = bars + 7;   // [2]
  uint64_t* s_full = bars + 9;    // [2 tiles]
  uint64_t* p_full = bars + 11;   // [2 tiles]
  uint64_t* o_full = bars + 13;   // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);
  __shared__ float red[2][2][2][AT_BM];  // [tile][j parity][column half][row]
  __shared__ int s_kend[2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (M + AT_BM - 1) / AT_BM;
  const int n_pairs = (n_qt + 1) / 2;
  int tile0, tile1;
  if (mirrored) {
    const int pidx = n_pairs - 1 - pair_y;
    tile0 = pidx;
    tile1 = n_qt - 1 - pidx;
    if (tile1 == tile0) tile1 = -1;
  } else {
    // adjacent pairs counted from the LAST tile (longest key ranges first, LPT);
    // an odd tile count leaves tile 0 -- the shortest -- without a partner
    const int hi = n_qt - 1 - 2 * pair_y;
    tile0 = hi - 1;
    tile1 = hi;
    if (tile0 < 0) { tile0 = hi; tile1 = -1; }
  }
  const int head = blockIdx.x;
  const int kvh = head / (H / Hkv);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4 * SPLIT);  // one elected arrive per softmax warp of the tile
      mbar_init(&o_full[s], 1);
    }
    fence_barrier_init();
    s_kend[0] = s_kend[1] = 0;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < 2 * AT_BM) {  // key range of each tile = 1 + max kmax over its rows
    const int t = threadIdx.x / AT_BM;
    const int tl = t ? tile1 : tile0;
    int v = 0;
    if (tl >= 0) {
      const int row = tl * AT_BM - rshift + (threadIdx.x % AT_BM);
      v = (row >= 0 && row < M) ? kmax[row] + 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMax(&s_kend[t], min(v, n_keys));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nt0_full = (s_kend[0] + AT_BN - 1) / AT_BN;
  const int nt1_full = (s_kend[1] + AT_BN - 1) / AT_BN;
  const int nfull = max(nt0_full, nt1_full);
  const int jb = chunk * nfull / n_split, je = (chunk + 1) * nfull / n_split;  // key tiles of this CTA
  const int nt0 = max(0, min(nt0_full, je) - jb);
  const int nt1 = max(0, min(nt1_full, je) - jb);
  const int nmax = max(nt0, nt1);

  if (warp == 0) {
    if (lane == 0 && nmax > 0) {  // ---------------- TMA producer
      mbar_expect_tx(q_full, (nt0 > 0 ? AT_TILE_BYTES : 0) + (nt1 > 0 ? AT_TILE_BYTES : 0));
      for (int t = 0; t < 2; ++t) {
        const int n_t = t ? nt1 : nt0, tl = t ? tile1 : tile0;
        if (n_t == 0) continue;
        tma_load_3d(sQ + t * AT_TILE_BYTES, &map_q, q_full, head * AT_D, tl * AT_BM - rshift, req);
        tma_load_3d(sQ + t * AT_TILE_BYTES + AT_TILE_BYTES / 2, &map_q, q_full, head * AT_D + 64,
                    tl * AT_BM - rshift, req);
      }
      auto load_k = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], AT_TILE_BYTES);
        uint8_t* k = sK + st * AT_TILE_BYTES;
        tma_load_3d(k, &map_k, &k_full[st], kvh * AT_D, (jb + j) * AT_BN, req);
        tma_load_3d(k + AT_TILE_BYTES / 2, &map_k, &k_full[st], kvh * AT_D + 64, (jb + j) * AT_BN, req);
      };
      auto load_v = [&](int j) {
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], AT_TILE_BYTES);
        uint8_t* v = sV + st * AT_TILE_BYTES;
        tma_load_3d(v, &map_v, &v_full[st], kvh * AT_D, (jb + j) * AT_BN, req);
        tma_load_3d(v + AT_TILE_BYTES / 2, &map_v, &v_full[st], kvh * AT_D + 64, (jb + j) * AT_BN, req);
      };
      load_k(0);
      for (int j = 0; j < nmax; ++j) {
        if (j + 1 < nmax) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    if (nmax > 0) {  // ---------------- MMA issuer (converged warp, elected lane)
      constexpr uint32_t idesc_s = idesc_bf16_f32(AT_BM, AT_BN);
      constexpr uint32_t idesc_o = idesc_bf16_f32(AT_BM, AT_D) | (1u << 16);  // B (V) MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int t, int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint8_t* q = sQ + t * AT_TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {
          const uint64_t a = umma_desc_k_sw128(q + (kk >> 2) * (AT_TILE_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
          const uint64_t b = umma_desc_k_sw128(sK + st * AT_TILE_BYTES + (kk >> 2) * (AT_TILE_BYTES / 2)) +
                             (uint64_t)((kk & 3) * 2);
          mma_bf16_e(tmem + t * 128, a, b, idesc_s, kk != 0);
        }
        mma_commit_e(&s_full[t]);
        const bool last_user = (t == 1) || (j >= nt1);
        if (last_user) mma_commit_e(&k_empty[st]);
      };
      auto issue_pv = [&](int t, int j) {
        const int st = j & 1;
        mbar_wait(&p_full[t], j & 1);
        mbar_wait(&v_full[st], (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_BN / 16; ++kk) {
          const uint64_t b = umma_desc_mn_sw128(sV + st * AT_TILE_BYTES + kk * 16 * 128);
          // P (packed bf16) of keys 16kk..16kk+15: each softmax thread writes its W keys at the start
          // of its own S columns -> col = ch*W + (16kk mod W)/2
          constexpr int W = A2Cfg<SPLIT>::W;
          const uint32_t pa = tmem + t * 128 + (kk * 16 / W) * W + ((kk * 16) % W) / 2;
          mma_bf16_ts_e(tmem + 256 + t * 128, pa, b, idesc_o, (j | kk) != 0);
        }
        const bool last_user = (t == 1) || (j >= nt1);
        if (last_user) mma_commit_e(&v_empty[st]);
        if (j == (t ? nt1 : nt0) - 1) mma_commit_e(&o_full[t]);
      };
      if (nt0 > 0) issue_s(0, 0);
      if (nt1 > 0) issue_s(1, 0);
      for (int j = 0; j < nmax; ++j) {
        if (j < nt0) {
          issue_pv(0, j);
          if (j + 1 < nt0) issue_s(0, j + 1);
        }
        if (j < nt1) {
          issue_pv(1, j);
          if (j + 1 < nt1) issue_s(1, j + 1);
        }
      }
    }
  } else if (SPLIT == 1) {  // ---------------- softmax / rescale / epilogue: warps 2..9, one row per thread
    const int t = (warp - 2) >> 2;        // query tile
    const int g = warp & 3;               // TMEM lane quarter
    const int r = g * 32 + lane;
    const int n_my = t ? nt1 : nt0;
    const int my_tile = t ? tile1 : tile0;
    const int row = my_tile * AT_BM - rshift + r;
    const int my_kmax = (my_tile >= 0 && row >= 0 && row < M) ? kmax[row] : -1;
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tO = tmem + 256 + t * 128 + lane_off;
    const uint64_t sc2 = f2(scale_log2, scale_log2);
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_my; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      const int lim = my_kmax - (jb + j) * AT_BN;  // columns <= lim are visible
      const bool all_vis = __all_sync(0xffffffffu, lim >= 127);
      const bool none_vis = __all_sync(0xffffffffu, lim < 0);
      uint32_t v0[32], v1[32], v2[32], v3[32];   // the whole S row stays in registers
      tmem_ld32(tS + 0, v0);
      tmem_ld32(tS + 32, v1);
      tmem_ld32(tS + 64, v2);
      tmem_ld32(tS + 96, v3);
      tmem_ld_wait();
#define SROW(i) __uint_as_float((i) < 32 ? v0[(i) & 31] : (i) < 64 ? v1[(i) & 31] : (i) < 96 ? v2[(i) & 31] : v3[(i) & 31])
      float pmax = -INFINITY;
      if (all_vis) {
#pragma unroll
        for (int i = 0; i < 128; i += 2) pmax = fmax3(pmax, SROW(i), SROW(i + 1));
      } else if (!none_vis) {
#pragma unroll
        for (int i = 0; i < 128; ++i) pmax = fmaxf(pmax, i <= lim ? SROW(i) : -INFINITY);
      }
      const float tmax = pmax * scale_log2;
      const bool need = tmax > m_ref + 8.f;  // lazily move the reference max
      float alpha = 1.f;
      if (need) {
        alpha = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - tmax);
        m_ref = tmax;
        l *= alpha;
      }
      const uint64_t nm2 = f2(-m_ref, -m_ref);
      // P = exp2(s*scale - m_ref) as packed bf16 into S columns 0..63 (S is in registers)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        uint32_t pk[16];
        if (none_vis) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = 0u;
        } else if (all_vis) {
          uint64_t l2 = f2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t x2 = ffma2(f2(SROW(hh * 32 + i), SROW(hh * 32 + i + 1)), sc2, nm2);
            uint64_t p2;
            if (A2_EMU(i >> 1)) {
              p2 = exp2_poly2(x2);
            } else {
              float a, b;
              f2_split(x2, a, b);
              p2 = f2(ex2_approx(a), ex2_approx(b));
            }
            l2 = fadd2(l2, p2);
            float p0, p1;
            f2_split(p2, p0, p1);
            pk[i >> 1] = bf16x2_bits(p0, p1);
          }
          float la, lb;
          f2_split(l2, la, lb);
          l += la + lb;
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const int c0 = hh * 32 + i;
            float p0 = ex2_approx(fmaf(SROW(c0), scale_log2, -m_ref));
            float p1 = ex2_approx(fmaf(SROW(c0 + 1), scale_log2, -m_ref));
            p0 = (c0 <= lim) ? p0 : 0.f;
            p1 = (c0 + 1 <= lim) ? p1 : 0.f;
            l += p0 + p1;
            pk[i >> 1] = bf16x2_bits(p0, p1);
          }
        }
        tmem_st16(tS + hh * 16, pk);
      }
#undef SROW
      // lazy O rescale; PV(t, j-1) is complete (S(t, j) was issued after it, in order)
      if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
          uint32_t o[32];
          tmem_ld32(tO + hh * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tO + hh * 32, o);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    if (n_my > 0) {  // epilogue: O / l for the whole row
      mbar_wait(&o_full[t], 0);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        uint32_t o[32];
        tmem_ld32(tO + hh * 32, o);
        tmem_ld_wait();
        if (row < M && my_kmax >= 0) {
          __nv_bfloat16* dst = out + ((int64_t)row * H + head) * AT_D + hh * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 pk4;
            __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk4);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              p2[u] = __floats2bfloat162_rn(__uint_as_float(o[i + 2 * u]) * inv,
                                            __uint_as_float(o[i + 2 * u + 1]) * inv);
            *reinterpret_cast<uint4*>(dst + i) = pk4;
          }
        }
      }
    }
  } else {  // ---------------- SPLIT == 2: softmax / rescale / epilogue: warps 2..17, half rows
    const int t = (warp - 2) >> 3;        // query tile
    const int ch = ((warp - 2) >> 2) & 1; // column half: keys / output dims 64ch..64ch+63
    const int g = warp & 3;               // TMEM lane quarter
    const int r = g * 32 + lane;
    const int n_my = t ? nt1 : nt0;
    const int my_tile = t ? tile1 : tile0;
    const int row = my_tile * AT_BM - rshift + r;
    const int my_kmax = (my_tile >= 0 && row >= 0 && row < M) ? kmax[row] : -1;
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tO = tmem + 256 + t * 128 + lane_off;
    const int bar_id = 1 + t * 4 + g;     // the 2 warps (column halves) of these 32 rows
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_my; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      const int lim = my_kmax - (jb + j) * AT_BN - ch * 64;  // columns <= lim are visible
      const bool all_vis = __all_sync(0xffffffffu, lim >= 63);
      const bool none_vis = __all_sync(0xffffffffu, lim < 0);
      float pmax = -INFINITY;
      if (!none_vis) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // pass 1: row max over this half's 64 columns
          uint32_t v[32];
          tmem_ld32(tS + ch * 64 + hh * 32, v);
          tmem_ld_wait();
          if (all_vis) {
            {  // two independent max chains (shorter dependency chain)
          float pm1 = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            pmax = fmax3(pmax, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            pm1 = fmax3(pm1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
          }
          pmax = fmaxf(pmax, pm1);
        }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              pmax = fmaxf(pmax, (hh * 32 + i <= lim) ? __uint_as_float(v[i]) : -INFINITY);
          }
        }
      }
      red[t][j & 1][ch][r] = pmax * scale_log2;
      named_bar(bar_id, 64);
      const float tmax = fmaxf(red[t][j & 1][0][r], red[t][j & 1][1][r]);
      const bool need = tmax > m_ref + 8.f;  // lazily move the reference max
      float alpha = 1.f;
      if (need) {
        alpha = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - tmax);
        m_ref = tmax;
        l *= alpha;
      }
      // pass 2: P = exp2(s*scale - m_ref) as packed bf16 over the first 32 of this
      // half's own 64 S columns (P cols 64ch + 16hh .. +15): no overlap with the
      // other half's S, so no second exchange is needed before the store
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t pk[16];
        if (none_vis) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = 0u;
        } else {
          uint32_t v[32];
          tmem_ld32(tS + ch * 64 + hh * 32, v);
          tmem_ld_wait();
          if (all_vis) {
            const uint64_t sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m_ref, -m_ref);
            uint64_t l2 = f2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const uint64_t x2 = ffma2(f2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sc2, nm2);
              uint64_t p2;
              if (A2_EMU(i >> 1)) {
                p2 = exp2_poly2(x2);
              } else {
                float a, b;
                f2_split(x2, a, b);
                p2 = f2(ex2_approx(a), ex2_approx(b));
              }
              l2 = fadd2(l2, p2);
              float p0, p1;
              f2_split(p2, p0, p1);
              pk[i >> 1] = bf16x2_bits(p0, p1);
            }
            float la, lb;
            f2_split(l2, la, lb);
            l += la + lb;
          } else {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              float p0 = ex2_approx(fmaf(__uint_as_float(v[i]), scale_log2, -m_ref));
              float p1 = ex2_approx(fmaf(__uint_as_float(v[i + 1]), scale_log2, -m_ref));
              p0 = (hh * 32 + i <= lim) ? p0 : 0.f;
              p1 = (hh * 32 + i + 1 <= lim) ? p1 : 0.f;
              l += p0 + p1;
              pk[i >> 1] = bf16x2_bits(p0, p1);
            }
          }
        }
        tmem_st16(tS + ch * 64 + hh * 16, pk);
      }
      // lazy O rescale; PV(t, j-1) is complete (S(t, j) was issued after it, in order)
      if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t o[32];
          tmem_ld32(tO + ch * 64 + hh * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tO + ch * 64 + hh * 32, o);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    // split-KV: this CTA's piece of the row -> (max, sum) + unnormalised fp32 O
    if (n_split > 1 && my_tile >= 0) {
      const int64_t base = (((int64_t)req * H + head) * n_qt + my_tile) * n_split + chunk;
      float lt = 0.f;
      if (n_my > 0) {
        named_bar(bar_id, 64);
        red[t][0][ch][r] = l;
        named_bar(bar_id, 64);
        lt = red[t][0][0][r] + red[t][0][1][r];
        mbar_wait(&o_full[t], 0);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t o[32];
          tmem_ld32(tO + ch * 64 + hh * 32, o);
          tmem_ld_wait();
          float* dst = ws_o + (base * AT_BM + r) * AT_D + ch * 64 + hh * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(o[i]), __uint_as_float(o[i + 1]),
                                                              __uint_as_float(o[i + 2]), __uint_as_float(o[i + 3]));
        }
      }
      if (ch == 0) ws_ml[base * AT_BM + r] = make_float2(n_my > 0 ? m_ref : -INFINITY, lt);
    } else if (n_my > 0) {
      // epilogue: combine the two half-row sums, then O / l for this warp's 64 output dims
      named_bar(bar_id, 64);
      red[t][0][ch][r] = l;
      named_bar(bar_id, 64);
      const float lt = red[t][0][0][r] + red[t][0][1][r];
      mbar_wait(&o_full[t], 0);
      tc_fence_after();
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t o[32];
        tmem_ld32(tO + ch * 64 + hh * 32, o);
        tmem_ld_wait();
        if (row < M && my_kmax >= 0) {
          __nv_bfloat16* dst = out + ((int64_t)row * H + head) * AT_D + ch * 64 + hh * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 pk4;
            __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk4);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              p2[u] = __floats2bfloat162_rn(__uint_as_float(o[i + 2 * u]) * inv,
                                            __uint_as_float(o[i + 2 * u + 1]) * inv);
            *reinterpret_cast<uint4*>(dst + i) = pk4;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// split-KV combine: out[row, head] = sum_c 2^(m_c - M) O_c / sum_c 2^(m_c - M) l_c
// (m in the log2 domain of the kernel's lazy reference max). One warp per
// (row, head), 4 output dims per lane.
__global__ void __launch_bounds__(128) attn_combine_kernel(const float* __restrict__ ws_o,
                                                           const float2* __restrict__ ws_ml, int M, int H,
                                                           int n_split, __nv_bfloat16* __restrict__ out,
                                                           int rshift) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.x * 4 + warp;
  const int row = blockIdx.y, req = blockIdx.z;
  if (head >= H) return;
  const int n_qt = (M + AT_BM - 1) / AT_BM;
  const int tile = (row + rshift) / AT_BM, r = (row + rshift) % AT_BM;
  const int64_t base0 = (((int64_t)req * H + head) * n_qt + tile) * n_split;
  float mx = -INFINITY;
  for (int c = 0; c < n_split; ++c) mx = fmaxf(mx, ws_ml[(base0 + c) * AT_BM + r].x);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float L = 0.f;
  for (int c = 0; c < n_split; ++c) {
    const float2 ml = ws_ml[(base0 + c) * AT_BM + r];
    if (ml.x == -INFINITY) continue;
    const float w = ex2_approx(ml.x - mx);
    const float4 o = *reinterpret_cast<const float4*>(ws_o + ((base0 + c) * AT_BM + r) * AT_D + lane * 4);
    acc.x += w * o.x; acc.y += w * o.y; acc.z += w * o.z; acc.w += w * o.w;
    L += w * ml.y;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv), hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  *reinterpret_cast<uint2*>(out + (((int64_t)req * M + row) * H + head) * AT_D + lane * 4) =
      make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

size_t attention_workspace(int64_t m, int n_req, int h, int n_split) {
  if (n_split <= 1) return 0;
  const int64_t n_qt = (m + AT_BM - 1) / AT_BM;
  return (size_t)n_req * h * n_qt * n_split * AT_BM * (AT_D * sizeof(float) + sizeof(float2)) + 256;
}

static int g_attn_ver = -1;  // QCF_ATTN env / qcf_set_attention_kernel: 1 = single-tile, 2 = ping-pong (default)

static int g_attn_split = 2;  // v2 softmax layout: 2 = half rows (default), 1 = full row per thread (knob 3)

void set_attention_kernel(int v) {
  g_attn_split = (v == 3) ? 1 : 2;
  if (v == 3) v = 2;
  g_attn_ver = (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
}

static int g_attn_nsplit = -1;  // QCF_ATTN_SPLIT env / qcf_set_attention_split: split-KV factor (one-wave grids)

void set_attention_split(int n) { g_attn_nsplit = n > 0 ? n : 0; }

// split-KV factor for a one-wave grid: ~2 waves of CTAs, at most 8 chunks
int attention_auto_split(int64_t m, int n_req, int h, int64_t n_keys) {
  if (g_attn_nsplit < 0) {
    const char* e = getenv("QCF_ATTN_SPLIT");
    g_attn_nsplit = e ? std::max(1, atoi(e)) : 0;
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  const int64_t n_pairs = ((m + AT_BM - 1) / AT_BM + 1) / 2;
  const int64_t grid = (int64_t)h * n_pairs * n_req;
  if (grid > sms) return 1;
  if (g_attn_nsplit > 0) return g_attn_nsplit;
  // auto only for grids far below one wave (query-only / decode-like shapes: a few
  // tiles over a long key range); at the one-request recompute shape (128 pairs)
  // single tiles measured faster (tools/attn_bench.py)
  if (grid * 4 > sms) return 1;
  const int64_t sp = std::min<int64_t>(8, std::max<int64_t>(2, (2 * sms + grid - 1) / grid));
  // at least four key tiles per chunk: the probe's anchor prefix (293 keys = 3 tiles)
  // stays whole -- split in two plus the combine it measured 12.7 vs 7.9 us
  return (int)std::min<int64_t>(sp, std::max<int64_t>(1, n_keys / (4 * AT_BN)));
}

int attention_tc_launch(const void* q, const void* k, const void* v, const int32_t* kmax, int64_t m, int h,
                        int hkv, int d, int64_t n_keys, void* out, cudaStream_t s, int n_req, void* ws,
                        size_t ws_bytes) {
  if (d != AT_D || m > INT32_MAX || n_keys > INT32_MAX || n_req > 65535) return QCF_EUNSUPPORTED;
  if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out) & 15) return QCF_EUNSUPPORTED;
  CUtensorMap mq, mk, mv;
  const int64_t qw = (int64_t)h * d, kw = (int64_t)hkv * d;
  int st = make_kmajor_map3(&mq, q, m, qw, qw, AT_BM, n_req, m * qw);
  if (st == QCF_OK) st = make_kmajor_map3(&mk, k, n_keys, kw, kw, AT_BN, n_req, n_keys * kw);
  if (st == QCF_OK) st = make_kmajor_map3(&mv, v, n_keys, kw, kw, AT_BN, n_req, n_keys * kw);
  if (st != QCF_OK) return st;
  if (g_attn_ver < 0) {
    const char* e = getenv("QCF_ATTN");
    g_attn_ver = (e && atoi(e) == 1) ? 1 : (e && atoi(e) == 2) ? 2 : (e && atoi(e) == 4) ? 4 : 0;  // 0 = by grid size
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_tc2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, A2_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_tc2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, A2_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_tc4_kernel<4, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, A4_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_tc8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, A8_SMEM);

    if (e != cudaSuccess) return cuda_status(e, "attn_tc attr");
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)d);
  const int n_qt = (int)((m + AT_BM - 1) / AT_BM);
  const int n_pairs = (n_qt + 1) / 2;
  // the partial query tile goes FIRST (rows sorted by position -> it is the one
  // with the fewest keys); the query rows at the end then fill a whole tile
  const int rshift = (int)((AT_BM - m % AT_BM) % AT_BM);
  // auto: tile pairs when they span more than one wave; a one-wave grid either
  // splits every pair's key range (split-KV + combine; needs the workspace and
  // QCF_ATTN_SPLIT) or runs single tiles (default: measured faster on B200)
  int n_split = 1;
  if (g_attn_ver == 0 && g_attn_split == 2 && ws) {
    n_split = attention_auto_split(m, n_req, h, n_keys);
    if (n_split > 1 && ws_bytes < attention_workspace(m, n_req, h, n_split)) n_split = 1;
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  // auto (tools/attn_bench.py, profiles/r2s3_attn_versions*.jsonl): v4 (two CTAs per SM
  // over 64-key tiles) once the grid fills both CTA slots of every SM -- batch recompute
  // 8 x 800 rows: 337 vs 366 us (v1), GQA-8 307 vs 381, full prefill 205 vs 232, Mistral
  // 32k 1141 vs 1202 -- or fills one slot with short uniform key ranges (probe rows of 8
  // requests: 10 vs 14 us); smaller grids of uneven tiles (one request: 224) run v1
  // (72-76 us for v4: its longest tiles would share SMs while others idle; v8 is 44 vs
  // 48 us alone but measured slower inside the step: TTFT 13.29 vs 13.0-13.2 ms);
  // split-KV grids on the pairs
  const int64_t ctas = (int64_t)h * n_qt * n_req;
  const int ver = g_attn_ver ? g_attn_ver
                             : n_split > 1 ? 2
                             : (ctas >= 2 * sms || (ctas > sms && n_keys <= 4 * AT_BN)) ? 4 : 1;
  if (ver == 2) {
    static int pair_mode = -1;  // QCF_ATTN_PAIR: 0 adjacent (default), 1 mirrored
    if (pair_mode == -1) {
      const char* e = getenv("QCF_ATTN_PAIR");
      pair_mode = e ? atoi(e) : 0;
    }
    float* ws_o = n_split > 1 ? reinterpret_cast<float*>(ws) : nullptr;
    float2* ws_ml = n_split > 1 ? reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(ws) +
                                                            (size_t)n_req * h * n_qt * n_split * AT_BM * AT_D * 4)
                                : nullptr;
    dim3 grid((unsigned)h, (unsigned)(n_pairs * n_split), (unsigned)n_req);
    if (g_attn_split == 2)
      QCF_LAUNCH("attn_tc2_kernel<2>", attn_tc2_kernel<2>, dim3(grid), dim3(A2Cfg<2>::THREADS), A2_SMEM, s, mq, mk, mv,
                 kmax, (int)m, h, hkv, (int)n_keys, scale_log2, (__nv_bfloat16*)out, pair_mode, n_split, ws_o, ws_ml,
                 rshift);
    else
      QCF_LAUNCH("attn_tc2_kernel<1>", attn_tc2_kernel<1>, dim3(grid), dim3(A2Cfg<1>::THREADS), A2_SMEM, s, mq, mk, mv,
                 kmax, (int)m, h, hkv, (int)n_keys, scale_log2, (__nv_bfloat16*)out, pair_mode, 1,
                 (float*)nullptr, (float2*)nullptr, rshift);
    QCF_LAUNCH_CHECK("qcf_attention(tcgen05 pairs)");
    if (n_split > 1) {
      QCF_LAUNCH("attn_combine_kernel", attn_combine_kernel, dim3((unsigned)((h + 3) / 4), (unsigned)m, (unsigned)n_req),
                 dim3(128), 0, s, (const float*)ws_o, (const float2*)ws_ml, (int)m, h, n_split, (__nv_bfloat16*)out,
                 rshift);
    }
  } else if (ver == 8) {
    dim3 grid((unsigned)h, (unsigned)n_qt, (unsigned)n_req);
    QCF_LAUNCH("attn_tc8_kernel", attn_tc8_kernel, dim3(grid), dim3(A8_THREADS), A8_SMEM, s, mq, mk, mv, kmax, (int)m,
               h, hkv, (int)n_keys, scale_log2, (__nv_bfloat16*)out, rshift);
  } else if (ver == 4) {
    CUtensorMap mk4, mv4;   // 64-key boxes
    st = make_kmajor_map3(&mk4, k, n_keys, kw, kw, A4_BN, n_req, n_keys * kw);
    if (st == QCF_OK) st = make_kmajor_map3(&mv4, v, n_keys, kw, kw, A4_BN, n_req, n_keys * kw);
    if (st != QCF_OK) return st;
    dim3 grid((unsigned)h, (unsigned)n_qt, (unsigned)n_req);
    QCF_LAUNCH("attn_tc4_kernel", (attn_tc4_kernel<4, 7>), dim3(grid), dim3(64 + 4 * 32), A4_SMEM, s, mq, mk4, mv4,
               kmax, (int)m, h, hkv, (int)n_keys, scale_log2, (__nv_bfloat16*)out, rshift);
  } else {
    dim3 grid((unsigned)h, (unsigned)n_qt, (unsigned)n_req);
    QCF_LAUNCH("attn_tc_kernel", attn_tc_kernel, dim3(grid), dim3(AT_THREADS), AT_SMEM, s, mq, mk, mv, kmax, (int)m,
               h, hkv, (int)n_keys, scale_log2, (__nv_bfloat16*)out, rshift);
  }
  QCF_LAUNCH_CHECK("qcf_attention(tcgen05)");
  return QCF_OK;
}

}  // namespace qcf

#ifdef QCF_ATTN_TRACE
extern "C" int qcf_debug_set_attn_trace(void* buf) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(qcf::g_attn_trace, &p, sizeof(p)) == cudaSuccess ? 0 : -1;
}
extern "C" int qcf_debug_set_attn_trace2(void* buf) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(qcf::g_attn_trace2, &p, sizeof(p)) == cudaSuccess ? 0 : -1;
}
#endif
