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

#include "attention.cuh"
#include "sm100.cuh"

namespace qcf {

using namespace sm100;

int make_kmajor_map3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld, int box_rows,
                     int64_t batch, int64_t batch_stride);

constexpr int AT_BM = 128, AT_BN = 128, AT_D = 128;
constexpr int AT_THREADS = 576;  // 2 control warps + 16 softmax warps
constexpr int AT_TILE_BYTES = AT_BM * AT_D * 2;  // 32 KB: two 16 KB SW128 atoms
constexpr int AT_SMEM = AT_TILE_BYTES * 6 + 1024 + 256;  // Q, K[2], V[2], P

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

__global__ void __launch_bounds__(AT_THREADS, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
               const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ kmax, int M, int H,
               int Hkv, int n_keys, float scale_log2, __nv_bfloat16* __restrict__ out) {
  // request (batch) index: q/out/kmax are [req][M]..., the K/V tables [req][n_keys]...
  const int req = blockIdx.z;
  kmax += (int64_t)req * M;
  out += (int64_t)req * M * H * AT_D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + AT_TILE_BYTES;          // [2]
  uint8_t* sV = smem + 3 * AT_TILE_BYTES;      // [2]
  uint8_t* sP = smem + 5 * AT_TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * AT_TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;     // [2]  K ring: freed as soon as S_j is computed
  uint64_t* k_empty = bars + 3;    // [2]
  uint64_t* s_full = bars + 5;     // [2]
  uint64_t* s_free = bars + 7;     // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* pv_done = bars + 10;
  uint64_t* v_full = bars + 11;    // [2]  V ring: freed when P_j.V_j is done
  uint64_t* v_empty = bars + 13;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);
  __shared__ float red[2][4][AT_BM];   // per-tile partial row max (double-buffered by tile parity)
  __shared__ int s_kend;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (M + AT_BM - 1) / AT_BM;
  const int qt = n_qt - 1 - blockIdx.y;  // longest tiles (largest positions) launch first
  const int head = blockIdx.x;
  const int kvh = head / (H / Hkv);
  const int m0 = qt * AT_BM;
  constexpr int N_SOFT = (AT_THREADS / 32 - 2) * 32;  // 512 softmax threads

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
      mbar_init(&s_free[s], N_SOFT);
    }
    mbar_init(p_full, N_SOFT);
    mbar_init(pv_done, 1);
    fence_barrier_init();
    s_kend = 0;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  __syncthreads();
  pdl_wait();  // barrier init + TMEM alloc overlap the previous kernel's tail
  pdl_trigger();
  // key range of this tile = 1 + max kmax over its rows (rows are normally
  // sorted by position, but the kernel does not rely on it)
  if (threadIdx.x < AT_BM) {
    int v = (m0 + (int)threadIdx.x < M) ? kmax[m0 + threadIdx.x] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s_kend, min(v + 1, n_keys));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_tiles = (s_kend + AT_BN - 1) / AT_BN;
  const uint32_t tS0 = tmem, tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_expect_tx(q_full, AT_TILE_BYTES);
      tma_load_3d(sQ, &map_q, q_full, head * AT_D, m0, req);
      tma_load_3d(sQ + AT_TILE_BYTES / 2, &map_q, q_full, head * AT_D + 64, m0, req);
      // K_j is consumed by S_j (early), V_j by P_j.V_j (late): two rings, and K
      // runs one tile ahead of V so S_{j+1} never waits on a V-gated slot
      auto load_k = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], AT_TILE_BYTES);
        uint8_t* k = sK + st * AT_TILE_BYTES;
        tma_load_3d(k, &map_k, &k_full[st], kvh * AT_D, j * AT_BN, req);
        tma_load_3d(k + AT_TILE_BYTES / 2, &map_k, &k_full[st], kvh * AT_D + 64, j * AT_BN, req);
      };
      auto load_v = [&](int j) {
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], AT_TILE_BYTES);
        uint8_t* v = sV + st * AT_TILE_BYTES;
        tma_load_3d(v, &map_v, &v_full[st], kvh * AT_D, j * AT_BN, req);
        tma_load_3d(v + AT_TILE_BYTES / 2, &map_v, &v_full[st], kvh * AT_D + 64, j * AT_BN, req);
      };
      load_k(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc_s = idesc_bf16_f32(AT_BM, AT_BN);                  // K-major A, K-major B
      constexpr uint32_t idesc_o = idesc_bf16_f32(AT_BM, AT_D) | (1u << 16);      // B (V) MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_pv = [&](int jj) {
        const int st = jj & 1;
        mbar_wait(p_full, jj & 1);
        mbar_wait(&v_full[st], (jj >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_BN / 16; ++kk) {
          const uint64_t a = umma_desc_k_sw128(sP + (kk >> 2) * (AT_TILE_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
          const uint64_t b = umma_desc_mn_sw128(sV + st * AT_TILE_BYTES + kk * 16 * 128);
          mma_bf16(tO, a, b, idesc_o, (jj | kk) != 0);
        }
        mma_commit(&v_empty[st]);
        mma_commit(pv_done);
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1, sb = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        mbar_wait(&s_free[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {
          const uint64_t a = umma_desc_k_sw128(sQ + (kk >> 2) * (AT_TILE_BYTES / 2)) + (uint64_t)((kk & 3) * 2);
          const uint64_t b = umma_desc_k_sw128(sK + st * AT_TILE_BYTES + (kk >> 2) * (AT_TILE_BYTES / 2)) +
                             (uint64_t)((kk & 3) * 2);
          mma_bf16(tS0 + sb * 128, a, b, idesc_s, kk != 0);
        }
        mma_commit(&s_full[sb]);
        mma_commit(&k_empty[st]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {  // ---------------- softmax / correction / epilogue (warps 2..17)
    const int g = warp & 3;               // TMEM lane quarter -> rows 32g..32g+31
    const int cg = (warp - 2) >> 2;       // column group: S keys / O dims 32cg..32cg+31
    const int r = g * 32 + lane;          // row within the tile == TMEM lane
    const int row = m0 + r;
    const int my_kmax = row < M ? kmax[row] : -1;
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const int bar_id = 1 + g;             // named barrier of the 4 warps sharing these rows
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tS0 + sb * 128 + cg * 32 + lane_off, v);
      tmem_ld_wait();
      const int lim = my_kmax - j * AT_BN - cg * 32;  // columns <= lim are visible
      const bool all_vis = __all_sync(0xffffffffu, lim >= 31);
      const bool none_vis = __all_sync(0xffffffffu, lim < 0);
      float pmax = -INFINITY;
      if (all_vis) {
#pragma unroll
        for (int i = 0; i < 32; ++i) pmax = fmaxf(pmax, __uint_as_float(v[i]));
      } else if (!none_vis) {
#pragma unroll
        for (int i = 0; i < 32; ++i) pmax = fmaxf(pmax, i <= lim ? __uint_as_float(v[i]) : -INFINITY);
      }
      red[sb][cg][r] = pmax * scale_log2;
      named_bar(bar_id, 128);
      const float tmax = fmaxf(fmaxf(red[sb][0][r], red[sb][1][r]), fmaxf(red[sb][2][r], red[sb][3][r]));
      // the previous P.V must be done before P is overwritten or O rescaled
      if (j > 0) {
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
      }
      const bool need = tmax > m_ref + 8.f;  // lazily move the reference max
      float alpha = 1.f;
      if (need) {
        alpha = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - tmax);
        m_ref = tmax;
        l *= alpha;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {  // rescale this warp's O slice in TMEM
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
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      // P = exp2(s*scale - m_ref) -> bf16, columns 32cg..32cg+31 of the SW128 K-major P tile
      uint32_t pk[16];
      float psum = 0.f;
      if (none_vis) {
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0u;
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p0 = ex2_approx(fmaf(__uint_as_float(v[i]), scale_log2, -m_ref));
          float p1 = ex2_approx(fmaf(__uint_as_float(v[i + 1]), scale_log2, -m_ref));
          if (!all_vis) {
            p0 = (i <= lim) ? p0 : 0.f;
            p1 = (i + 1 <= lim) ? p1 : 0.f;
          }
          psum += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pk[i >> 1] = *reinterpret_cast<uint32_t*>(&b2);
        }
      }
      l += psum;
      const uint32_t atom = smem_u32(sP + (cg >> 1) * (AT_TILE_BYTES / 2) + r * 128);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int chunk = ((cg & 1) * 4 + q) ^ (r & 7);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(atom + chunk * 16), "r"(pk[4 * q]),
                     "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3]) : "memory");
      }
      tc_fence_before();
      mbar_arrive(&s_free[sb]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
      mbar_arrive(p_full);
    }
    // epilogue: combine the 4 partial row sums, then O / l for this warp's 32 columns
    named_bar(bar_id, 128);
    red[0][cg][r] = l;
    named_bar(bar_id, 128);
    const float lt = (red[0][0][r] + red[0][1][r]) + (red[0][2][r] + red[0][3][r]);
    mbar_wait(pv_done, (n_tiles - 1) & 1);
    tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    uint32_t o[32];
    tmem_ld32(tO + cg * 32 + lane_off, o);
    tmem_ld_wait();
    if (row < M) {
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
  }
}

int attention_tc_launch(const void* q, const void* k, const void* v, const int32_t* kmax, int64_t m, int h,
                        int hkv, int d, int64_t n_keys, void* out, cudaStream_t s, int n_req) {
  if (d != AT_D || m > INT32_MAX || n_keys > INT32_MAX || n_req > 65535) return QCF_EUNSUPPORTED;
  if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out) & 15) return QCF_EUNSUPPORTED;
  CUtensorMap mq, mk, mv;
  const int64_t qw = (int64_t)h * d, kw = (int64_t)hkv * d;
  int st = make_kmajor_map3(&mq, q, m, qw, qw, AT_BM, n_req, m * qw);
  if (st == QCF_OK) st = make_kmajor_map3(&mk, k, n_keys, kw, kw, AT_BN, n_req, n_keys * kw);
  if (st == QCF_OK) st = make_kmajor_map3(&mv, v, n_keys, kw, kw, AT_BN, n_req, n_keys * kw);
  if (st != QCF_OK) return st;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    if (e != cudaSuccess) return cuda_status(e, "attn_tc attr");
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)d);
  dim3 grid((unsigned)h, (unsigned)((m + AT_BM - 1) / AT_BM), (unsigned)n_req);
  QCF_LAUNCH("attn_tc_kernel", attn_tc_kernel, dim3(grid), dim3(AT_THREADS), AT_SMEM, s, mq, mk, mv, kmax, (int)m, h, hkv, (int)n_keys, scale_log2,
                                                   (__nv_bfloat16*)out);
  QCF_LAUNCH_CHECK("qcf_attention(tcgen05)");
  return QCF_OK;
}

}  // namespace qcf
