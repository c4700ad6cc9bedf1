// K5: Top-N token selection (fusion.py:141-158). The reference sorts
// -float64(score) with a stable argsort, keeps the first N and returns them
// ascending + 1. Equivalent single-CTA formulation: an 8-bit-digit radix
// select finds the N-th largest key T (keys are the order-preserving uint32
// image of the float32 scores), then an index-ordered block scan keeps every
// key > T plus the first N - count(> T) keys == T (ties -> lower index) and
// compacts them in ascending order. Bit-exact by construction.
// Key map = the order numpy's stable argsort of -float64(score) induces:
// -0.0 and +0.0 compare equal (one key, so the lower index wins), and NaN
// sorts after every number (key 0: selected last, lower index first).
// float64 scores (the public select_topn, fusion.py:156) use 64-bit keys
// and 8 digit passes instead of 4.
#include "common.cuh"

namespace qcf {

constexpr int TN_THREADS = 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
  if (f != f) return 0u;                       // NaN: after every number
  uint32_t b = __float_as_uint(f);
  if (b == 0x80000000u) b = 0u;                // -0.0 == +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t order_key(double f) {
  if (f != f) return 0ull;
  uint64_t b = (uint64_t)__double_as_longlong(f);
  if (b == 0x8000000000000000ull) b = 0ull;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename S> struct KeyOf;
template <> struct KeyOf<float> { using T = uint32_t; };
template <> struct KeyOf<double> { using T = uint64_t; };

// inclusive block scan of one int per thread (1024 threads)
__device__ __forceinline__ int block_scan_incl(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) warp_tot[w] = v;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    warp_tot[lane] = t;  // inclusive prefix of warp totals
  }
  __syncthreads();
  const int add = w > 0 ? warp_tot[w - 1] : 0;
  total = warp_tot[31];
  __syncthreads();
  return v + add;
}

// One CTA per request (blockIdx.x). Keys are staged once in shared memory when
// they fit (n <= TN_SMEM_KEYS), so the 4 radix passes and the compaction re-read
// on-chip memory instead of L2. `dst` (optional) receives idx + r*dst_add, the
// request's rows in the batched fused table (the recompute scatter targets).
constexpr int TN_SMEM_KEYS = 48 * 1024;

template <bool SMEM, typename S>
__global__ void __launch_bounds__(TN_THREADS) topn_kernel(const S* __restrict__ scores, int64_t n,
                                                          int64_t n_sel, int32_t base,
                                                          int32_t* __restrict__ out, int64_t out_stride,
                                                          int32_t* __restrict__ dst, int32_t dst_add) {
  using K = typename KeyOf<S>::T;
  constexpr int TOP = 8 * (int)sizeof(K) - 8;
  extern __shared__ __align__(16) unsigned char s_raw[];
  K* s_keys = reinterpret_cast<K*>(s_raw);
  __shared__ int hist[256];
  __shared__ int warp_tot[32];
  __shared__ K s_prefix;
  __shared__ int s_need;
  const int tid = threadIdx.x;
  const int req = blockIdx.x;
  scores += (int64_t)req * n;
  out += (int64_t)req * out_stride;
  if (dst) dst += (int64_t)req * out_stride;
  const int32_t dadd = req * dst_add;
  if (tid == 0) { s_prefix = 0; s_need = (int)n_sel; }
  pdl_wait();
  pdl_trigger();
  if (SMEM) {
    for (int64_t i = tid; i < n; i += blockDim.x) s_keys[i] = order_key(scores[i]);
  }
  auto key_at = [&](int64_t i) -> K { return SMEM ? s_keys[i] : order_key(scores[i]); };
  // ---- radix select of the n_sel-th largest key, digits of 8 bits (MSB first)
  for (int shift = TOP; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const K prefix = s_prefix;
    const K hi_mask = shift == TOP ? (K)0 : (~(K)0 << (shift + 8));
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const K key = key_at(i);
      if ((key & hi_mask) == (prefix & hi_mask)) atomicAdd(&hist[(key >> shift) & 0xff], 1);
    }
    __syncthreads();
    if (tid < 32) {  // warp 0: find the digit holding the need-th largest key
      const int need = s_need;
      __syncwarp();    // every lane has read s_need before the owning lane rewrites it
      // suffix sums over the 256 bins, 8 per lane, highest bins in lane 31
      int cnt[8], tot = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) { cnt[u] = hist[tid * 8 + u]; tot += cnt[u]; }
      int suf = tot;  // inclusive suffix sum over lanes >= tid
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_down_sync(0xffffffffu, suf, o);
        if (tid + o < 32) suf += t;
      }
      const int above = suf - tot;  // keys in bins of lanes > tid
      // the lane whose bins contain the need-th largest key
      const bool mine = above < need && above + tot >= need;
      if (mine) {
        int rem = need - above, b = tid * 8 + 7;
        for (int u = 7; u > 0; --u, --b) {
          if (cnt[u] >= rem) break;
          rem -= cnt[u];
        }
        s_prefix = prefix | ((K)b << shift);
        s_need = rem;  // how many keys equal to the final threshold must be taken
      }
    }
    __syncthreads();
  }
  const K T = s_prefix;
  const int need_eq = s_need;
  // ---- ordered compaction: key > T always, key == T for the first need_eq (index order)
  int eq_before = 0, sel_before = 0;
  for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const int64_t i = c0 + tid;
    const K key = i < n ? key_at(i) : (K)0;
    const int is_eq = (i < n && key == T) ? 1 : 0;
    int eq_total;
    const int eq_incl = block_scan_incl(is_eq, warp_tot, eq_total);
    const int take = (i < n) && (key > T || (is_eq && eq_before + eq_incl <= need_eq)) ? 1 : 0;
    int sel_total;
    const int sel_incl = block_scan_incl(take, warp_tot, sel_total);
    if (take) {
      const int slot = sel_before + sel_incl - 1;
      out[slot] = (int32_t)i + base;
      if (dst) dst[slot] = (int32_t)i + base + dadd;
    }
    eq_before += eq_total;
    sel_before += sel_total;
    if (sel_before >= n_sel) break;  // uniform across the block
  }
}

template <typename S>
static int topn_launch(const S* scores, int64_t n, int n_req, int64_t n_sel, int32_t base, int32_t* idx_out,
                       int64_t out_stride, int32_t* dst_out, int32_t dst_add, qcf_stream_t stream) {
  QCF_REQUIRE(scores && (idx_out || n_sel == 0), QCF_EINVAL, "qcf_topn: null pointer");
  QCF_REQUIRE(n >= 0 && n_sel >= 0 && n_sel <= n && n_req >= 1, QCF_EINVAL, "qcf_topn: need 0 <= n_sel <= n");
  QCF_REQUIRE(n_req == 1 || out_stride >= n_sel, QCF_EINVAL, "qcf_topn: output stride < n_sel");
  QCF_REQUIRE(n < 0x7fffffff, QCF_EUNSUPPORTED, "qcf_topn: n too large");
  if (n_sel == 0) return QCF_OK;
  auto s = as_stream(stream);
  constexpr int64_t kSmemKeys = TN_SMEM_KEYS * 4 / (int64_t)sizeof(typename KeyOf<S>::T);
  if (n <= kSmemKeys) {
    static bool attr = false;
    const size_t smem = (size_t)n * sizeof(typename KeyOf<S>::T);
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(topn_kernel<true, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           TN_SMEM_KEYS * (int)sizeof(uint32_t));
      if (e != cudaSuccess) return cuda_status(e, "qcf_topn attr");
      attr = true;
    }
    QCF_LAUNCH("topn_kernel", (topn_kernel<true, S>), dim3(n_req), dim3(TN_THREADS), smem, s, scores, n, n_sel,
               base, idx_out, out_stride, dst_out, dst_add);
  } else {
    QCF_LAUNCH("topn_kernel", (topn_kernel<false, S>), dim3(n_req), dim3(TN_THREADS), 0, s, scores, n, n_sel,
               base, idx_out, out_stride, dst_out, dst_add);
  }
  QCF_LAUNCH_CHECK("qcf_topn");
  return QCF_OK;
}
}  // namespace qcf

extern "C" size_t qcf_topn_workspace(int64_t n) { (void)n; return 0; }

extern "C" int qcf_topn_batched(const float* scores, int64_t n, int n_req, int64_t n_sel, int32_t base,
                                int32_t* idx_out, int64_t out_stride, int32_t* dst_out, int32_t dst_add,
                                qcf_stream_t stream) {
  return qcf::topn_launch<float>(scores, n, n_req, n_sel, base, idx_out, out_stride, dst_out, dst_add, stream);
}

extern "C" int qcf_topn(const float* scores, int64_t n, int64_t n_sel, int32_t base,
                        int32_t* idx_out, void* workspace, size_t ws_bytes, qcf_stream_t stream) {
  (void)workspace; (void)ws_bytes;
  return qcf_topn_batched(scores, n, 1, n_sel, base, idx_out, n_sel, nullptr, 0, stream);
}

extern "C" int qcf_topn_f64(const double* scores, int64_t n, int64_t n_sel, int32_t base, int32_t* idx_out,
                            qcf_stream_t stream) {
  return qcf::topn_launch<double>(scores, n, 1, n_sel, base, idx_out, n_sel, nullptr, 0, stream);
}
