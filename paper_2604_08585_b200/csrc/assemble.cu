// K1: fused-context assembly with RoPE re-alignment (fusion.py:234-263,
// model.py:271-292). HBM-bound: every chunk K/V element is read once and the
// fused table written once, with 16-byte vector accesses; the chunk offset
// rotation uses a float64 cos/sin table built on the host exactly as the
// reference builds its angles (model.py:278-281).
#include <stdlib.h>
#include "common.cuh"

namespace qcf {

template <typename T> struct Vec16;
template <> struct Vec16<float> { static constexpr int N = 4; };
template <> struct Vec16<__nv_bfloat16> { static constexpr int N = 8; };

__device__ __forceinline__ int find_chunk(const qcf_chunk_desc* ch, int n_chunks, int row) {
  int lo = 0, hi = n_chunks - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (ch[mid].offset <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// rotate the interleaved pairs of one 16-byte vector (value in, value out)
template <typename T>
__device__ __forceinline__ uint4 rotate_vec(uint4 raw, int j0, const double* ctab, const double* stab);

template <>
__device__ __forceinline__ uint4 rotate_vec<float>(uint4 raw, int j0, const double* ctab, const double* stab) {
  float4 x = *reinterpret_cast<float4*>(&raw);
  float4 y;
  rotate_pair_exact(x.x, x.y, ctab[j0], stab[j0], y.x, y.y);
  rotate_pair_exact(x.z, x.w, ctab[j0 + 1], stab[j0 + 1], y.z, y.w);
  return *reinterpret_cast<uint4*>(&y);
}

template <>
__device__ __forceinline__ uint4 rotate_vec<__nv_bfloat16>(uint4 raw, int j0, const double* ctab,
                                                           const double* stab) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&raw);
  uint4 outr;
  __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(&outr);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float2 f = __bfloat1622float2(p[t]);
    float oe, oo;
    rotate_pair_fast(f.x, f.y, (float)ctab[j0 + t], (float)stab[j0 + t], oe, oo);
    q[t] = __floats2bfloat162_rn(oe, oo);
  }
  return outr;
}

// One CTA per (run of ASM_ROWS fused rows, layer): the chunk descriptor is looked
// up only when a row leaves the cached chunk, and for bf16 the chunk's (cos, sin)
// row is staged once in shared memory as float pairs (the same float casts of the
// float64 table as before: bit-identical). Every thread moves ASM_UNROLL 16-byte
// vectors of K and of V per row with all loads issued before the stores.
constexpr int ASM_THREADS = 128, ASM_UNROLL = 4, ASM_ROWS = 4, ASM_MAX_HALF = 256;

template <typename T>
__global__ void __launch_bounds__(ASM_THREADS) assemble_kernel(
    const qcf_chunk_desc* __restrict__ chunks, int n_chunks, int n_rows /* 1 + n_ctx */,
    const T* __restrict__ bos_k, const T* __restrict__ bos_v, T* __restrict__ fk,
    T* __restrict__ fv, int64_t fstride, int row_elems, int d,
    const double* __restrict__ ctab, const double* __restrict__ stab, const int32_t* __restrict__ deltas,
    int layer0, const uint32_t* __restrict__ skip) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = Vec16<T>::N;
  constexpr bool kBf16 = sizeof(T) == 2;
  const int layer = layer0 + blockIdx.y;
  const int vpr = row_elems / V;
  const bool has_v = fv != nullptr;   // K only (fp32 scoring keys) when null
  const int half = d >> 1;
  __shared__ qcf_chunk_desc sc;
  __shared__ int64_t s_delta;
  __shared__ float2 s_cs[ASM_MAX_HALF];   // bf16: (float cos, float sin) of the chunk's delta
  int c_lo = 1, c_hi = 0;                 // fused rows of the cached chunk: [c_lo, c_hi)
  for (int run = blockIdx.x * ASM_ROWS; run < n_rows; run += gridDim.x * ASM_ROWS) {
    for (int row = run; row < min(run + ASM_ROWS, n_rows); ++row) {
      // rows the recompute rewrites in every layer (bit set) are not copied (CTA-uniform)
      if (skip && ((__ldg(skip + (row >> 5)) >> (row & 31)) & 1u)) continue;
      T* dk = fk + layer * fstride + (int64_t)row * row_elems;
      T* dv = fv + layer * fstride + (int64_t)row * row_elems;
      if (row == 0) {
        for (int i = threadIdx.x; i < vpr; i += blockDim.x) {
          reinterpret_cast<uint4*>(dk)[i] = reinterpret_cast<const uint4*>(bos_k + (int64_t)layer * row_elems)[i];
          if (has_v)
            reinterpret_cast<uint4*>(dv)[i] = reinterpret_cast<const uint4*>(bos_v + (int64_t)layer * row_elems)[i];
        }
        continue;
      }
      if (row < c_lo || row >= c_hi) {  // uniform: every thread tracks the same range
        __syncthreads();
        if (threadIdx.x == 0) {
          const int ci = find_chunk(chunks, n_chunks, row);
          sc = chunks[ci];
          s_delta = deltas ? deltas[ci] : sc.offset;  // rotation delta (default: the fused row)
        }
        __syncthreads();
        c_lo = sc.offset;
        c_hi = sc.offset + sc.n_tok;
        if (kBf16) {
          for (int t = threadIdx.x; t < half; t += blockDim.x)
            s_cs[t] = make_float2((float)ctab[s_delta * half + t], (float)stab[s_delta * half + t]);
          __syncthreads();
        }
      }
      const int64_t src_off = layer * sc.layer_stride + (int64_t)(row - sc.offset) * row_elems;
      const uint4* sk = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(sc.k) + src_off);
      const uint4* sv = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(sc.v) + src_off);
      const double* ct = ctab + s_delta * half;
      const double* st = stab + s_delta * half;
      for (int i0 = threadIdx.x; i0 < vpr; i0 += blockDim.x * ASM_UNROLL) {
        uint4 kv[ASM_UNROLL], vv[ASM_UNROLL];
#pragma unroll
        for (int u = 0; u < ASM_UNROLL; ++u) {
          const int i = i0 + u * blockDim.x;
          if (i < vpr) {
            kv[u] = __ldg(sk + i);
            if (has_v) vv[u] = __ldg(sv + i);
          }
        }
#pragma unroll
        for (int u = 0; u < ASM_UNROLL; ++u) {
          const int i = i0 + u * blockDim.x;
          if (i < vpr) {
            if (has_v) reinterpret_cast<uint4*>(dv)[i] = vv[u];
            const int j0 = ((i * V) % d) >> 1;
            if constexpr (kBf16) {
              const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&kv[u]);
              uint4 outr;
              __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(&outr);
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float2 f = __bfloat1622float2(p[t]);
                const float2 cs = s_cs[j0 + t];
                float oe, oo;
                rotate_pair_fast(f.x, f.y, cs.x, cs.y, oe, oo);
                q[t] = __floats2bfloat162_rn(oe, oo);
              }
              reinterpret_cast<uint4*>(dk)[i] = outr;
            } else {
              reinterpret_cast<uint4*>(dk)[i] = rotate_vec<T>(kv[u], j0, ct, st);
            }
          }
        }
      }
    }
  }
}

template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ sk, const T* __restrict__ sv, int64_t sstride,
                                   const int32_t* __restrict__ rows, int64_t n_rows,
                                   T* __restrict__ dk, T* __restrict__ dv, int64_t dstride,
                                   int64_t row_elems) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = Vec16<T>::N;
  const int layer = blockIdx.y;
  const int64_t vpr = row_elems / V;
  const int64_t total = n_rows * vpr;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / vpr, e = (idx - i * vpr) * V;
    const int64_t src = layer * sstride + (int64_t)rows[i] * row_elems + e;
    const int64_t dst = layer * dstride + i * row_elems + e;
    *reinterpret_cast<uint4*>(dk + dst) = __ldg(reinterpret_cast<const uint4*>(sk + src));
    *reinterpret_cast<uint4*>(dv + dst) = __ldg(reinterpret_cast<const uint4*>(sv + src));
  }
}

}  // namespace qcf

static int assemble_impl(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx, const void* bos_k,
                         const void* bos_v, void* fused_k, void* fused_v, int64_t fused_layer_stride, int layer0,
                         int n_layers, int hkv, int d, const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                         const int32_t* deltas, int max_delta, int dtype, qcf_stream_t stream,
                         const uint32_t* skip = nullptr) {
  QCF_REQUIRE(chunks && bos_k && fused_k && cos_tbl && sin_tbl && (!fused_v || bos_v), QCF_EINVAL,
              "qcf_assemble: null pointer");
  QCF_REQUIRE(n_chunks >= 1 && n_ctx >= 1 && n_layers >= 1 && hkv >= 1 && layer0 >= 0, QCF_EINVAL,
              "qcf_assemble: bad sizes");
  QCF_REQUIRE(d % 8 == 0, QCF_EUNSUPPORTED, "qcf_assemble: d_head must be a multiple of 8");
  QCF_REQUIRE(n_ctx < n_pos && max_delta < n_pos, QCF_ESHAPE, "qcf_assemble: RoPE table too short (%lld)",
              (long long)n_pos);
  const int row_elems = hkv * d;
  QCF_REQUIRE(fused_layer_stride >= (int64_t)(n_ctx + 1) * row_elems, QCF_ESHAPE,
              "qcf_assemble: fused layer stride too small");
  auto s = qcf::as_stream(stream);
  QCF_REQUIRE(row_elems % (dtype == QCF_F32 ? 4 : 8) == 0, QCF_EUNSUPPORTED, "qcf_assemble: row not 16B multiple");
  QCF_REQUIRE(d / 2 <= qcf::ASM_MAX_HALF, QCF_EUNSUPPORTED, "qcf_assemble: d_head > %d", 2 * qcf::ASM_MAX_HALF);
  dim3 grid((unsigned)std::min<int64_t>((n_ctx + 1 + qcf::ASM_ROWS - 1) / qcf::ASM_ROWS, 65535), n_layers);
  const dim3 block(qcf::ASM_THREADS);
  if (dtype == QCF_F32)
    QCF_LAUNCH("assemble_kernel", qcf::assemble_kernel<float>, dim3(grid), block, 0, s, chunks, n_chunks, n_ctx + 1, (const float*)bos_k,
        (const float*)bos_v, (float*)fused_k, (float*)fused_v, fused_layer_stride, row_elems, d, cos_tbl, sin_tbl,
        deltas, layer0, skip);
  else if (dtype == QCF_BF16)
    QCF_LAUNCH("assemble_kernel", qcf::assemble_kernel<__nv_bfloat16>, dim3(grid), block, 0, s, chunks, n_chunks, n_ctx + 1,
        (const __nv_bfloat16*)bos_k, (const __nv_bfloat16*)bos_v, (__nv_bfloat16*)fused_k,
        (__nv_bfloat16*)fused_v, fused_layer_stride, row_elems, d, cos_tbl, sin_tbl, deltas, layer0, skip);
  else
    QCF_REQUIRE(false, QCF_EINVAL, "qcf_assemble: bad dtype");
  QCF_LAUNCH_CHECK("qcf_assemble");
  return QCF_OK;
}

extern "C" int qcf_assemble_rot(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                                const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                                int64_t fused_layer_stride, int n_layers, int hkv, int d,
                                const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                                const int32_t* deltas, int max_delta, int dtype, qcf_stream_t stream) {
  return assemble_impl(chunks, n_chunks, n_ctx, bos_k, bos_v, fused_k, fused_v, fused_layer_stride, 0, n_layers,
                       hkv, d, cos_tbl, sin_tbl, n_pos, deltas, max_delta, dtype, stream);
}

extern "C" int qcf_assemble_range(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                                  const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                                  int64_t fused_layer_stride, int layer0, int n_layers, int hkv, int d,
                                  const double* cos_tbl, const double* sin_tbl, int64_t n_pos, int dtype,
                                  qcf_stream_t stream) {
  return assemble_impl(chunks, n_chunks, n_ctx, bos_k, bos_v, fused_k, fused_v, fused_layer_stride, layer0,
                       n_layers, hkv, d, cos_tbl, sin_tbl, n_pos, nullptr, 0, dtype, stream);
}

extern "C" int qcf_assemble_range_skip(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                                       const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                                       int64_t fused_layer_stride, int layer0, int n_layers, int hkv, int d,
                                       const double* cos_tbl, const double* sin_tbl, int64_t n_pos, int dtype,
                                       const uint32_t* skip_rows, qcf_stream_t stream) {
  return assemble_impl(chunks, n_chunks, n_ctx, bos_k, bos_v, fused_k, fused_v, fused_layer_stride, layer0,
                       n_layers, hkv, d, cos_tbl, sin_tbl, n_pos, nullptr, 0, dtype, stream, skip_rows);
}

namespace qcf {
// bitmap of the fused rows named in pos[r * stride + i] (i < n_per_req), one block
// per request: cleared, then one atomicOr per row; rows <= 0 (BOS / padding) ignored
__global__ void rows_bitmap_kernel(const int32_t* __restrict__ pos, int64_t stride, int64_t n_per_req,
                                   uint32_t* __restrict__ bm, int64_t words) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  uint32_t* b = bm + (int64_t)r * words;
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) b[i] = 0u;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n_per_req; i += blockDim.x) {
    const int32_t p = pos[(int64_t)r * stride + i];
    if (p > 0 && (p >> 5) < words) atomicOr(b + (p >> 5), 1u << (p & 31));
  }
}
}  // namespace qcf

extern "C" int qcf_rows_bitmap(const int32_t* pos, int64_t stride, int n_req, int64_t n_per_req, uint32_t* bitmap,
                               int64_t words_per_req, qcf_stream_t stream) {
  QCF_REQUIRE(pos && bitmap && n_req >= 1 && n_req <= 65535 && n_per_req >= 0 && words_per_req >= 1, QCF_EINVAL,
              "qcf_rows_bitmap: bad arguments");
  QCF_LAUNCH("rows_bitmap_kernel", qcf::rows_bitmap_kernel, dim3((unsigned)n_req), dim3(256), 0, qcf::as_stream(stream),
             pos, stride, n_per_req, bitmap, words_per_req);
  QCF_LAUNCH_CHECK("qcf_rows_bitmap");
  return QCF_OK;
}

extern "C" int qcf_assemble(const qcf_chunk_desc* chunks, int n_chunks, int n_ctx,
                            const void* bos_k, const void* bos_v, void* fused_k, void* fused_v,
                            int64_t fused_layer_stride, int n_layers, int hkv, int d,
                            const double* cos_tbl, const double* sin_tbl, int64_t n_pos,
                            int dtype, qcf_stream_t stream) {
  return qcf_assemble_rot(chunks, n_chunks, n_ctx, bos_k, bos_v, fused_k, fused_v, fused_layer_stride, n_layers,
                          hkv, d, cos_tbl, sin_tbl, n_pos, nullptr, 0, dtype, stream);
}

extern "C" int qcf_gather_rows(const void* src_k, const void* src_v, int64_t src_layer_stride,
                               const int32_t* rows, int64_t n_rows, void* dst_k, void* dst_v,
                               int64_t dst_layer_stride, int n_layers, int64_t row_elems,
                               int dtype, qcf_stream_t stream) {
  QCF_REQUIRE(src_k && src_v && rows && dst_k && dst_v, QCF_EINVAL, "qcf_gather_rows: null pointer");
  QCF_REQUIRE(row_elems % 8 == 0, QCF_EUNSUPPORTED, "qcf_gather_rows: row must be 16B multiple");
  if (n_rows == 0 || n_layers == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  const int vec = dtype == QCF_F32 ? 4 : 8;
  int gx = (int)std::min<int64_t>((n_rows * (row_elems / vec) + 255) / 256, 65535);
  dim3 grid(gx, n_layers);
  if (dtype == QCF_F32)
    QCF_LAUNCH("gather_rows_kernel", qcf::gather_rows_kernel<float>, dim3(grid), dim3(256), 0, s, (const float*)src_k, (const float*)src_v,
        src_layer_stride, rows, n_rows, (float*)dst_k, (float*)dst_v, dst_layer_stride, row_elems);
  else
    QCF_LAUNCH("gather_rows_kernel", qcf::gather_rows_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, (const __nv_bfloat16*)src_k,
        (const __nv_bfloat16*)src_v, src_layer_stride, rows, n_rows, (__nv_bfloat16*)dst_k,
        (__nv_bfloat16*)dst_v, dst_layer_stride, row_elems);
  QCF_LAUNCH_CHECK("qcf_gather_rows");
  return QCF_OK;
}
