// Dispatch of the public GEMM / attention entry points onto the sm_100a
// tensor-core kernels (bf16) or the FFMA parity kernels (f32).
#include "attention.cuh"
#include "common.cuh"
#include "gemm.cuh"

#include <atomic>
#include <cstdlib>

namespace qcf {

// bf16 calls that left the tcgen05 kernels for the SIMT (FFMA) ones because
// the shape is outside the tensor-core contract (head dim != 128, K % 8, toy
// widths). Counted so a speed-mode run can prove it never fell back; with
// strict mode on (qcf_set_strict_tc(1) or QCF_STRICT_TC=1) such a call fails
// with QCF_EUNSUPPORTED instead.
static std::atomic<long long> g_simt_fallbacks{0};
static std::atomic<int> g_strict_tc{-1};

static bool strict_tc() {
  int v = g_strict_tc.load();
  if (v < 0) {
    const char* e = std::getenv("QCF_STRICT_TC");
    v = (e && e[0] == '1') ? 1 : 0;
    g_strict_tc.store(v);
  }
  return v == 1;
}

// returns QCF_OK when the SIMT path may run, QCF_EUNSUPPORTED in strict mode
static int note_bf16_fallback(const char* what) {
  g_simt_fallbacks.fetch_add(1);
  if (strict_tc()) {
    set_error("%s: bf16 shape outside the tcgen05 contract and strict tensor-core mode is on", what);
    return QCF_EUNSUPPORTED;
  }
  return QCF_OK;
}

static int g_tc_state = -1;  // -1 unknown, 0 no, 1 yes

static bool tc_ok() {
  if (g_tc_state < 0) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    g_tc_state = (major == 10 && minor == 0) ? 1 : 0;
  }
  return g_tc_state == 1;
}

bool tc_available() { return tc_ok(); }
void set_attention_kernel(int v);
void set_gemm_plan(int p);

}  // namespace qcf

extern "C" int qcf_tc_available(void) { return qcf::tc_ok() ? 1 : 0; }

extern "C" long long qcf_simt_fallbacks(void) { return qcf::g_simt_fallbacks.load(); }

extern "C" int qcf_set_strict_tc(int on) {
  QCF_REQUIRE(on == 0 || on == 1, QCF_EINVAL, "qcf_set_strict_tc: 0 or 1");
  qcf::g_strict_tc.store(on);
  return QCF_OK;
}

extern "C" int qcf_gemm(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb, void* c,
                        int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue, int out_dtype,
                        qcf_stream_t stream) {
  int st = qcf::gemm_check_args(dtype, a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype);
  if (st != QCF_OK) return st;
  if (m == 0 || n == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  if (dtype == QCF_BF16) {
    QCF_REQUIRE(qcf::tc_ok(), QCF_EUNSUPPORTED, "qcf_gemm: bf16 path needs an sm_100 (B200) device");
    st = qcf::gemm_tc_launch(a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s);
    if (st != QCF_EUNSUPPORTED) return st;
    // shapes outside the tcgen05 kernel's alignment contract (K % 8 != 0, tiny
    // toy widths) run on the SIMT kernel; still on the GPU, never on the host
    st = qcf::note_bf16_fallback("qcf_gemm");
    if (st != QCF_OK) return st;
  }
  return qcf::gemm_simt_launch(dtype, a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s);
}

extern "C" int qcf_attention_split(int64_t m, int n_req, int h, int64_t n_keys) {
  return qcf::attention_auto_split(m, n_req, h, n_keys);
}

extern "C" size_t qcf_attention_workspace(int64_t m, int n_req, int h, int64_t n_keys) {
  return qcf::attention_workspace(m, n_req, h, qcf::attention_auto_split(m, n_req, h, n_keys));
}

extern "C" int qcf_attention_batched_ws(int dtype, const void* q, const void* k, const void* v,
                                        const int32_t* kmax, int64_t m, int n_req, int h, int hkv, int d,
                                        int64_t n_keys, void* out, void* ws, size_t ws_bytes,
                                        qcf_stream_t stream) {
  QCF_REQUIRE(q && k && v && kmax && out, QCF_EINVAL, "qcf_attention: null pointer");
  QCF_REQUIRE(h > 0 && hkv > 0 && h % hkv == 0 && n_keys > 0 && n_req >= 1, QCF_EINVAL,
              "qcf_attention: bad shape");
  QCF_REQUIRE(dtype == QCF_F32 || dtype == QCF_BF16, QCF_EINVAL, "qcf_attention: bad dtype");
  QCF_REQUIRE(n_req <= 65535, QCF_EUNSUPPORTED, "qcf_attention: too many requests");
  if (m == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  if (dtype == QCF_BF16 && qcf::tc_ok()) {
    int st = qcf::attention_tc_launch(q, k, v, kmax, m, h, hkv, d, n_keys, out, s, n_req, ws, ws_bytes);
    if (st != QCF_EUNSUPPORTED) return st;
    st = qcf::note_bf16_fallback("qcf_attention");
    if (st != QCF_OK) return st;
  }
  return qcf::attention_simt_launch(dtype, q, k, v, kmax, m, h, hkv, d, n_keys, out, s, n_req);
}

extern "C" int qcf_attention_batched(int dtype, const void* q, const void* k, const void* v,
                                     const int32_t* kmax, int64_t m, int n_req, int h, int hkv, int d,
                                     int64_t n_keys, void* out, qcf_stream_t stream) {
  return qcf_attention_batched_ws(dtype, q, k, v, kmax, m, n_req, h, hkv, d, n_keys, out, nullptr, 0, stream);
}

extern "C" int qcf_attention(int dtype, const void* q, const void* k, const void* v,
                             const int32_t* kmax, int64_t m, int h, int hkv, int d, int64_t n_keys,
                             void* out, qcf_stream_t stream) {
  return qcf_attention_batched(dtype, q, k, v, kmax, m, 1, h, hkv, d, n_keys, out, stream);
}

extern "C" size_t qcf_gemm_workspace(int64_t m, int64_t n, int64_t k) { return qcf::gemm_workspace_bytes(m, n, k); }

extern "C" int qcf_gemm_ws(int dtype, const void* a, int64_t lda, const void* b, int64_t ldb, void* c,
                           int64_t ldc, int64_t m, int64_t n, int64_t k, int epilogue, int out_dtype, int b_layout,
                           void* ws, size_t ws_bytes, qcf_stream_t stream) {
  int st = qcf::gemm_check_args(dtype, a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype);
  if (st != QCF_OK) return st;
  QCF_REQUIRE(b_layout == QCF_B_ROWMAJOR || b_layout == QCF_B_TILE64, QCF_EINVAL, "qcf_gemm_ws: bad b_layout");
  if (m == 0 || n == 0) return QCF_OK;
  auto s = qcf::as_stream(stream);
  if (dtype == QCF_BF16 && qcf::tc_ok() && m <= 256) {
    st = qcf::gemm_tc_skinny(a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, b_layout, ws, ws_bytes, s);
    if (st != QCF_EUNSUPPORTED) return st;
  }
  if (b_layout == QCF_B_TILE64) {
    QCF_REQUIRE(dtype == QCF_BF16 && qcf::tc_ok(), QCF_EUNSUPPORTED, "qcf_gemm_ws: tile-major B needs tcgen05");
    st = qcf::gemm_tc_launch(a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s, 1, ws, ws_bytes);
    if (st == QCF_EUNSUPPORTED) qcf::set_error("qcf_gemm_ws: shape not covered for tile-major B");
    return st;
  }
  if (dtype == QCF_BF16 && qcf::tc_ok()) {
    st = qcf::gemm_tc_launch(a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, s, 0, ws, ws_bytes);
    if (st != QCF_EUNSUPPORTED) return st;
  }
  return qcf_gemm(dtype, a, lda, b, ldb, c, ldc, m, n, k, epilogue, out_dtype, stream);
}

extern "C" int qcf_gemm_qkv_rope(const void* a, int64_t lda, const void* w, int64_t ldb, int b_layout, int64_t m,
                                 int64_t k, int h, int hkv, int d, const int32_t* pos, const int32_t* dst_rows,
                                 const float* cs_tbl, int64_t n_pos, void* q_out,
                                 void* k_tab, void* v_tab, void* ws, size_t ws_bytes, qcf_stream_t stream) {
  (void)n_pos;
  QCF_REQUIRE(a && w && pos && dst_rows && cs_tbl && q_out && k_tab && v_tab, QCF_EINVAL,
              "qcf_gemm_qkv_rope: null pointer");
  QCF_REQUIRE(h > 0 && hkv > 0 && h % hkv == 0 && d > 0 && d % 2 == 0 && k > 0 && m >= 0, QCF_EINVAL,
              "qcf_gemm_qkv_rope: bad shape");
  if (m == 0) return QCF_OK;
  QCF_REQUIRE(qcf::tc_ok(), QCF_EUNSUPPORTED, "qcf_gemm_qkv_rope: needs an sm_100 device");
  const int st = qcf::gemm_qkv_rope_launch(a, lda, w, ldb, m, k, h, hkv, d, pos, dst_rows, cs_tbl,
                                           q_out, k_tab, v_tab, qcf::as_stream(stream), b_layout, ws, ws_bytes);
  if (st == QCF_EUNSUPPORTED) qcf::set_error("qcf_gemm_qkv_rope: shape not covered (d %% 32, alignment)");
  return st;
}

extern "C" int qcf_set_attention_kernel(int version) {
  QCF_REQUIRE(version >= 0 && version <= 8 && version != 5 && version != 6 && version != 7, QCF_EINVAL,
              "qcf_set_attention_kernel: version 0 (auto), 1, 2, 3, 4 or 8");
  qcf::set_attention_kernel(version);
  return QCF_OK;
}

extern "C" int qcf_set_gemm_plan(int plan) {
  QCF_REQUIRE(plan >= 0 && plan < 16, QCF_EINVAL, "qcf_set_gemm_plan: 0 (auto) .. 7, +8 = stream-K on");
  qcf::set_gemm_plan(plan);
  return QCF_OK;
}

extern "C" int qcf_set_attention_split(int n_split) {
  QCF_REQUIRE(n_split >= 0 && n_split <= 16, QCF_EINVAL, "qcf_set_attention_split: 0 (off) .. 16");
  qcf::set_attention_split(n_split);
  return QCF_OK;
}
