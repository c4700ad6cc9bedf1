// Library-level entry points: version, error reporting, small device helpers.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace qcf {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QCF_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return QCF_ECUDA;
}

__global__ void iota_add_kernel(const int32_t* a, int64_t n, int32_t add, int32_t* out) {
  pdl_wait();
  pdl_trigger();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (a ? a[i] : 0) + add + (a ? 0 : (int32_t)i);
}

}  // namespace qcf

extern "C" {

const char* qcf_version(void) { return "qcfuse_b200 0.1 (sm_100a)"; }

const char* qcf_last_error(void) { return qcf::g_err; }

int qcf_iota_add(const int32_t* a, int64_t n, int32_t add, int32_t* out, qcf_stream_t stream) {
  QCF_REQUIRE(a && out && n >= 0, QCF_EINVAL, "qcf_iota_add: bad args");
  if (n == 0) return QCF_OK;
  QCF_LAUNCH("iota_add_kernel", qcf::iota_add_kernel, dim3(qcf::ceil_div(n, 256)), dim3(256), 0, qcf::as_stream(stream), a, n, add, out);
  QCF_LAUNCH_CHECK("qcf_iota_add");
  return QCF_OK;
}

int qcf_iota(int64_t n, int32_t start, int32_t* out, qcf_stream_t stream) {
  QCF_REQUIRE(out && n >= 0, QCF_EINVAL, "qcf_iota: bad args");
  if (n == 0) return QCF_OK;
  QCF_LAUNCH("iota_add_kernel", qcf::iota_add_kernel, dim3(qcf::ceil_div(n, 256)), dim3(256), 0, qcf::as_stream(stream), nullptr, n, start, out);
  QCF_LAUNCH_CHECK("qcf_iota");
  return QCF_OK;
}

}  // extern "C"
