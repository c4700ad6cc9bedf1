// Attention launch declarations.
#pragma once
#include "common.cuh"

namespace qcf {
int attention_simt_launch(int dtype, const void* q, const void* k, const void* v,
                          const int32_t* kmax, int64_t m, int h, int hkv, int d, int64_t n_keys,
                          void* out, cudaStream_t s, int n_req = 1, const uint32_t* mask = nullptr,
                          int64_t mask_words = 0);
// tensor-core path (bf16); returns QCF_EUNSUPPORTED for shapes it does not cover
int attention_tc_launch(const void* q, const void* k, const void* v, const int32_t* kmax,
                        int64_t m, int h, int hkv, int d, int64_t n_keys, void* out,
                        cudaStream_t s, int n_req = 1, void* ws = nullptr, size_t ws_bytes = 0);
size_t attention_workspace(int64_t m, int n_req, int h, int n_split);
int attention_auto_split(int64_t m, int n_req, int h, int64_t n_keys);
void set_attention_split(int n);
}  // namespace qcf
