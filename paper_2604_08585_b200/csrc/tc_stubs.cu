// Placeholder for the tensor-core attention entry point (see attention_tc.cu when built).
#include "attention.cuh"
namespace qcf {
int attention_tc_launch(const void*, const void*, const void*, const int32_t*, int64_t, int, int,
                        int, int64_t, void*, cudaStream_t) { return QCF_EUNSUPPORTED; }
}
