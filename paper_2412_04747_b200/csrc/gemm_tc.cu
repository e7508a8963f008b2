// tcgen05 typed segment GEMM (placeholder until the sm_100a kernel lands).
#include "ops.cuh"

namespace rgnn {
bool gemm_tc_supported(const GemmArgs&) { return false; }
void gemm_tc(const GemmArgs&, cudaStream_t) { RGNN_FAIL(RGNN_ERR_UNSUPPORTED, "tcgen05 GEMM not built"); }
}  // namespace rgnn
