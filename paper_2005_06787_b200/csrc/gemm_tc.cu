// tcgen05 split-TF32 complex GEMM (placeholder until the sm_100a kernel lands).
#include "kernels.h"

namespace stn {

bool gemm_tc_supported(const GemmShape &) { return false; }
size_t gemm_tc_workspace_bytes(const GemmShape &) { return 0; }
cudaError_t launch_gemm_tc(const GemmShape &, const BatchPtrs &, void *, size_t, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace stn
