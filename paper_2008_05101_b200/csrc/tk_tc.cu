// tk_tc.cu -- tcgen05 kind::i8 tensor-core GEMM (placeholder until the
// kernel lands; the dispatcher only selects it when supported).
#include "tk_internal.cuh"

bool tk_tc_supported(int, int, int) { return false; }

cudaError_t tk_launch_gemm_tc(const int8_t*, int, int, const tk_layer*,
                              tk_epilogue, cudaStream_t) {
  return cudaErrorNotSupported;
}
