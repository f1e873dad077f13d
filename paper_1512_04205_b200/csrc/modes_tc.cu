// modes_tc.cu — tcgen05 (kind::i8) mode projection.  PLACEHOLDER until the
// tensor-core kernel lands: routes to the dp4a kernel (bit-identical numerics).
#include "common.cuh"

namespace cdmd {

cudaError_t launch_modes_tc(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi,
                            cudaStream_t st) {
  return launch_modes_simt(v, M, Phi, ldphi, st);
}

}  // namespace cdmd
