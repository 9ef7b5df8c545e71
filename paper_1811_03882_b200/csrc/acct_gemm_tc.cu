// gemm_nn on the 5th-generation tensor cores: placeholder until the tcgen05
// 3xTF32 kernel lands; AUTO mode falls back to the SIMT kernels.
#include "acct_common.cuh"

namespace acct {

int gemm_tc(int, int, int, float, const float *, int64_t, const float *, int64_t, float, float *,
            int64_t, const float *, int, cudaStream_t) {
  return ACCT_ENOTSUP;
}

}  // namespace acct
