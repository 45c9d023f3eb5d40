// tcgen05 / TMEM 3xTF32 GEMM for sm_100a -- placeholder until the kernel lands.
#include "common.cuh"
#include "gemm.h"

namespace skp {
bool tc_available() { return false; }
int gemm_tc_3xtf32(int, int, int64_t, int64_t, int64_t, float, const float*, int64_t,
                   const float*, int64_t, float, float*, int64_t, void*, int64_t, cudaStream_t) {
    return SKP_ERR_UNSUPPORTED;
}
int64_t gemm_tc_ws_bytes(int, int, int64_t, int64_t, int64_t) { return 0; }
}  // namespace skp
