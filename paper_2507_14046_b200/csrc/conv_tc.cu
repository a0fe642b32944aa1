// tcgen05 implicit-GEMM convolutions (placeholder until the kernel lands).
#include "common.cuh"
#include "kernels.h"

namespace d2ip {

bool conv_tc_supported(int, int, int, int, int) { return false; }

int conv_fwd_tc(d2ip_act, const float*, const float*, long long, int, int, d2ip_act, int, int, int,
                cudaStream_t) {
  set_error("tcgen05 conv not built");
  return D2IP_E_UNSUPPORTED;
}

}  // namespace d2ip
