// Placeholder translation unit for the legacy b1 mma.sync AND-popc conv variant.
#include "xnc_common.cuh"

namespace xnc {
int launch_conv_b1mma(const uint32_t*, const uint32_t*, const float*, const float*, int, int, int,
                      int, int, int, int, int, float*, int32_t*, cudaStream_t) {
  return XNC_ENOTSUP;
}
}  // namespace xnc
