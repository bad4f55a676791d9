// krp_sketch_tc.cu — tcgen05 3xTF32 fused sketch (placeholder until the kernel lands).
#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {
bool tc_sketch_supported(const Dims&, int, const bool*) { return false; }
size_t tc_sketch_ws_bytes(const Dims&, int, const bool*) { return 0; }
int tc_sketch(const float*, const Dims&, const OmegaPtrs&, int, const bool*, float* const*, Arena&, cudaStream_t) {
  set_error("tcgen05 sketch not available");
  return KRP_EUNSUPPORTED;
}
}  // namespace krp
