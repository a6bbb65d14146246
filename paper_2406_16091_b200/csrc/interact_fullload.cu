// a6.2: full load (All-in-SM, Alg. 4, §5.1) -- placeholder until the
// sub-box kernel lands; reports "not applicable".
#include "interact_common.cuh"

namespace pi {
cudaError_t launch_interact_fullload(const Geom &, const KParams &, const InteractArgs &, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace pi
