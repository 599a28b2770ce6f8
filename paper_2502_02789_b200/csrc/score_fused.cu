// Fused tcgen05 score kernel (placeholder until the kernel lands).
#include "sp_internal.h"

namespace sp {
bool fused_supported(const Geom&, const Layout&, const void*, const void*) { return false; }
size_t fused_score_ws_bytes(const Geom&) { return 0; }
cudaError_t fused_score(const __nv_bfloat16*, const __nv_bfloat16*, const Geom&, const Layout&, float*, void*, size_t,
                        cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace sp
