// tcgen05 tensor-core path (placeholder until the sm_100a kernels land).
#include "mbx_internal.h"

namespace mbx {
bool tc_supported(const Geometry&, int, int) { return false; }
size_t tc_workspace_bytes(const Geometry&) { return 0; }
cudaError_t tc_forward(const Geometry&, const void*, const void*, const void*, void*, void*,
                       cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace mbx
