// scan_m.cu — the M super-tile shape of the scans (see scan_impl.cuh).
#include "scan_impl.cuh"

namespace ga {
namespace scan_impl {
GA_SCAN_INSTANTIATE(SHAPE_M)
}  // namespace scan_impl
}  // namespace ga
