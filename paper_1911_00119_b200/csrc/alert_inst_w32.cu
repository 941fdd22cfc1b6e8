// Kernel instantiations for 32 lane(s) per stream.
#include "alert_kernels.cuh"

namespace alert {
ALERT_INSTANTIATE(32)
}  // namespace alert
