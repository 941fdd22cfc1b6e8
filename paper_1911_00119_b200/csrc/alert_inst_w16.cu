// Kernel instantiations for 16 lane(s) per stream.
#include "alert_kernels.cuh"

namespace alert {
ALERT_INSTANTIATE(16)
}  // namespace alert
