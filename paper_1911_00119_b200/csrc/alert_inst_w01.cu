// Kernel instantiations for 1 lane(s) per stream.
#include "alert_kernels.cuh"

namespace alert {
ALERT_INSTANTIATE(1)
}  // namespace alert
