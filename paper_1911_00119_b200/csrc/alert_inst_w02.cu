// Kernel instantiations for 2 lane(s) per stream.
#include "alert_kernels.cuh"

namespace alert {
ALERT_INSTANTIATE(2)
}  // namespace alert
