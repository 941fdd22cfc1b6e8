// Kernel instantiations for 4 lane(s) per stream.
#include "alert_kernels.cuh"

namespace alert {
ALERT_INSTANTIATE(4)
}  // namespace alert
