// Kernel instantiations for 8 lane(s) per stream.
#include "alert_kernels.cuh"

namespace alert {
ALERT_INSTANTIATE(8)
}  // namespace alert
