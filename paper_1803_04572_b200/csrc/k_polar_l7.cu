// k_polar_l7.cu — instantiations of the wide polar kernel for smooth_l <= 7 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void polar_wide_L7(Handle& h) { polar_wide_n<7>(h); }
}  // namespace copa
