// k_polar_l4.cu — instantiations of the wide polar kernel for smooth_l <= 4 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void polar_wide_L4(Handle& h) { polar_wide_n<4>(h); }
}  // namespace copa
