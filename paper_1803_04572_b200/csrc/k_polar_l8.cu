// k_polar_l8.cu — instantiations of the wide polar kernel for smooth_l <= 8 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void polar_wide_L8(Handle& h) { polar_wide_n<8>(h); }
}  // namespace copa
