// k_polar_l12.cu — instantiations of the wide polar kernel for smooth_l <= 12 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void polar_wide_L12(Handle& h) { polar_wide_n<12>(h); }
}  // namespace copa
