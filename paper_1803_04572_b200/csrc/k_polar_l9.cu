// k_polar_l9.cu — instantiations of the wide polar kernel for smooth_l <= 9 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void polar_wide_L9(Handle& h) { polar_wide_n<9>(h); }
}  // namespace copa
