// k_passB_m1.cu — instantiations of the wide W pass for smooth_l <= 8 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_M1(Handle& h) { passB_wide_n<1>(h); }
}  // namespace copa
