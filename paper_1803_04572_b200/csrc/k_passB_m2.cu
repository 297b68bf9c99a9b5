// k_passB_m2.cu — instantiations of the wide W pass for 8 < smooth_l <= 16 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_M2(Handle& h) { passB_wide_n<2>(h); }
}  // namespace copa
