// k_passB_g1.cu — instantiations of the wide W pass, smooth_l <= 8, R <= 32 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g1(Handle& h, int nt) { passB_wide_group<1, 1, 4>(h, nt); }
}  // namespace copa
