// k_passB_g3.cu — instantiations of the wide W pass, 8 < smooth_l <= 16, R <= 32 (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g3(Handle& h, int nt) { passB_wide_group<2, 1, 4>(h, nt); }
}  // namespace copa
