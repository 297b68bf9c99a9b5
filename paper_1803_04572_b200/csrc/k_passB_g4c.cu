// k_passB_g4c.cu — instantiation of the wide W pass, 8 < smooth_l <= 16, NT = 7 (R in (48, 56]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g4c(Handle& h) { passB_wide_inst<2, 7>(h); }
}  // namespace copa
