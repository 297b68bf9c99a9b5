// k_passB_g2c.cu — instantiation of the wide W pass, smooth_l <= 8, NT = 7 (R in (48, 56]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g2c(Handle& h) { passB_wide_inst<1, 7>(h); }
}  // namespace copa
