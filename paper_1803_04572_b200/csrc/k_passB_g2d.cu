// k_passB_g2d.cu — instantiation of the wide W pass, smooth_l <= 8, NT = 8 (R in (56, 64]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g2d(Handle& h) { passB_wide_inst<1, 8>(h); }
}  // namespace copa
