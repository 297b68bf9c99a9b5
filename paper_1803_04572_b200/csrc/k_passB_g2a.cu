// k_passB_g2a.cu — instantiation of the wide W pass, smooth_l <= 8, NT = 5 (R in (32, 40]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g2a(Handle& h) { passB_wide_inst<1, 5>(h); }
}  // namespace copa
