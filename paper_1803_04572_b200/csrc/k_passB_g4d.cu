// k_passB_g4d.cu — instantiation of the wide W pass, 8 < smooth_l <= 16, NT = 8 (R in (56, 64]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g4d(Handle& h) { passB_wide_inst<2, 8>(h); }
}  // namespace copa
