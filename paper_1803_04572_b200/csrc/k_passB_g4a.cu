// k_passB_g4a.cu — instantiation of the wide W pass, 8 < smooth_l <= 16, NT = 5 (R in (32, 40]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g4a(Handle& h) { passB_wide_inst<2, 5>(h); }
}  // namespace copa
