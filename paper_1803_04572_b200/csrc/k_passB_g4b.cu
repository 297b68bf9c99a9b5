// k_passB_g4b.cu — instantiation of the wide W pass, 8 < smooth_l <= 16, NT = 6 (R in (40, 48]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g4b(Handle& h) { passB_wide_inst<2, 6>(h); }
}  // namespace copa
