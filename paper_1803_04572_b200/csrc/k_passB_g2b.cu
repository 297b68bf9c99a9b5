// k_passB_g2b.cu — instantiation of the wide W pass, smooth_l <= 8, NT = 6 (R in (40, 48]; see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
void passB_wide_g2b(Handle& h) { passB_wide_inst<1, 6>(h); }
}  // namespace copa
