// k_passB_s.cu — instantiations of the configured (R, l) shapes of the wide W pass (see k_dense.cuh).
#include "k_dense.cuh"

namespace copa {
bool passB_wide_special(Handle& h) {
  if (h.l == 7 && h.R == 20) { passB_wide_inst<1, 3, 20, 7>(h); return true; }
  if (h.l == 7 && h.R == 15) { passB_wide_inst<1, 2, 15, 7>(h); return true; }
  if (h.l == 9 && h.R == 40) { passB_wide_inst<2, 5, 40, 9>(h); return true; }
  return false;
}
}  // namespace copa
