// Instantiation of the dimension-templated kernels for d = 40.
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d40(bool fast) {
  if (fast) {
    KernelTriple k{(void *)&walk_units<40, true>, (void *)&iz_probes<40, true>, (void *)&decisions<40, true>,
                   nullptr, (void *)&walk_units<40, true, WALK_CMC>, nullptr,
                   (void *)&walk_units<40, true, WALK_CMC_LOWER>};
    k.walk_cmc_colconst = (void *)&walk_units<40, true, WALK_CMC_COLCONST>;
    return k;
  }
  return KernelTriple{(void *)&walk_units<40, false>, (void *)&iz_probes<40, false>, (void *)&decisions<40, false>,
                      nullptr, (void *)&walk_units<40, false, WALK_CMC>};
}
}  // namespace brm
