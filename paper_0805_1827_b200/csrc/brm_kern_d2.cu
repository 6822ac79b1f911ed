// Instantiation of the dimension-templated kernels for d = 2.
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d2(bool fast) {
  if (fast)
    return KernelTriple{(void *)&walk_units<2, true>, (void *)&iz_probes<2, true>, (void *)&decisions<2, true>,
                        nullptr, (void *)&walk_units<2, true, WALK_CMC>,
                        (void *)&walk_units<2, true, WALK_CMC_UNIT>};
  return KernelTriple{(void *)&walk_units<2, false>, (void *)&iz_probes<2, false>, (void *)&decisions<2, false>,
                      (void *)&iz_probes<2, false, 1>, (void *)&walk_units<2, false, WALK_CMC>,
                      (void *)&walk_units<2, false, WALK_CMC_UNIT>, nullptr,
                      (void *)&walk_units<2, false, WALK_CMC_LOG>, (void *)&iz_probes<2, false, 2>,
                      (void *)&iz_probes<2, false, 3>};
}
}  // namespace brm
