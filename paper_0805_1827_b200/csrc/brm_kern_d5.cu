// Instantiation of the dimension-templated kernels for d = 5.
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d5(bool fast) {
  if (fast)
    return KernelTriple{(void *)&walk_units<5, true>, (void *)&iz_probes<5, true>, (void *)&decisions<5, true>,
                        nullptr, (void *)&walk_units<5, true, WALK_CMC>,
                        (void *)&walk_units<5, true, WALK_CMC_UNIT>};
  return KernelTriple{(void *)&walk_units<5, false>, (void *)&iz_probes<5, false>, (void *)&decisions<5, false>,
                      (void *)&iz_probes<5, false, 1>, (void *)&walk_units<5, false, WALK_CMC>,
                      (void *)&walk_units<5, false, WALK_CMC_UNIT>, nullptr,
                      (void *)&walk_units<5, false, WALK_CMC_LOG>, (void *)&iz_probes<5, false, 2>,
                      (void *)&iz_probes<5, false, 3>};
}
}  // namespace brm
