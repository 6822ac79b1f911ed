// Instantiation of the dimension-templated kernels for d = 10.
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d10(bool fast) {
  if (fast)
    return KernelTriple{(void *)&walk_units<10, true>, (void *)&iz_probes<10, true>, (void *)&decisions<10, true>,
                        nullptr, (void *)&walk_units<10, true, WALK_CMC>,
                        (void *)&walk_units<10, true, WALK_CMC_UNIT>};
  return KernelTriple{(void *)&walk_units<10, false>, (void *)&iz_probes<10, false>, (void *)&decisions<10, false>,
                      (void *)&iz_probes<10, false, 1>, (void *)&walk_units<10, false, WALK_CMC>,
                      (void *)&walk_units<10, false, WALK_CMC_UNIT>, nullptr,
                      (void *)&walk_units<10, false, WALK_CMC_LOG>, (void *)&iz_probes<10, false, 2>,
                      (void *)&iz_probes<10, false, 3>};
}
}  // namespace brm
