// Instantiation of the dimension-templated kernels for d = 3.
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d3(bool fast) {
  if (fast)
    return KernelTriple{(void *)&walk_units<3, true>, (void *)&iz_probes<3, true>, (void *)&decisions<3, true>,
                        nullptr, (void *)&walk_units<3, true, WALK_CMC>,
                        (void *)&walk_units<3, true, WALK_CMC_UNIT>};
  return KernelTriple{(void *)&walk_units<3, false>, (void *)&iz_probes<3, false>, (void *)&decisions<3, false>,
                      (void *)&iz_probes<3, false, 1>, (void *)&walk_units<3, false, WALK_CMC>,
                      (void *)&walk_units<3, false, WALK_CMC_UNIT>, nullptr,
                      (void *)&walk_units<3, false, WALK_CMC_LOG>, (void *)&iz_probes<3, false, 2>,
                      (void *)&iz_probes<3, false, 3>};
}
}  // namespace brm
