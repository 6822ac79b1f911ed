// Instantiation of the dimension-templated kernels for d = 1.
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d1(bool fast) {
  if (fast) return KernelTriple{(void *)&walk_units<1, true>, (void *)&iz_probes<1, true>, (void *)&decisions<1, true>};
  return KernelTriple{(void *)&walk_units<1, false>, (void *)&iz_probes<1, false>, (void *)&decisions<1, false>};
}
}  // namespace brm
