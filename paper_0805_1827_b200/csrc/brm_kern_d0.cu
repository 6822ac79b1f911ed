// Instantiation of the dimension-templated kernels for d = any (runtime d).
#include "brm_kernels.cuh"

namespace brm {
KernelTriple kernels_d0(bool fast) {
  if (fast) return KernelTriple{(void *)&walk_units<0, true>, (void *)&iz_probes<0, true>, (void *)&decisions<0, true>};
  return KernelTriple{(void *)&walk_units<0, false>, (void *)&iz_probes<0, false>, (void *)&decisions<0, false>};
}
}  // namespace brm
