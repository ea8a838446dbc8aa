// Generic operator kernels instantiated for dim = 2, space degree k = 2.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d2_k2() { return DegreeOps<2, 2>::table(); }
}  // namespace dgb
