// Generic operator kernels instantiated for dim = 2, space degree k = 1.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d2_k1() { return DegreeOps<2, 1>::table(); }
}  // namespace dgb
