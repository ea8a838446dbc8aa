// Generic operator kernels instantiated for dim = 3, space degree k = 1.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d3_k1() { return DegreeOps<3, 1>::table(); }
}  // namespace dgb
