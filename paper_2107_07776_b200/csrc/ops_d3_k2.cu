// Generic operator kernels instantiated for dim = 3, space degree k = 2.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d3_k2() { return DegreeOps<3, 2>::table(); }
}  // namespace dgb
