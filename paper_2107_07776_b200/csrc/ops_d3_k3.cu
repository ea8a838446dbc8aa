// Generic operator kernels instantiated for dim = 3, space degree k = 3.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d3_k3() { return DegreeOps<3, 3>::table(); }
}  // namespace dgb
