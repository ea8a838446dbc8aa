// Generic operator kernels instantiated for dim = 2, space degree k = 3.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d2_k3() { return DegreeOps<2, 3>::table(); }
}  // namespace dgb
