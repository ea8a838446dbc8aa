// Generic operator kernels instantiated for dim = 2, space degree k = 4.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d2_k4() { return DegreeOps<2, 4>::table(); }
}  // namespace dgb
