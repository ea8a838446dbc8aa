// Generic operator kernels instantiated for dim = 3, space degree k = 4.
#include "ops_dispatch.cuh"

namespace dgb {
const OpTable& ops_d3_k4() { return DegreeOps<3, 4>::table(); }
}  // namespace dgb
