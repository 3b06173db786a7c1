// Tensor-core (tcgen05, 3xTF32) fused stencil + scattering GEMM apply.  Placeholder until the
// tcgen05 kernel lands: reports "unsupported" so rte_apply takes the SIMT kernel in apply.cu.
#include "common.h"

namespace rte {
bool apply_tc_supported(int) { return false; }
void free_tc_state(rte_problem*) {}
void launch_apply_tc(const rte_problem*, const float*, float*, const double*, int, cudaStream_t) {
  set_error("tensor-core apply not available");
  throw Fail{RTE_EINTERNAL};
}
}  // namespace rte
