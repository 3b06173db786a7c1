// Tensor-core (tcgen05, 3xTF32) implicit-GEMM convolutions.  Placeholder until the tcgen05
// kernel lands: every shape falls back to the SIMT implicit GEMM in mgnet.cu.
#include "mgnet.h"

namespace rte {
bool conv_tc_try(const ConvDesc&, const float*, float*, const float*, float, const double*, int, bool, bool,
                 cudaStream_t) {
  return false;
}
void conv_tc_prepare(mgnet_net* net) { net->tc = false; }
}  // namespace rte
