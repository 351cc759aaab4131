// K3 tensor-core path (tcgen05 / TMA implicit GEMM) -- see DESIGN.md.
#include "conv.cuh"
#include "ts_common.cuh"

namespace ts {

bool conv_tc_supported(const ConvOp& op, int precision) {
  (void)op; (void)precision;
  return false;
}

int launch_conv_tc(const ConvOp& op, int precision, void* stream) {
  (void)op; (void)precision; (void)stream;
  return TS_E_INVALID;
}

}  // namespace ts
