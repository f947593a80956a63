// conv_tc.cu -- tcgen05 implicit-GEMM convolution (placeholder until the
// tensor-core kernel lands: nothing is eligible, so the executor selects the
// CUDA-core kernels at compile time).
#include "conv_tc.hpp"

namespace mrb200 {

struct TcConvPlan {
  ConvGeom g;
};

bool tc_conv_eligible(int, int, int, int, int) { return false; }
int tc_conv_weight_cstride(int C, int) { return (C + 3) / 4 * 4; }
TcConvPlan* tc_conv_create(const ConvGeom& g, int) { return new TcConvPlan{g}; }
void tc_conv_launch(TcConvPlan*, const void*, const void*, float, const EpiDev&, const OutDev&, cudaStream_t) {}
void tc_conv_destroy(TcConvPlan* p) { delete p; }

}  // namespace mrb200
