// conv_tc.hpp -- tcgen05 implicit-GEMM convolution (conv_tc.cu).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace mrb200 {

struct TcConvPlan;

// Compile-time eligibility (channel counts / tile shapes the kernel handles).
bool tc_conv_eligible(int C, int OC, int KH, int KW, int elem_bytes);
// Channel stride of the hoisted weight rows the kernel expects.
int tc_conv_weight_cstride(int C, int elem_bytes);
TcConvPlan* tc_conv_create(const ConvGeom& g, int elem_bytes);
void tc_conv_launch(TcConvPlan* p, const void* x, const void* w, float acc_scale, const EpiDev& epi,
                    const OutDev& out, cudaStream_t s);
void tc_conv_destroy(TcConvPlan* p);

}  // namespace mrb200
