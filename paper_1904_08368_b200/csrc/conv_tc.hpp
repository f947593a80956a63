// conv_tc.hpp -- tcgen05 implicit-GEMM convolution (conv_tc.cu).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace mrb200 {

struct TcConvPlan;

// Compile-time eligibility of a conv group (stride-1 3x3/pad-1 or 1x1, channel
// counts in whole 32-byte MMA K steps, halo within one TMA box).
bool tc_conv_eligible(const ConvGeom& g, int elem_bytes);
TcConvPlan* tc_conv_create(const ConvGeom& g, int elem_bytes);
// x: P16 activations (pad kPad), w: [taps][C/cpc][OC][cpc] weights (WL_TC).
bool tc_conv_launch(TcConvPlan* p, const void* x, const void* w, float acc_scale, const EpiDev& epi,
                    const OutDev& out, cudaStream_t s);
void tc_conv_destroy(TcConvPlan* p);
const char* tc_conv_describe(const TcConvPlan* p, char* buf, int n);

}  // namespace mrb200
