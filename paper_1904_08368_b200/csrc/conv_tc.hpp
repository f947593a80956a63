// conv_tc.hpp -- tcgen05 implicit-GEMM convolution (conv_tc.cu).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace mrb200 {

// Which halo formulation a conv group uses (decided at compile time).
enum TcKind : int {
  TC_S1 = 0,        // stride-1 3x3/pad-1 or 1x1 over a LAY_NORMAL input
  TC_S2_PHASE = 1,  // stride-2 3x3/pad-1 or 1x1 over a LAY_PHASE input
  TC_STEM_S2D = 2,  // KxK stride-2 stem over the LAY_S2D network input
  TC_STEM_POOL = 3, // 7x7/s2 stem fused with a 3x3/s2/p1 max_pool2d over the LAY_S2DP input:
                    // M rows = pooled pixels, the 9 window taps = 3 super-tiles x 3 sub-tiles
};

struct TcConvSpec {
  int kind;
  int elem_bytes;  // 1: int8 (kind::i8), 2: bf16 (kind::f16)
  int N, C, H, W, OC, OH, OW, KH, KW;
  int Hs, Ws;      // TC_STEM_S2D input grid
  // Fused max_pool2d consumer (cross-group fusion of conv -> max_pool2d, the
  // conv output never leaves the SM): window, stride, padding, pooled dims.
  int pool = 0, pkh = 0, pkw = 0, psh = 1, psw = 1, pph = 0, ppw = 0, poh = 0, pow = 0;
  // the epilogue adds a residual (an epilogue-bound conv: the CTA-pair plan,
  // which helps weight-streaming convs, does not pay there -- measured)
  int residual = 0;
  // Fused 1x1/stride-2 shortcut (cross-group fusion of a ResNet downsampling
  // block): the residual operand of this 3x3 stride-1 conv is computed in the
  // same kernel -- a second accumulator over sc_C input channels read from a
  // stride-2 decimated int8 copy of the block input on this conv's own padded
  // grid (chunk width sc_kb, the shortcut weights' layout) -- instead of being
  // read back from the shortcut conv's float32 output.  0: none.
  int sc_C = 0, sc_kb = 0;
  // filled by planning
  int taps = 0, wplanes = 0;  // weight layout [taps][wplanes][OC][kb bytes]
  int kb = 0;                 // operand chunk bytes (the data representation's chunk width)
};

struct TcConvPlan;

// Device operands of the fused shortcut (TcConvSpec::sc_C): decimated codes
// (LAY_NORMAL on this conv's output grid), the shortcut's tcgen05 weights
// [1][sc_C/cpc][OC][cpc], its accumulator scale and bias vector.
struct TcShortcut {
  const void* x = nullptr;
  Lay lay{};
  const void* w = nullptr;
  float acc_scale = 1.f;
  const float* bias = nullptr;
};

// Compile-time eligibility (fills taps / wplanes).
bool tc_conv_plan_ok(TcConvSpec& spec);
TcConvPlan* tc_conv_create(const TcConvSpec& spec);
bool tc_conv_launch(TcConvPlan* p, const void* x, const Lay& xl, const void* w, float acc_scale, const EpiDev& epi,
                    const OutDev& out, cudaStream_t s, const TcShortcut* sc = nullptr);
void tc_conv_destroy(TcConvPlan* p);
const char* tc_conv_describe(const TcConvPlan* p, char* buf, int n);

}  // namespace mrb200
