// launch.hpp -- host entry points of the CUDA kernels (one per kernel family).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace mrb200 {

// Launches a graph kernel with programmatic stream serialization (PDL): it may
// start while its predecessor drains; the kernel calls pdl_wait() before
// reading or writing activations.  MRB200_NO_PDL=1 launches plainly.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// pdl_launch with thread-block clusters of `cluster` CTAs along x (CTA pairs
// for the tcgen05 cta_group::2 conv plans); cluster 1 is pdl_launch.
template <typename... KArgs, typename... Args>
inline void pdl_launch_cluster(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                               Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = static_cast<unsigned>(cluster);
    at[n].val.clusterDim.y = 1;
    at[n++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

enum WeightLayout : int { WL_ROWS = 0, WL_TC = 1, WL_S2D = 2 };

void launch_input_convert(const float* x, int N, int C, int H, int W, void* out, int fmt, const Lay& L,
                          int s2d_pad, float pre_mul, QDev q, cudaStream_t s);
void launch_to_nchw(const void* x, int fmt, const Lay& L, float c2, float* y, int N, int C, int H, int W, int is4d,
                    cudaStream_t s, const QDev* rq = nullptr);
void launch_zero_border(void* buf, const Lay& L, int N, cudaStream_t s);
void launch_weight_prep(const float* w, int O, int I, int KH, int KW, int Cs, int wl, const float* oc_scale,
                        float scalar, int fmt, int quant, QDev q, void* out, cudaStream_t s);
void launch_conv_i8_simt(const int8_t* x, const int8_t* w, const ConvGeom& g, float acc_scale,
                         const EpiDev& epi, const OutDev& out, cudaStream_t s);
void launch_conv_bf16_simt(const uint16_t* x, const uint16_t* w, const ConvGeom& g, const EpiDev& epi,
                           const OutDev& out, cudaStream_t s);
void launch_conv_f32_strict(const float* x, const float* w, const ConvGeom& g, const EpiDev& epi,
                            const OutDev& out, cudaStream_t s);
void launch_dwconv(const void* x, int xfmt, const float* w, const ConvGeom& g, int strict, const EpiDev& epi,
                   const OutDev& out, cudaStream_t s);
void launch_maxpool(const void* x, int xfmt, const ConvGeom& g, const OutDev& out, cudaStream_t s);
// The consumer dense's A operand written by the sum itself (cross-group fusion of
// sum -> multiply(1/HW) -> realize -> dense): [Npad][Kp] int8 codes / bf16 / tf32.
struct SumOperand {
  void* ptr = nullptr;
  int eb = 1, Kp = 0;
  float pre_mul = 0.f;
  int quant = 0;
  QDev q{};
};
void launch_sum_hw(const float* x, const Lay& L, int N, int H, int W, int C, float* y, cudaStream_t s,
                   const SumOperand* op = nullptr);
void launch_dense_weight_t(const float* w, int M, int K, int Kp, const float* oc_scale, float scalar, int fmt,
                           int quant, QDev q, void* out, cudaStream_t s);
void launch_dense(const float* x, int N, int K, int Kp, const void* w, int M, int mode, float pre_mul,
                  int quant, QDev q, float acc_scale, const EpiDev& epi, const OutDev& out, cudaStream_t s);

}  // namespace mrb200
