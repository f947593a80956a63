// dense_tc.hpp -- tcgen05 dense (dense_tc.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace mrb200 {

struct DenseTcSpec {
  int eb;       // 1: int8 codes (kind::i8), 2: bf16 (kind::f16)
  int N, K, M;  // x [N, K] (float32 row-major), w [M, K], y [N, M]
};

struct DenseTcPlan;

DenseTcPlan* dense_tc_create(const DenseTcSpec& spec);
void dense_tc_destroy(DenseTcPlan* p);
int dense_tc_kp(int K, int eb);                            // padded K (elements): a multiple of 128 bytes
int64_t dense_tc_operand_bytes(const DenseTcPlan* p);      // A operand scratch [Npad, Kp]
int64_t dense_tc_workspace_bytes(const DenseTcPlan* p);    // split-K partials (0: no split)
int64_t dense_tc_weight_rows(const DenseTcPlan* p);        // B rows (M padded to the column tile)
int dense_tc_launches(const DenseTcPlan* p);
const char* dense_tc_describe(const DenseTcPlan* p, char* buf, int n);
// [M, K] float32 weight (+ folded per-row scale, scalar, realize chain) -> B [Mpad, Kp]
void dense_tc_prep_weight(const DenseTcPlan* p, const float* w, const float* oc_scale, float scalar, int quant,
                          QDev q, void* out, cudaStream_t s);
// operand prologue + tcgen05 contraction (+ split-K reduction); false: TMA encoding failed.
// x == nullptr: `operand` was written by the producer (the fused sum_hw).
bool dense_tc_launch(DenseTcPlan* p, const float* x, float pre_mul, int quant, QDev q, void* operand, const void* w,
                     void* ws, float acc_scale, const EpiDev& epi, const OutDev& out, cudaStream_t s);

}  // namespace mrb200
