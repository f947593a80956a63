// lower.hpp -- fused-group lowering: Primitive function bodies -> GroupDesc.
//
// FuseOps (fuse.cpp:115-163) guarantees every group has at most one
// ComplexOutFusable op (conv2d / dense / max_pool2d / depthwise_conv2d), that
// everything fused before it is <= Injective on its inputs (prologue chains)
// and that the group has exactly one output (the anchor's post-dominating
// chain).  The realize pass (quantize.cpp:181-201, 233-240)
// expands each quantize site into the fixed 6-op chain
//     multiply(x, c1) -> round -> clip(lo, hi) -> cast(int8) -> cast(float32)
//     -> multiply(c2)
// which this lowering recognises as one Requant op.  A body that does not
// decompose into  prologue(data) , prologue(weight) -> anchor -> epilogue
// is rejected with MR_ERR_UNSUPPORTED_GROUP at compile time (no fallback).
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "relay_text.hpp"

namespace mrb200 {

// A realized quantize site: value' = cast_f32(cast_i8(clip(round(v*c1), lo, hi))) * c2
// (quantize.cpp:181-201 + the standalone-site rescale quantize.cpp:233-240).
struct QParams {
  float c1 = 1.f, lo = -128.f, hi = 127.f, c2 = 1.f;
  bool is_signed = true;  // cast to int8 (sign=1) or uint8
  bool operator==(const QParams& o) const {
    return c1 == o.c1 && lo == o.lo && hi == o.hi && c2 == o.c2 && is_signed == o.is_signed;
  }
};

enum class EpiKind : int32_t {
  MulScalar = 1,   // multiply(v, const scalar)            kernels.cpp:174-179 (double, then f32)
  MulChannel = 2,  // multiply(v, const [C,1,1])           "
  Bias = 3,        // bias_add(v, %b)                      kernels.cpp:718-739
  Residual = 4,    // add(v, %r) / add(%r, v), same shape  kernels.cpp:160-165
  Relu = 5,        // x > 0 ? x : 0.0f                     kernels.cpp:281-286
  Requant = 6,     // the 6-op realize chain               quantize.cpp:181-201
  Clip = 7,        // clip(v, lo, hi)                      kernels.cpp:296-316
  SumHW = 8,       // sum(v, axis=(2,3)), must be last     kernels.cpp:519-575
  Flatten = 9,     // reshape [N,C,H,W] -> [N, C*H*W] (a view: row-major NCHW order), must be last
                   //                                      kernels.cpp:390-397
};

struct EpiOp {
  EpiKind kind;
  float s = 0.f;            // MulScalar
  std::vector<float> vec;   // MulChannel
  int value = -1;           // Bias / Residual: @main-level value index
  QParams q;                // Requant
  float lo = 0.f, hi = 0.f; // Clip
};

// One @main-level tensor: a parameter of @main or a group's output.
struct ValueInfo {
  std::string name;
  std::vector<int64_t> shape;  // logical (NCHW / [N,C]), batch bound
  int producer = -1;           // group index, -1 for a @main parameter
  int param_index = -1;        // @main parameter position
  bool is_data = false;        // one of the n_data_inputs leading params
  bool quantized = false;      // producer's epilogue ends in Requant: value == code * q.c2
  QParams q;
  std::vector<int> consumers;  // groups reading it
  bool is_result = false;
  // @main-level `let %t = <constant>` (weights embedded in the module's
  // metadata pool, e.g. after `fold`): a hidden parameter the executor uploads
  // itself, param_index >= the module's own parameter count
  int hidden = -1;  // index into Program::hidden_data
  // layout pass (passes.cpp:481-486): the reference value is the NHWC
  // transpose of this NCHW tensor (its producer ended in transpose(0,2,3,1));
  // only NHWC conv2d consumers read it (data layouts here are physical)
  bool nhwc_view = false;
};

enum class GroupKind { Conv, Dense, MaxPool, DwConv };

// A weight operand: @main param (or constant) with its weight-only prologue,
// hoisted to weight-load time.
struct WeightOperand {
  int value = -1;                // @main param value index, or -1 if constant
  std::vector<float> constant;   // literal weight when value == -1
  std::vector<int64_t> shape;    // OIHW / [M,K]
  std::vector<float> oc_scale;   // multiply(w, const[OC,1,1,1]) (fold-scale), empty if none
  float scalar_scale = 0.f;      // multiply(w, const scalar), 0 if none
  bool quant = false;
  QParams q;
};

struct DataOperand {
  int value = -1;
  float pre_mul = 0.f;  // multiply(x, const scalar) before quantize (head 1/HW), 0 if none
  bool quant = false;   // realize chain applied to the input in this group
  QParams q;
};

struct GroupDesc {
  std::string name;       // %fusedN
  std::string out_name;   // let-bound result
  GroupKind kind = GroupKind::Conv;
  DataOperand data;
  WeightOperand weight;
  int window_value = -1;  // max_pool2d / depthwise shape-only window
  int64_t kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
  std::vector<EpiOp> epi;
  std::vector<int> param_values;  // fn params in order (= free_vars order, fuse.cpp:296-302)
  int out_value = -1;
  std::vector<int64_t> in_shape;   // data operand logical shape
  std::vector<int64_t> out_shape;  // group output logical shape
  std::vector<int64_t> pre_sum_shape;  // conv output before SumHW (if any)
};

struct Program {
  std::vector<ValueInfo> values;
  std::vector<GroupDesc> groups;  // in call (topological) order
  int result_value = -1;
  int n_params = 0;  // @main parameters + hidden constant parameters
  std::vector<std::vector<float>> hidden_data;  // float32 literal per hidden parameter
  bool any_quant = false;
};

struct LowerError {
  int code;  // mr_status
  std::string msg;
};

// Lowers the parsed fused module with the symbolic batch bound to `batch`.
// `coded_inputs` marks data params that carry realize-coded values (code * c2,
// as another group's Requant epilogue leaves them) -- the group level's view
// of an operand its producer quantized.
Program lower_module(const Module& m, int64_t batch, int n_data_inputs,
                     const std::map<std::string, QParams>* coded_inputs = nullptr);

std::string describe_group(const Program& p, const GroupDesc& g);

// One Primitive group of a fused module as a module of its own (the group
// level of the boundary: one closure application,
// interp.cpp:86-101).  `group` names the function (%fusedN) or the value its
// call binds (%vN).
struct GroupModule {
  Module m;               // @main takes the group's distinct call arguments,
                          // activations first (their shapes bound to the batch),
                          // then the @main weight params
  std::vector<int> perm;  // m's param k = the group's call argument perm[k]
  int n_data = 0;         // activations among m's params
  std::map<std::string, QParams> coded;  // activations the full module holds realize-coded
  bool module_quant = false;             // the full module has quantize sites (float format choice)
};
GroupModule extract_group_module(const Module& m, const std::string& group, int64_t batch, int n_data_inputs);

}  // namespace mrb200
