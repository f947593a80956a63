// ref_ext.hpp -- TEST INFRASTRUCTURE (oracle): the extension operators the
// reference lacks, registered through its public
// OpRegistry API.  Shared by oracle/ref_harness.cpp (mr_ref) and
// integration/ref_b200_run.cpp, which must parse the same modules.
//
//   max_pool2d(x, win[C,C,KH,KW], strides, padding)   -> ComplexOutFusable
//   depthwise_conv2d(x, win[C,C,KH,KW], w[C,1,KH,KW], strides, padding)
// Kernels follow kernels.cpp:640-716 conventions: NCHW, padded taps skipped,
// sequential accumulation (max seeded with the first valid tap, then std::max
// like reduce_impl kernels.cpp:519-566).
#pragma once

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "microrelay/interp.hpp"
#include "microrelay/registry.hpp"

namespace mr_ext {
using namespace microrelay;

inline const TensorLiteral& tens(const ValueRef& v) {
  if (!v || v->kind != ValueKind::Tensor) diag_throw(DiagCode::TypeMismatch, "expected tensor");
  return v->tensor;
}

inline ValueRef k_max_pool2d(const std::vector<ValueRef>& args, const AttrMap& attrs,
                      const SourceSpan& s) {
  const TensorLiteral& x = tens(args[0]);
  const TensorLiteral& win = tens(args[1]);
  if (!(x.dtype.is_float() && x.dtype.bits == 32))
    diag_throw(DiagCode::TypeMismatch, "max_pool2d: float32 only", s);
  auto strides = attr_int_list_opt(attrs, "strides").value_or(std::vector<int64_t>{1, 1});
  auto padding = attr_int_list_opt(attrs, "padding").value_or(std::vector<int64_t>{0, 0});
  auto xd = x.shape.to_ints();
  auto wd = win.shape.to_ints();
  int64_t N = xd[0], C = xd[1], H = xd[2], W = xd[3], KH = wd[2], KW = wd[3];
  int64_t sh = strides[0], sw = strides[1], ph = padding[0], pw = padding[1];
  int64_t OH = (H - KH + 2 * ph) / sh + 1, OW = (W - KW + 2 * pw) / sw + 1;
  TensorLiteral out = TensorLiteral::zeros(Shape::of({N, C, OH, OW}), x.dtype);
  const float* xp = x.f32s().data();
  float* op = out.f32s().data();
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          float acc = 0.0f;
          bool seeded = false;
          for (int64_t kh = 0; kh < KH; ++kh)
            for (int64_t kw = 0; kw < KW; ++kw) {
              int64_t h = oh * sh - ph + kh, w = ow * sw - pw + kw;
              if (h < 0 || h >= H || w < 0 || w >= W) continue;
              float v = xp[((n * C + c) * H + h) * W + w];
              if (!seeded) {
                acc = v;
                seeded = true;
              } else {
                acc = std::max(acc, v);
              }
            }
          op[((n * C + c) * OH + oh) * OW + ow] = acc;
        }
  return make_tensor_value(std::move(out));
}

inline ValueRef k_depthwise_conv2d(const std::vector<ValueRef>& args, const AttrMap& attrs,
                            const SourceSpan& s) {
  const TensorLiteral& x = tens(args[0]);
  const TensorLiteral& w = tens(args[2]);
  if (!(x.dtype.is_float() && x.dtype.bits == 32))
    diag_throw(DiagCode::TypeMismatch, "depthwise_conv2d: float32 only", s);
  auto strides = attr_int_list_opt(attrs, "strides").value_or(std::vector<int64_t>{1, 1});
  auto padding = attr_int_list_opt(attrs, "padding").value_or(std::vector<int64_t>{0, 0});
  auto xd = x.shape.to_ints();
  auto wd = w.shape.to_ints();
  int64_t N = xd[0], C = xd[1], H = xd[2], W = xd[3], KH = wd[2], KW = wd[3];
  if (wd[0] != C || wd[1] != 1)
    diag_throw(DiagCode::TypeMismatch, "depthwise_conv2d: weight must be [C,1,KH,KW]", s);
  int64_t sh = strides[0], sw = strides[1], ph = padding[0], pw = padding[1];
  int64_t OH = (H - KH + 2 * ph) / sh + 1, OW = (W - KW + 2 * pw) / sw + 1;
  TensorLiteral out = TensorLiteral::zeros(Shape::of({N, C, OH, OW}), x.dtype);
  const float* xp = x.f32s().data();
  const float* wp = w.f32s().data();
  float* op = out.f32s().data();
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          float facc = 0.0f;
          for (int64_t kh = 0; kh < KH; ++kh)
            for (int64_t kw = 0; kw < KW; ++kw) {
              int64_t h = oh * sh - ph + kh, ww = ow * sw - pw + kw;
              if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
              facc += xp[((n * C + c) * H + h) * W + ww] * wp[(c * KH + kh) * KW + kw];
            }
          op[((n * C + c) * OH + oh) * OW + ow] = facc;
        }
  return make_tensor_value(std::move(out));
}

inline std::shared_ptr<const OpRegistry> ext_registry() {
  static std::shared_ptr<const OpRegistry> reg = [] {
    auto r = std::make_shared<OpRegistry>(*builtin_registry());
    std::map<std::string, AttrKind> schema = {{"strides", AttrKind::IntList},
                                              {"padding", AttrKind::IntList},
                                              {"layout", AttrKind::String}};
    r->register_op(OperatorDecl{"max_pool2d", 2, schema, "Conv2D",
                                FusionPattern::ComplexOutFusable, k_max_pool2d});
    r->register_op(OperatorDecl{"depthwise_conv2d", 3, schema, "Conv2D",
                                FusionPattern::ComplexOutFusable, k_depthwise_conv2d});
    return std::shared_ptr<const OpRegistry>(r);
  }();
  return reg;
}

// ---- binary tensor files ---------------------------------------------------
// Format (little endian): int32 count; per tensor: int32 ndim, int64 dims[ndim],
// float32 data[prod(dims)].

inline std::vector<TensorLiteral> read_tensors(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) diag_throw(DiagCode::Internal, "cannot open " + path);
  int32_t n = 0;
  std::vector<TensorLiteral> out;
  if (std::fread(&n, 4, 1, f) != 1) diag_throw(DiagCode::Internal, "short read " + path);
  for (int32_t i = 0; i < n; ++i) {
    int32_t nd = 0;
    if (std::fread(&nd, 4, 1, f) != 1) diag_throw(DiagCode::Internal, "short read");
    std::vector<int64_t> dims(nd);
    if (nd && std::fread(dims.data(), 8, nd, f) != static_cast<size_t>(nd))
      diag_throw(DiagCode::Internal, "short read");
    int64_t cnt = 1;
    for (auto d : dims) cnt *= d;
    std::vector<float> v(cnt);
    if (cnt && std::fread(v.data(), 4, cnt, f) != static_cast<size_t>(cnt))
      diag_throw(DiagCode::Internal, "short read");
    out.push_back(TensorLiteral::from_f32(Shape::of(dims), std::move(v)));
  }
  std::fclose(f);
  return out;
}

inline void write_tensors(const std::string& path, const std::vector<const TensorLiteral*>& ts) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) diag_throw(DiagCode::Internal, "cannot open " + path);
  int32_t n = static_cast<int32_t>(ts.size());
  std::fwrite(&n, 4, 1, f);
  for (const TensorLiteral* t : ts) {
    if (!(t->dtype.is_float() && t->dtype.bits == 32))
      diag_throw(DiagCode::Internal, "result is not float32");
    auto dims = t->shape.to_ints();
    int32_t nd = static_cast<int32_t>(dims.size());
    std::fwrite(&nd, 4, 1, f);
    std::fwrite(dims.data(), 8, nd, f);
    std::fwrite(t->f32s().data(), 4, t->f32s().size(), f);
  }
  std::fclose(f);
}

inline std::string read_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) diag_throw(DiagCode::Internal, "cannot open " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

}  // namespace mr_ext
