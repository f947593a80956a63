// b200_backend.cpp -- see b200_backend.hpp.  Host tensors cross the C ABI as
// mr_tensor views of TensorLiteral's row-major float32 storage
// (literal.hpp:21-58); the module crosses it as print_module text
// (printer.hpp:16), which libmrb200 parses itself.
#include "b200_backend.hpp"

#include <cuda_runtime.h>

#include "microrelay/diagnostics.hpp"
#include "microrelay/literal.hpp"
#include "microrelay/printer.hpp"

namespace microrelay {
namespace {

const TensorLiteral& tensor_of(const ValueRef& v) {  // the check of kernels.cpp:19-23
  if (!v || v->kind != ValueKind::Tensor) diag_throw(DiagCode::TypeMismatch, "b200: expected a tensor argument");
  return v->tensor;
}

mr_tensor view(const TensorLiteral& t) {
  if (!(t.dtype.is_float() && t.dtype.bits == 32)) diag_throw(DiagCode::TypeMismatch, "b200: float32 tensors only");
  mr_tensor m{};
  m.data = const_cast<float*>(t.f32s().data());
  auto dims = t.shape.to_ints();
  m.ndim = static_cast<int32_t>(dims.size());
  for (size_t i = 0; i < dims.size(); ++i) m.shape[i] = dims[i];
  m.type_code = MR_FLOAT;
  m.bits = 32;
  return m;
}

// mr_status -> the reference's Diagnostic: codes 1..99 mirror DiagCode + 1.
[[noreturn]] void raise(mr_status st) {
  const std::string msg = std::string("b200: ") + mr_last_error_message();
  if (st > 0 && st < 100) diag_throw(static_cast<DiagCode>(static_cast<int>(st) - 1), msg);
  diag_throw(DiagCode::Internal, msg);
}

void check(mr_status st) {
  if (st != MR_OK) raise(st);
}

std::vector<int64_t> dims_of(const mr_tensor& t) { return std::vector<int64_t>(t.shape, t.shape + t.ndim); }

}  // namespace

ValueRef interp_b200(const ModuleEnv& fused, const std::vector<ValueRef>& args) {
  if (args.empty()) diag_throw(DiagCode::ArityMismatch, "b200: @main needs its data argument");
  std::vector<ValueRef> w(args.begin() + 1, args.end());
  B200Session s(fused, tensor_of(args[0]).shape.to_ints().at(0), w);
  return s.run(args[0]);
}

B200Session::B200Session(const ModuleEnv& fused, int64_t batch, const std::vector<ValueRef>& weights, int device) {
  mr_exec_options o;
  mr_exec_default_options(&o);
  o.batch = batch;
  o.device = device;
  const std::string text = print_module(fused);
  check(mr_exec_create(text.c_str(), &o, &ex_));
  std::vector<mr_tensor> w;
  for (const ValueRef& v : weights) w.push_back(view(tensor_of(v)));
  mr_status st = mr_exec_set_weights(ex_, static_cast<int32_t>(w.size()), w.empty() ? nullptr : w.data());
  if (st != MR_OK) {
    mr_exec_destroy(ex_);
    ex_ = nullptr;
    raise(st);
  }
  mr_tensor shape{};
  check(mr_exec_output_shape(ex_, &shape));
  out_dims_ = dims_of(shape);
}

B200Session::~B200Session() { mr_exec_destroy(ex_); }

ValueRef B200Session::run(const ValueRef& batch) {
  TensorLiteral out = TensorLiteral::zeros(Shape::of(out_dims_), BaseType::f32());
  mr_tensor in = view(tensor_of(batch)), res = view(out);
  check(mr_exec_run_host(ex_, &in, &res, nullptr));
  return make_tensor_value(std::move(out));
}

B200Group::B200Group(const ModuleEnv& fused, const std::string& group, int64_t batch, int device) {
  mr_exec_options o;
  mr_exec_default_options(&o);
  o.batch = batch;
  o.device = device;
  const std::string text = print_module(fused);
  check(mr_group_compile(text.c_str(), group.c_str(), &o, &g_));
  int32_t n = 0;
  mr_tensor shape{};
  check(mr_group_signature(g_, &n, &shape));
  n_operands_ = n;
  out_dims_ = dims_of(shape);
}

B200Group::~B200Group() { mr_group_destroy(g_); }

// Interpreter::apply's Closure case for a compiled group: the arguments are
// staged on the device, the group launches, the result comes back as a fresh
// TensorLiteral (the reference's value semantics, value.hpp:15-16).
ValueRef B200Group::apply(const std::vector<ValueRef>& args) {
  struct Dev {
    std::vector<void*> p;
    ~Dev() {
      for (void* q : p) cudaFree(q);
    }
  } dev;
  std::vector<mr_tensor> in;
  for (const ValueRef& a : args) {
    mr_tensor t = view(tensor_of(a));
    const size_t bytes = tensor_of(a).f32s().size() * sizeof(float);
    void* d = nullptr;
    if (cudaMalloc(&d, bytes ? bytes : 4) != cudaSuccess) diag_throw(DiagCode::Internal, "b200: cudaMalloc");
    dev.p.push_back(d);
    if (bytes && cudaMemcpy(d, t.data, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      diag_throw(DiagCode::Internal, "b200: upload");
    t.data = d;
    in.push_back(t);
  }
  TensorLiteral out = TensorLiteral::zeros(Shape::of(out_dims_), BaseType::f32());
  mr_tensor res = view(out);
  void* dout = nullptr;
  if (cudaMalloc(&dout, out.f32s().size() * sizeof(float)) != cudaSuccess) diag_throw(DiagCode::Internal, "b200: cudaMalloc");
  dev.p.push_back(dout);
  void* host = res.data;
  res.data = dout;
  check(mr_group_launch(g_, in.data(), static_cast<int32_t>(in.size()), &res, nullptr));
  if (cudaMemcpy(host, dout, out.f32s().size() * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
    diag_throw(DiagCode::Internal, "b200: download");
  return make_tensor_value(std::move(out));
}

}  // namespace microrelay
