// ref_harness.cpp -- TEST INFRASTRUCTURE (oracle), never linked by the product.
// Built as the executable oracle/_ref/mr_ref (a subprocess, not a ctypes .so:
// the reference library crashed when loaded into a numpy-importing process).
//
// A thin CLI over the UNMODIFIED reference library (MicroRelay, built from
// /root/reference/proj/core/src by oracle/Makefile) so pytest drives it as a
// subprocess (oracle/ref.py):
//   * parse_module            parser.hpp:17-19
//   * run_pipeline / passes   passes.cpp:490-501, passes.cpp:452-486
//   * quant_annotate/_calibrate/_realize   quantize.cpp:92-110, 138-177, 212-245
//   * interp                  interp.cpp:218-222
//   * print_module            printer.hpp:17
//
// Extension operators: the reference has no
// pooling or depthwise operator. They are registered through the reference's
// own public operator API (OpRegistry::register_op on a copy of the builtin
// registry, as test_registry.cpp:21-31 does), reusing the existing "Conv2D"
// type relation (registry.cpp:412-469) with a shape-only window argument:
//   max_pool2d(x, win[C,C,KH,KW], strides, padding)   -> ComplexOutFusable
//   depthwise_conv2d(x, win[C,C,KH,KW], w[C,1,KH,KW], strides, padding)
// Their kernels follow kernels.cpp:640-716 conventions: NCHW, padded taps
// skipped, sequential accumulation (max seeded with the first valid tap,
// then std::max like reduce_impl kernels.cpp:519-566).
#include <chrono>
#include <climits>
#include <cstdio>
#include <fstream>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "microrelay/analysis.hpp"
#include "microrelay/expr.hpp"
#include "microrelay/infer.hpp"
#include "microrelay/interp.hpp"
#include "microrelay/parser.hpp"
#include "microrelay/passes.hpp"
#include "microrelay/printer.hpp"
#include "microrelay/quantize.hpp"
#include "microrelay/registry.hpp"
#include "ref_ext.hpp"

using namespace microrelay;

namespace {

using mr_ext::ext_registry;
using mr_ext::read_file;
using mr_ext::read_tensors;
using mr_ext::tens;
using mr_ext::write_tensors;

// ---- fixed-scale quantization ---------------------------------------------

bool is_simq(const ExprRef& e) {
  return e->kind == ExprKind::Call && e->a->kind == ExprKind::OperatorRef &&
         e->a->name == "simulated_quantize";
}

// Sets attr scale on every simulated_quantize call: the same rewrite
// quant_calibrate applies per trial (with_global_scale, quantize.cpp:123-134).
ExprRef set_scale(const ExprRef& e, double scale) {
  if (!e) return e;
  switch (e->kind) {
    case ExprKind::LocalVar:
    case ExprKind::GlobalVar:
    case ExprKind::Constant:
    case ExprKind::OperatorRef:
    case ExprKind::ConstructorRef:
      return e;
    default: {
      auto copy = std::make_shared<Expr>(*e);
      copy->checked_type = nullptr;
      if (e->a) copy->a = set_scale(e->a, scale);
      if (e->b) copy->b = set_scale(e->b, scale);
      if (e->c) copy->c = set_scale(e->c, scale);
      copy->elems.clear();
      for (const auto& x : e->elems) copy->elems.push_back(set_scale(x, scale));
      copy->clauses.clear();
      for (const auto& cl : e->clauses) copy->clauses.push_back({cl.pattern, set_scale(cl.body, scale)});
      if (is_simq(copy)) copy->attrs["scale"] = scale;
      return copy;
    }
  }
}

double find_scale(const ExprRef& e) {
  if (!e) return 0;
  if (is_simq(e)) {
    auto s = attr_float_opt(e->attrs, "scale");
    if (s) return *s;
  }
  for (const ExprRef& c : {e->a, e->b, e->c}) {
    double s = find_scale(c);
    if (s != 0) return s;
  }
  for (const auto& x : e->elems) {
    double s = find_scale(x);
    if (s != 0) return s;
  }
  return 0;
}

std::vector<std::string> split_passes(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

ModuleEnv run_passes(const ModuleEnv& m, const std::vector<std::string>& passes) {
  std::string joined;
  for (const auto& p : passes) joined += (joined.empty() ? "" : ",") + p;
  if (joined.empty()) return infer(m);
  return run_pipeline(m, PassContext::from_pass_list(joined));
}

// passes before "quantize", "quantize" itself (fixed k), passes after.
ModuleEnv compile_fixed_k(const ModuleEnv& m0, const std::string& passes, int k) {
  auto list = split_passes(passes);
  std::vector<std::string> pre, post;
  bool quant = false;
  for (const auto& p : list) {
    if (p == "quantize") {
      quant = true;
    } else {
      (quant ? post : pre).push_back(p);
    }
  }
  ModuleEnv m = run_passes(m0, pre);
  if (quant) {
    // apply_one_pass "quantize" (passes.cpp:471-478) with quant_calibrate
    // replaced by its result for global scale 2^k.
    QuantConfig cfg;
    ModuleEnv annotated = infer(quant_annotate(m, QuantRules::defaults(), cfg));
    ModuleEnv calibrated = annotated;
    for (auto& [name, fn] : calibrated.globals) fn = set_scale(fn, std::ldexp(1.0, k));
    m = infer(quant_realize(infer(calibrated), cfg));
  }
  return run_passes(m, post);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int usage() {
  std::fprintf(stderr,
               "usage:\n"
               "  mr_ref compile  MODEL.rly PASSES K            -> fused module on stdout\n"
               "  mr_ref calibrated MODEL.rly PASSES ARGS.bin   -> run_pipeline w/ quant_calibrate\n"
               "  mr_ref calibrate MODEL.rly PRE_PASSES ARGS.bin -> k on stdout\n"
               "  mr_ref run FUSED.rly WEIGHTS.bin IMAGES.bin OUT.bin\n"
               "      interp(@main) once per image of IMAGES.bin's first tensor ([B,...] ->\n"
               "      batch-1 calls), WEIGHTS.bin = the remaining @main args in order;\n"
               "      per-image seconds on stderr as 'image i t'\n"
               "  mr_ref runall FUSED.rly WEIGHTS.bin IMAGES.bin OUT.bin\n"
               "      one interp(@main) over the whole batch (static-batch modules, e.g. a\n"
               "      reshape to (B, C*H*W)); seconds on stderr as 'batch t'\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  std::string cmd = argv[1];
  try {
    if (cmd == "compile" && argc == 5) {
      ModuleEnv m = parse_module(read_file(argv[2]), argv[2], ext_registry());
      std::fputs(print_module(compile_fixed_k(m, argv[3], std::atoi(argv[4]))).c_str(), stdout);
      return 0;
    }
    if ((cmd == "calibrate" || cmd == "calibrated") && argc == 5) {
      ModuleEnv m = parse_module(read_file(argv[2]), argv[2], ext_registry());
      std::vector<ValueRef> args;
      for (auto& t : read_tensors(argv[4])) args.push_back(make_tensor_value(std::move(t)));
      if (cmd == "calibrated") {
        // The stock pipeline end to end (passes.cpp:471-478 calls quant_calibrate).
        PassContext ctx = PassContext::from_pass_list(argv[3]);
        ctx.calibration_inputs.push_back(args);
        std::fputs(print_module(run_pipeline(m, ctx)).c_str(), stdout);
        return 0;
      }
      ModuleEnv pre = run_passes(m, split_passes(argv[3]));
      ModuleEnv cal = quant_calibrate(infer(quant_annotate(pre)), {args}, "main");
      double s = 0;
      for (const auto& [name, fn] : cal.globals)
        if ((s = find_scale(fn)) != 0) break;
      if (s == 0) diag_throw(DiagCode::Internal, "no simulated_quantize site");
      std::printf("%d\n", static_cast<int>(std::lround(std::log2(s))));
      return 0;
    }
    if (cmd == "runall" && argc == 6) {
      ModuleEnv m = parse_module(read_file(argv[2]), argv[2], ext_registry());
      std::vector<TensorLiteral> weights = read_tensors(argv[3]);
      std::vector<TensorLiteral> images = read_tensors(argv[4]);
      if (images.size() != 1) diag_throw(DiagCode::Internal, "IMAGES.bin must hold one tensor");
      std::vector<ValueRef> args{make_tensor_value(images[0])};
      for (auto& w : weights) args.push_back(make_tensor_value(std::move(w)));
      InterpOptions opts;
      opts.fuel = INT64_MAX / 2;
      double t0 = now_s();
      ValueRef r = interp(m, "main", args, opts);
      std::fprintf(stderr, "batch %.6f\n", now_s() - t0);
      TensorLiteral out = tens(r);
      write_tensors(argv[5], {&out});
      return 0;
    }
    if (cmd == "run" && argc == 6) {
      ModuleEnv m = parse_module(read_file(argv[2]), argv[2], ext_registry());
      std::vector<TensorLiteral> weights = read_tensors(argv[3]);
      std::vector<TensorLiteral> images = read_tensors(argv[4]);
      if (images.size() != 1) diag_throw(DiagCode::Internal, "IMAGES.bin must hold one tensor");
      const TensorLiteral& batch = images[0];
      auto dims = batch.shape.to_ints();
      int64_t B = dims[0], per = batch.num_elements() / std::max<int64_t>(B, 1);
      std::vector<int64_t> one = dims;
      one[0] = 1;
      std::vector<ValueRef> wargs;
      for (auto& w : weights) wargs.push_back(make_tensor_value(std::move(w)));
      std::vector<TensorLiteral> results;
      InterpOptions opts;
      opts.fuel = INT64_MAX / 2;
      for (int64_t i = 0; i < B; ++i) {
        std::vector<float> img(batch.f32s().begin() + i * per, batch.f32s().begin() + (i + 1) * per);
        std::vector<ValueRef> args{make_tensor_value(TensorLiteral::from_f32(Shape::of(one), std::move(img)))};
        args.insert(args.end(), wargs.begin(), wargs.end());
        double t0 = now_s();
        ValueRef r = interp(m, "main", args, opts);
        std::fprintf(stderr, "image %lld %.6f\n", static_cast<long long>(i), now_s() - t0);
        results.push_back(tens(r));
      }
      // Concatenate the batch-1 results along axis 0.
      std::vector<float> all;
      std::vector<int64_t> rd = results.empty() ? std::vector<int64_t>{0} : results[0].shape.to_ints();
      for (auto& r : results) all.insert(all.end(), r.f32s().begin(), r.f32s().end());
      rd[0] = B;
      TensorLiteral out = TensorLiteral::from_f32(Shape::of(rd), std::move(all));
      write_tensors(argv[5], {&out});
      return 0;
    }
    return usage();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "mr_ref: %s\n", e.what());
    return 1;
  }
}
