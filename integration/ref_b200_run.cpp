// ref_b200_run.cpp -- the reference CLI's `run` (tools/microrelay.cpp:100-131)
// with the B200 hook in place of interp(): the module is parsed by the
// REFERENCE parser (parse_module, parser.hpp:17-19), then
//   interp   ModuleEnv -> interp(m, "main", args)      (the reference itself)
//   b200     ModuleEnv -> interp_b200(m, args)          (b200_backend.cpp)
//   session  B200Session created once, run twice (server loop)
//   group    B200Group(m, GROUP).apply(args)            (Interpreter::apply hook)
// usage: ref_b200_run MODE FUSED.rly ARGS.bin OUT.bin [GROUP BATCH]
// ARGS.bin = every argument in order (@main's, or the group's), the binary
// tensor format of oracle/ref_harness.cpp.
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "b200_backend.hpp"
#include "microrelay/parser.hpp"
#include "ref_ext.hpp"

using namespace microrelay;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: ref_b200_run interp|b200|session|group FUSED.rly ARGS.bin OUT.bin [GROUP BATCH]\n");
    return 2;
  }
  const std::string mode = argv[1];
  try {
    ModuleEnv m = parse_module(mr_ext::read_file(argv[2]), argv[2], mr_ext::ext_registry());
    std::vector<ValueRef> args;
    for (auto& t : mr_ext::read_tensors(argv[3])) args.push_back(make_tensor_value(std::move(t)));
    ValueRef r;
    if (mode == "interp") {
      InterpOptions opts;
      opts.fuel = INT64_MAX / 2;
      r = interp(m, "main", args, opts);
    } else if (mode == "b200") {
      r = interp_b200(m, args);
    } else if (mode == "session") {
      std::vector<ValueRef> w(args.begin() + 1, args.end());
      B200Session s(m, args[0]->tensor.shape.to_ints().at(0), w);
      ValueRef r1 = s.run(args[0]);
      r = s.run(args[0]);
      if (std::memcmp(r1->tensor.f32s().data(), r->tensor.f32s().data(), r->tensor.f32s().size() * 4) != 0)
        diag_throw(DiagCode::Internal, "session: two runs differ");
    } else if (mode == "group" && argc == 7) {
      B200Group g(m, argv[5], std::atoll(argv[6]));
      r = g.apply(args);
    } else {
      std::fprintf(stderr, "bad mode %s\n", mode.c_str());
      return 2;
    }
    const TensorLiteral& out = mr_ext::tens(r);
    mr_ext::write_tensors(argv[4], {&out});
    return 0;
  } catch (const Diagnostic& d) {
    std::fprintf(stderr, "ref_b200_run: diag %d: %s\n", static_cast<int>(d.code()), d.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_b200_run: %s\n", e.what());
    return 1;
  }
}
