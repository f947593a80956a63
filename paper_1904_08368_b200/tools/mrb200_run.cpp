// mrb200_run -- C++ host program over the C ABI (include/mrb200.h): the B200
// counterpart of the reference CLI's `run` command (tools/microrelay.cpp:100-131),
// for a module after run_pipeline(..., "fuse") (print_module text).
//
//   mrb200_run FUSED.rly ARGS.bin OUT.bin [--fp32-strict] [--repeat R]
//
// ARGS.bin / OUT.bin: int32 count, then per tensor int32 ndim, int64 dims[ndim],
// float32 row-major data (little endian).  ARGS holds the @main arguments in
// parameter order, the batch first (its dim 0 binds ?n).  Exit status: 0, or
// the mr_status of the failing call (DiagCode ordinal + 1, 100-103 backend).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/mrb200.h"

namespace {

struct HostTensor {
  std::vector<int64_t> dims;
  std::vector<float> data;
};

bool read_tensors(const char* path, std::vector<HostTensor>* out) {
  std::ifstream f(path, std::ios::binary);
  int32_t n = 0;
  if (!f.read(reinterpret_cast<char*>(&n), 4) || n < 0) return false;
  for (int32_t i = 0; i < n; ++i) {
    int32_t nd = 0;
    if (!f.read(reinterpret_cast<char*>(&nd), 4) || nd < 0 || nd > 8) return false;
    HostTensor t;
    t.dims.resize(static_cast<size_t>(nd));
    if (nd && !f.read(reinterpret_cast<char*>(t.dims.data()), 8 * nd)) return false;
    int64_t cnt = 1;
    for (int64_t d : t.dims) cnt *= d;
    t.data.resize(static_cast<size_t>(cnt));
    if (cnt && !f.read(reinterpret_cast<char*>(t.data.data()), 4 * cnt)) return false;
    out->push_back(std::move(t));
  }
  return true;
}

bool write_tensor(const char* path, const HostTensor& t) {
  std::ofstream f(path, std::ios::binary);
  const int32_t n = 1, nd = static_cast<int32_t>(t.dims.size());
  f.write(reinterpret_cast<const char*>(&n), 4);
  f.write(reinterpret_cast<const char*>(&nd), 4);
  f.write(reinterpret_cast<const char*>(t.dims.data()), 8 * nd);
  f.write(reinterpret_cast<const char*>(t.data.data()), static_cast<std::streamsize>(4 * t.data.size()));
  return static_cast<bool>(f);
}

mr_tensor view(HostTensor& t) {
  mr_tensor m;
  std::memset(&m, 0, sizeof(m));
  m.data = t.data.data();
  m.ndim = static_cast<int32_t>(t.dims.size());
  for (size_t i = 0; i < t.dims.size(); ++i) m.shape[i] = t.dims[i];
  m.type_code = MR_FLOAT;
  m.bits = 32;
  return m;
}

int fail(mr_status st, const char* what) {
  std::fprintf(stderr, "mrb200_run: %s: status %d: %s\n", what, static_cast<int>(st), mr_last_error_message());
  return static_cast<int>(st);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s FUSED.rly ARGS.bin OUT.bin [--fp32-strict] [--repeat R]\n(%s)\n", argv[0],
                 mr_build_info());
    return 2;
  }
  bool strict = false;
  int repeat = 1;
  for (int i = 4; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--fp32-strict")) strict = true;
    else if (!std::strcmp(argv[i], "--repeat") && i + 1 < argc) repeat = std::atoi(argv[++i]);
  }
  std::ifstream mf(argv[1]);
  if (!mf) {
    std::fprintf(stderr, "mrb200_run: cannot read %s\n", argv[1]);
    return 2;
  }
  std::stringstream ss;
  ss << mf.rdbuf();
  const std::string text = ss.str();
  std::vector<HostTensor> args;
  if (!read_tensors(argv[2], &args) || args.empty()) {
    std::fprintf(stderr, "mrb200_run: bad tensor file %s\n", argv[2]);
    return 2;
  }
  mr_exec_options o;
  mr_exec_default_options(&o);
  o.batch = args[0].dims.empty() ? 1 : args[0].dims[0];
  if (strict) o.float_mode = MR_FLOAT_FP32_STRICT;
  mr_exec_t ex = nullptr;
  mr_status st = mr_exec_create(text.c_str(), &o, &ex);
  if (st != MR_OK) return fail(st, "mr_exec_create");
  std::vector<mr_tensor> w;
  for (size_t i = 1; i < args.size(); ++i) w.push_back(view(args[i]));
  st = mr_exec_set_weights(ex, static_cast<int32_t>(w.size()), w.data());
  if (st != MR_OK) return fail(st, "mr_exec_set_weights");
  mr_tensor shape;
  st = mr_exec_output_shape(ex, &shape);
  if (st != MR_OK) return fail(st, "mr_exec_output_shape");
  HostTensor out;
  int64_t cnt = 1;
  for (int i = 0; i < shape.ndim; ++i) {
    out.dims.push_back(shape.shape[i]);
    cnt *= shape.shape[i];
  }
  out.data.resize(static_cast<size_t>(cnt));
  mr_tensor in = view(args[0]), res = view(out);
  for (int r = 0; r < repeat; ++r) {
    st = mr_exec_run_host(ex, &in, &res, nullptr);
    if (st != MR_OK) return fail(st, "mr_exec_run_host");
  }
  mr_exec_destroy(ex);
  if (!write_tensor(argv[3], out)) {
    std::fprintf(stderr, "mrb200_run: cannot write %s\n", argv[3]);
    return 2;
  }
  return 0;
}
