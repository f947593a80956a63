// exec.cpp -- the executor behind the C ABI (include/mrb200.h).
//
// Replaces Interpreter::run / eval_in (interp.cpp:21-26, 124-216) for a fused
// module: the let-chain walk becomes a static launch list (one kernel per
// Primitive group, plus boundary conversions), every intermediate gets a fixed
// address in one device arena (liveness-based first-fit, planned once), the
// weight-only prologues are hoisted to mr_exec_set_weights, and the launch
// list is captured once into a CUDA graph and replayed per call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/mrb200.h"
#include "conv_tc.hpp"
#include "dense_tc.hpp"
#include "kernels.cuh"
#include "launch.hpp"
#include "lower.hpp"
#include "relay_text.hpp"

namespace mrb200 {

thread_local std::string g_last_error;

struct Status {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Status{code, msg}; }

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(MR_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Set while a calibration trial executor is built and its weights prepared:
// every QDev then carries the trial's device overflow flag (mr_calibrate).
thread_local int32_t* g_calib_ovf = nullptr;

QDev to_qdev(const QParams& q) { return QDev{q.c1, q.lo, q.hi, q.c2, q.is_signed ? 1 : 0, g_calib_ovf}; }

// The module with every quantize site at global scale rho = 2^k
// (with_global_scale, quantize.cpp:123-134): realize's constants are
// c1 = 2^(bits-sign) / rho and c2 = rho / 2^(bits-sign) (quantize.cpp:181-201).
void rescale_sites(Program& P, int k) {
  auto fix = [k](QParams& q) {
    const int e = (q.is_signed ? 7 : 8) - k;
    q.c1 = std::ldexp(1.0f, e);
    q.c2 = std::ldexp(1.0f, -e);
  };
  for (auto& v : P.values) fix(v.q);
  for (auto& g : P.groups) {
    fix(g.data.q);
    fix(g.weight.q);
    for (auto& e : g.epi) fix(e.q);
  }
}

bool is_pow2(float v) {
  if (!(v > 0.f) || !std::isfinite(v)) return false;
  int e;
  float m = std::frexp(v, &e);
  return m == 0.5f;
}

// A physical representation of one @main-level value.
struct Rep {
  int fmt = FMT_F32;
  bool nchw_user = false;  // the caller's input buffer
  bool has_q = false;      // I8: codes of Q(v)
  QParams q;
  int64_t elems = 0;       // including the zero border and chunk padding
  Lay lay{};               // P16 (4-D) or row-major (2-D)
  int buf = -1;            // arena buffer id
  // stride-2 decimated int8 codes (pixel (2i, 2j) at (i, j)): written by the
  // producer next to its side codes, read as A2 by a conv with a fused shortcut
  bool dec = false;
};

struct Buffer {
  int64_t bytes = 0;
  int first = 0, last = 0;  // launch indices
  int64_t offset = -1;
  std::string what;
  // zero border forever: its producer writes only interior pixels, so the
  // buffer gets arena space of its own (never aliased) zeroed once at build
  bool zero_border = false;
  // no launch reads it (e.g. the float32 output of a stage's last residual
  // block, whose consumers all take the producer's int8 side codes): the
  // producer skips the stores and the arena gives it no space
  bool dead = false;
};

struct LaunchRec {
  std::string name;   // group / conversion
  std::string kernel;
  int kernels = 1;    // device kernels this record launches
  double bytes = 0;   // algorithmic HBM bytes
  double flops = 0;   // algorithmic ops (2 per MAC)
  int opt_primary = -1;  // a primary output buffer the kernel can skip (tcgen05 conv with a side output)
  std::function<void(cudaStream_t)> fn;
};

}  // namespace

struct Exec {
  mr_exec_options opt{};
  Program P;
  std::vector<std::vector<Rep>> reps;  // per value
  std::vector<Buffer> bufs;
  std::vector<LaunchRec> launches;
  char* arena = nullptr;
  int64_t arena_bytes = 0;
  cudaStream_t side_stream = nullptr;
  // weights
  std::vector<void*> param_dev;             // raw float32 per @main param (nullptr for data)
  std::vector<void*> group_w;               // hoisted weight per group
  std::vector<std::vector<void*>> group_vecs;  // uploaded constant vectors per group
  std::vector<int> group_kp;                // weight row length per group
  std::vector<int> group_cs;                // weight channel stride per tap (row layouts)
  std::vector<int> group_path;              // kernel choice
  std::vector<std::string> group_exact;     // int8 exactness proof per group
  std::vector<std::string> group_note;      // kernel plan description
  std::vector<TcConvSpec> group_tc;         // tcgen05 formulation per conv group
  std::map<int, int> want_kb;               // value -> chunk width its tcgen05 consumers read
  std::set<int> f32_wide;                   // float32 values read only by depthwise convs: 128-byte chunks
  std::vector<int> fused_pool;              // conv group -> its max_pool2d consumer executed in-kernel, or -1
  std::vector<char> fused_away;             // group executed inside another group's launch
  std::vector<int> sc_of;                   // 3x3 conv -> the 1x1/stride-2 shortcut group fused into it (-1)
  bool weights_ready = false;
  int64_t zero_bytes = 0;  // arena prefix of the zero-border buffers
  // io
  std::vector<const float*> cur_inputs;  // one per data input (@main params 0 .. n_data_inputs-1)
  float* out_internal = nullptr;  // result buffer (NCHW float32)
  int out_alias_buf = -1;         // >= 0: out_internal is this arena buffer (row-major fp32 result)
  float* out_redirect = nullptr;  // mr_exec_run: the final launch writes the caller's buffer
  bool enforce_exact = true;      // int8 groups must prove the 2^24 bound (off for calibration trials)
  int64_t out_elems = 0;
  std::vector<int64_t> out_shape;
  // captured launch lists, one per input buffer address (the input pointer is
  // baked into the graph): the caller's buffer and the two pipeline stages
  struct GraphEnt {
    std::vector<const float*> in;
    float* out;
    cudaGraph_t g;
    cudaGraphExec_t e;
  };
  std::vector<GraphEnt> graphs;
  // asynchronous host pipeline (mr_exec_submit_host): double-buffered input
  // stages filled on copy_stream while the previous batch computes
  cudaStream_t copy_stream = nullptr;
  float* stage[2] = {nullptr, nullptr};
  cudaEvent_t loaded[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr}, fresh = nullptr;
  int64_t submitted = 0;
  bool pipe_fresh = true;
  cudaStream_t pipe_stream = nullptr;
  float* host_stage_in = nullptr;
  float* host_stage_out = nullptr;
  std::vector<float*> dev_in;    // mr_exec_run_host staging, one per data input
  std::vector<int64_t> in_elems;
  std::string describe;
  std::vector<TcConvPlan*> tc_plans;
  std::vector<DenseTcPlan*> group_dense;    // tcgen05 dense plan per group (nullptr: none)
  std::map<int, int> sum_operand;            // dense group -> operand buffer its producer's sum_hw writes

  void drop_graphs() {
    for (auto& g : graphs) {
      cudaGraphExecDestroy(g.e);
      cudaGraphDestroy(g.g);
    }
    graphs.clear();
  }

  ~Exec() {
    drop_graphs();
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
    }
    for (int i = 0; i < 2; ++i) {
      if (stage[i]) cudaFree(stage[i]);
      if (loaded[i]) cudaEventDestroy(loaded[i]);
      if (consumed[i]) cudaEventDestroy(consumed[i]);
    }
    if (fresh) cudaEventDestroy(fresh);
    for (auto* p : tc_plans) tc_conv_destroy(p);
    for (auto* p : group_dense) if (p) dense_tc_destroy(p);
    if (arena) cudaFree(arena);
    for (void* p : param_dev) if (p) cudaFree(p);
    for (void* p : group_w) if (p) cudaFree(p);
    for (auto& v : group_vecs) for (void* p : v) if (p) cudaFree(p);
    if (out_internal && out_alias_buf < 0) cudaFree(out_internal);
    for (float* p : dev_in)
      if (p) cudaFree(p);
    if (host_stage_in) cudaFreeHost(host_stage_in);
    if (host_stage_out) cudaFreeHost(host_stage_out);
  }

  void* ptr(int buf) const {
    if (buf == out_alias_buf && out_redirect) return out_redirect;
    return arena + bufs[buf].offset;
  }
  float* out_dst() const { return out_redirect ? out_redirect : out_internal; }
};

// Makes `dev` current for one API call and restores the caller's device: an
// executor can be driven from any host thread whatever its current device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) {
      cudaError_t e = cudaSetDevice(dev);
      if (e != cudaSuccess) throw Status{MR_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)};
    } else {
      prev = -1;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

namespace {

enum Path { P_NONE = 0, P_CONV_I8_SIMT, P_CONV_I8_TC, P_CONV_BF16_SIMT, P_CONV_BF16_TC, P_CONV_F32, P_DENSE_I8,
            P_DENSE_F32, P_DENSE_BF16, P_POOL, P_DW, P_DENSE_I8_TC, P_DENSE_BF16_TC, P_CONV_TF32_TC,
            P_DENSE_TF32_TC };

const char* path_name(int p) {
  static const char* n[] = {"none", "conv_i8_simt", "conv_i8_tcgen05", "conv_bf16_simt", "conv_bf16_tcgen05",
                            "conv_f32_strict", "dense_i8", "dense_f32_strict", "dense_bf16", "max_pool", "dwconv",
                            "dense_i8_tcgen05", "dense_bf16_tcgen05", "conv_tf32_tcgen05", "dense_tf32_tcgen05"};
  return n[p];
}


int float_fmt(const Exec& ex) {
  // int8 pipelines keep the float residual stream exact in float32; the
  // strict mode computes everything in float32; bf16 mode stores bf16.
  if (ex.P.any_quant || ex.opt.float_mode == MR_FLOAT_FP32_STRICT || ex.opt.float_mode == MR_FLOAT_TF32) return FMT_F32;
  return FMT_BF16;
}

int64_t elem_bytes(int fmt) { return fmt == FMT_F32 ? 4 : fmt == FMT_BF16 ? 2 : 1; }

// Layout of a representation: P16 (NORMAL / PHASE / S2D) with a kPad
// border for 4-D values, row-major for 2-D ones.  Plane strides are padded to
// 8 pixels (128-byte TMA rows).  S2D takes the stem's input padding.
Lay make_lay(const std::vector<int64_t>& s, int fmt, int kind, int s2d_pad = 0, int kb = 16) {
  Lay L{};
  L.C = s.size() >= 2 ? static_cast<int32_t>(s[1]) : 1;
  L.kind = LAY_NORMAL;
  L.kb = kb;
  if (s.size() == 4) {
    L.cpc = static_cast<int32_t>(kb / elem_bytes(fmt));
    L.kind = kind;
    L.Hp = static_cast<int32_t>(s[2] + 2 * kPad);
    L.Wp = static_cast<int32_t>(s[3] + 2 * kPad);
    if (kind == LAY_NORMAL) {
      L.Pp = round_up(s[0] * L.Hp * L.Wp, 8);
    } else if (kind == LAY_PHASE) {
      L.Hq = (L.Hp + 1) / 2;
      L.Wq = (L.Wp + 1) / 2;
      L.Pp = round_up(s[0] * L.Hq * L.Wq, 8);
    } else if (kind == LAY_S2D) {  // 4*C s2d channels on a ceil((H+2p)/2) grid
      L.C = static_cast<int32_t>(4 * s[1]);
      // float32 (the tf32 stem): an even number of 16-byte planes -- one
      // kind::tf32 K step spans two; the extra channels are zeros
      if (fmt == FMT_F32) L.C = static_cast<int32_t>(round_up(L.C, 2 * L.cpc));
      L.Hq = static_cast<int32_t>((s[2] + 2 * s2d_pad + 1) / 2);
      L.Wq = static_cast<int32_t>((s[3] + 2 * s2d_pad + 1) / 2);
      L.Pp = round_up(s[0] * L.Hq * L.Wq, 8);
    } else {  // LAY_S2DP: the s2d grid shifted by 2, split into 4 phase sub-grids
      L.C = static_cast<int32_t>(4 * s[1]);
      const int32_t hs = static_cast<int32_t>((s[2] + 2 * s2d_pad + 1) / 2);
      const int32_t ws = static_cast<int32_t>((s[3] + 2 * s2d_pad + 1) / 2);
      L.Hq = (hs + 3) / 2 + 1;
      L.Wq = (ws + 3) / 2 + 1;
      L.Pp = round_up(s[0] * L.Hq * L.Wq, 8);
    }
  } else {
    L.cpc = 0;
    L.Pp = s.empty() ? 1 : s[0];
  }
  return L;
}

int64_t lay_elems(const Lay& L) {
  if (L.cpc == 0) return L.Pp * L.C;
  int64_t planes = (L.C + L.cpc - 1) / L.cpc;
  return planes * (L.kind == LAY_PHASE || L.kind == LAY_S2DP ? 4 : 1) * L.Pp * L.cpc;
}


// Finds or adds a representation of value v.  kb 0 = any chunk width (the
// value's preferred one when creating).
int want_rep(Exec& ex, int v, int fmt, const QParams* q, int kind = LAY_NORMAL, int s2d_pad = 0, int kb = 0) {
  auto& rs = ex.reps[v];
  if (ex.P.values[v].shape.size() != 4) kind = LAY_NORMAL;
  // float32 values are P16 (16-byte chunks: warp-coalesced residual loads),
  // except in the tf32 mode, where tcgen05 convs read them in 128-byte chunks
  // and every consumer shares that one representation
  const bool tf32 = ex.opt.float_mode == MR_FLOAT_TF32 && !ex.P.any_quant;
  if ((fmt == FMT_F32 && !tf32 && !ex.f32_wide.count(v)) || kind == LAY_S2D || kind == LAY_S2DP) kb = 16;
  for (size_t i = 0; i < rs.size(); ++i) {
    const Rep& r = rs[i];
    if (r.nchw_user) continue;
    if (r.fmt != fmt || r.lay.kind != kind) continue;
    if (kb && r.lay.kb != kb) continue;
    if (fmt == FMT_I8) {
      if (!q || !r.has_q || !(r.q == *q)) continue;
    }
    return static_cast<int>(i);
  }
  Rep r;
  r.fmt = fmt;
  if (q) {
    r.has_q = true;
    r.q = *q;
  }
  if (!kb) {
    auto it = ex.want_kb.find(v);
    kb = it != ex.want_kb.end() ? it->second : 16;
  }
  r.lay = make_lay(ex.P.values[v].shape, fmt, kind, s2d_pad, kb);
  r.elems = lay_elems(r.lay);
  rs.push_back(r);
  return static_cast<int>(rs.size()) - 1;
}

// tcgen05 formulation per conv group, decided at compile time from the
// geometry: stride-1 halo (3x3/1x1), stride-2 over phase-split inputs, or
// the space-to-depth stem; anything else runs on the CUDA-core kernel.
// A tail op after the element epilogue (sum over HW or flatten): the anchor
// kernel writes the float32 pre-tail tensor, a second launch finishes it.
bool g_has_sum(const GroupDesc& g) {
  if (g.epi.empty()) return false;
  for (const auto& e : g.epi)
    if (e.kind == EpiKind::Flatten) return true;
  return g.epi.back().kind == EpiKind::SumHW;
}

void decide_tc(Exec& ex) {
  Program& P = ex.P;
  std::map<int, int> phase_kb;
  ex.fused_pool.assign(P.groups.size(), -1);
  ex.fused_away.assign(P.groups.size(), 0);
  ex.group_tc.assign(P.groups.size(), TcConvSpec{});
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    int& path = ex.group_path[gi];
    const GroupDesc& g = P.groups[gi];
    if (path != P_CONV_I8_TC && path != P_CONV_BF16_TC && path != P_CONV_TF32_TC) continue;
    bool has_sum = g_has_sum(g);
    const auto& os = has_sum ? g.pre_sum_shape : g.out_shape;
    TcConvSpec sp{};
    sp.elem_bytes = path == P_CONV_I8_TC ? 1 : path == P_CONV_TF32_TC ? 4 : 2;
    sp.N = static_cast<int>(g.in_shape[0]);
    sp.C = static_cast<int>(g.in_shape[1]);
    sp.H = static_cast<int>(g.in_shape[2]);
    sp.W = static_cast<int>(g.in_shape[3]);
    sp.OC = static_cast<int>(os[1]);
    sp.OH = static_cast<int>(os[2]);
    sp.OW = static_cast<int>(os[3]);
    sp.KH = static_cast<int>(g.kh);
    sp.KW = static_cast<int>(g.kw);
    bool same3 = g.kh == 3 && g.kw == 3 && g.ph == 1 && g.pw == 1;
    bool one = g.kh == 1 && g.kw == 1 && g.ph == 0 && g.pw == 0;
    bool ok = false;
    if (g.sh == 1 && g.sw == 1 && (same3 || one)) {
      sp.kind = TC_S1;
      ok = tc_conv_plan_ok(sp);
    } else if (g.sh == 2 && g.sw == 2 && (same3 || one)) {
      sp.kind = TC_S2_PHASE;
      auto pk = phase_kb.find(g.data.value);  // one phase-split copy per value
      if (pk != phase_kb.end()) sp.kb = pk->second;
      ok = tc_conv_plan_ok(sp);
    }
    if (!ok && g.sh == 2 && g.sw == 2 && g.kh == g.kw && (g.kh & 1) && g.ph == g.kh / 2 && g.pw == g.kw / 2 &&
        P.values[g.data.value].is_data) {
      // a stride-2 stem over the network input (e.g. 3x3/s2 on 3 channels, which
      // fills no chunk for the phase formulation): space-to-depth
      TcConvSpec s2 = sp;
      s2.kind = TC_STEM_S2D;
      s2.kb = 0;
      s2.Hs = static_cast<int>((sp.H + 2 * g.ph + 1) / 2);
      s2.Ws = static_cast<int>((sp.W + 2 * g.pw + 1) / 2);
      if (tc_conv_plan_ok(s2)) {
        sp = s2;
        ok = true;
      }
    }
    if (ok && sp.kind == TC_STEM_S2D) {
      // cross-group fusion: conv -> max_pool2d when the
      // pool is the conv output's only consumer; same arithmetic, the conv
      // tensor never reaches HBM
      const ValueInfo& ov = P.values[g.out_value];
      bool epi_ok = true;
      for (const auto& op : g.epi) epi_ok = epi_ok && (op.kind == EpiKind::Bias || op.kind == EpiKind::Relu);
      if (ov.consumers.size() == 1 && !ov.is_result && epi_ok && !ov.quantized) {
        const int pj = ov.consumers[0];
        const GroupDesc& pg = P.groups[pj];
        if (pg.kind == GroupKind::MaxPool && pg.data.value == g.out_value && ex.group_path[pj] == P_POOL) {
          TcConvSpec fs = sp;
          fs.pool = 1;
          fs.pkh = static_cast<int>(pg.kh);
          fs.pkw = static_cast<int>(pg.kw);
          fs.psh = static_cast<int>(pg.sh);
          fs.psw = static_cast<int>(pg.sw);
          fs.pph = static_cast<int>(pg.ph);
          fs.ppw = static_cast<int>(pg.pw);
          fs.poh = static_cast<int>(pg.out_shape[2]);
          fs.pow = static_cast<int>(pg.out_shape[3]);
          // int8, 3-channel 7x7/s2/p3 stem + 3x3/s2/p1 pool: the pool window
          // is part of the GEMM's M (TC_STEM_POOL); otherwise staged pooling
          TcConvSpec wp = fs;
          wp.kind = TC_STEM_POOL;
          const bool win_ok = sp.C == 3 && g.ph == 3 && tc_conv_plan_ok(wp);
          if (win_ok || tc_conv_plan_ok(fs)) {
            sp = win_ok ? wp : fs;
            ex.fused_pool[gi] = pj;
            ex.fused_away[pj] = 1;
          }
        }
      }
    }
    if (ok) {
      ex.group_tc[gi] = sp;
      if (sp.kind == TC_S1) ex.want_kb[g.data.value] = sp.kb;
      if (sp.kind == TC_S2_PHASE) phase_kb[g.data.value] = sp.kb;
    } else {
      path = path == P_CONV_I8_TC ? P_CONV_I8_SIMT : path == P_CONV_TF32_TC ? P_CONV_F32 : P_CONV_BF16_SIMT;
    }
  }
}

void plan(Exec& ex, bool use_tc) {
  Program& P = ex.P;
  const int ffmt = float_fmt(ex);
  ex.reps.assign(P.values.size(), {});
  ex.group_path.assign(P.groups.size(), P_NONE);
  ex.group_exact.assign(P.groups.size(), "");

  // kernel path per group
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    const GroupDesc& g = P.groups[gi];
    switch (g.kind) {
      case GroupKind::Conv:
        if (g.weight.quant) {
          ex.group_path[gi] = use_tc ? P_CONV_I8_TC : P_CONV_I8_SIMT;
        } else if (ex.opt.float_mode == MR_FLOAT_TF32 && !P.any_quant) {
          ex.group_path[gi] = use_tc ? P_CONV_TF32_TC : P_CONV_F32;
        } else if (ffmt == FMT_F32) {
          ex.group_path[gi] = P_CONV_F32;
        } else {
          ex.group_path[gi] = use_tc ? P_CONV_BF16_TC : P_CONV_BF16_SIMT;
        }
        break;
      case GroupKind::Dense:
      {
        static const bool no_dense_tc = [] {  // A/B switch: the CUDA-core dense
          const char* e = std::getenv("MRB200_NO_DENSE_TC");
          return e && std::atoi(e);
        }();
        const bool tc = use_tc && !no_dense_tc;
        const bool tf32 = ex.opt.float_mode == MR_FLOAT_TF32 && !P.any_quant;
        ex.group_path[gi] = g.weight.quant ? (tc ? P_DENSE_I8_TC : P_DENSE_I8)
                            : tf32 ? (tc ? P_DENSE_TF32_TC : P_DENSE_F32)
                            : ffmt == FMT_F32 ? P_DENSE_F32 : (tc ? P_DENSE_BF16_TC : P_DENSE_BF16);
      }
        break;
      case GroupKind::MaxPool: ex.group_path[gi] = P_POOL; break;
      case GroupKind::DwConv: ex.group_path[gi] = P_DW; break;
    }
  }
  decide_tc(ex);
  // bf16 depthwise inputs in 128-byte chunks (64 channels per plane): a pixel's
  // channels are one contiguous 128-byte row, so 16 lanes of k_dw3x3_rb read
  // (and the producing conv writes) whole lines instead of 16-byte pieces
  static const bool dw_wide = [] {
    const char* e = std::getenv("MRB200_DW_PL16");
    return !e || std::atoi(e) != 0;
  }();
  for (size_t gi = 0; gi < P.groups.size() && dw_wide; ++gi) {
    const GroupDesc& g = P.groups[gi];
    // (float32 inputs -- the int8 modules' float path -- likewise: 32 channels per
    // 128-byte row, 8 lanes per pixel, and the int8 codes written as whole sectors)
    const bool f32_in = ffmt == FMT_F32 && g.in_shape[1] % 32 == 0 && P.any_quant;
    if (g.kind != GroupKind::DwConv || (!f32_in && (ffmt != FMT_BF16 || g.in_shape[1] % 64 != 0)) || g.kh != 3 ||
        g.kw != 3)
      continue;
    const ValueInfo& dv = P.values[g.data.value];
    bool only_dw = !dv.is_data;
    for (int c : dv.consumers) only_dw = only_dw && P.groups[c].kind == GroupKind::DwConv;
    if (only_dw && !ex.want_kb.count(g.data.value)) {
      ex.want_kb[g.data.value] = 128;
      if (f32_in) ex.f32_wide.insert(g.data.value);
    }
  }
  // primary representations of group outputs (chunk width from want_kb)
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    const GroupDesc& g = P.groups[gi];
    const ValueInfo& ov = P.values[g.out_value];
    bool flat = false;
    for (const auto& e : g.epi) flat = flat || e.kind == EpiKind::Flatten;
    if (flat || (ov.quantized && ov.shape.size() == 2)) {
      // the flatten tail / a dense epilogue writes row-major float32; a trailing
      // realize chain leaves code * c2 there, the reference's exact value, and a
      // dense consumer re-quantizes it exactly (GroupIO::requant_data)
      want_rep(ex, g.out_value, FMT_F32, nullptr);
    } else if (ov.quantized) {
      want_rep(ex, g.out_value, FMT_I8, &ov.q);
    } else if (g.kind == GroupKind::Dense || ov.shape.size() == 2) {
      want_rep(ex, g.out_value, FMT_F32, nullptr);
    } else {
      want_rep(ex, g.out_value, ov.is_result ? FMT_F32 : ffmt, nullptr);
    }
  }
  // @main data inputs: the caller's NCHW float32 buffer
  for (size_t v = 0; v < P.values.size(); ++v) {
    if (!P.values[v].is_data) continue;
    Rep r;
    r.nchw_user = true;
    r.fmt = FMT_F32;
    ex.reps[v].push_back(r);
  }
}

}  // namespace

// Representation index a group reads for its data operand / residual.
struct GroupIO {
  int data_rep = -1;
  std::vector<int> res_rep;  // per epi op (Residual only)
  float data_scale = 1.f;    // c2 of the data codes (int8)
  // dense over a realized (coded) value: the float rep holds code * c2 exactly;
  // the prologue re-quantizes with the same chain (c1 * c2 == 1: the codes come back exactly)
  bool requant_data = false;
  QParams requant_q;
  int sc_rep = -1;  // fused shortcut: the decimated codes rep of the block input (Exec::sc_of)
};

namespace {

GroupIO resolve_inputs(Exec& ex, int gi) {
  const Program& P = ex.P;
  const GroupDesc& g = P.groups[gi];
  GroupIO io;
  const int ffmt = float_fmt(ex);
  const ValueInfo& dv = P.values[g.data.value];
  int path = ex.group_path[gi];
  // data layout kind the tcgen05 formulation needs (CUDA-core kernels read NORMAL)
  int kind = LAY_NORMAL, s2d_pad = 0, kb = 0;
  if (path == P_CONV_I8_TC || path == P_CONV_BF16_TC || path == P_CONV_TF32_TC) {
    const TcConvSpec& sp = ex.group_tc[gi];
    kind = sp.kind == TC_S2_PHASE ? LAY_PHASE : sp.kind == TC_STEM_S2D ? LAY_S2D : sp.kind == TC_STEM_POOL ? LAY_S2DP : LAY_NORMAL;
    s2d_pad = static_cast<int>(g.ph);
    kb = sp.kb;
  }
  if (path == P_CONV_I8_SIMT || path == P_CONV_I8_TC) {
    if (g.data.quant) {
      io.data_rep = want_rep(ex, g.data.value, FMT_I8, &g.data.q, kind, s2d_pad, kb);
      io.data_scale = g.data.q.c2;
    } else {
      io.data_rep = want_rep(ex, g.data.value, FMT_I8, &dv.q, kind, s2d_pad, kb);
      io.data_scale = dv.q.c2;
    }
  } else if (g.kind == GroupKind::Dense) {
    if (dv.shape.size() != 2) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": dense over a 4-D value");
    io.data_rep = want_rep(ex, g.data.value, FMT_F32, nullptr);
    if (g.data.quant) {
      io.data_scale = g.data.q.c2;
    } else if (dv.quantized) {
      if (!(dv.q.c1 * dv.q.c2 == 1.f)) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": dense over a coded value");
      io.requant_data = true;
      io.requant_q = dv.q;
      io.data_scale = dv.q.c2;
    }
  } else if (path == P_CONV_F32 || path == P_CONV_BF16_SIMT || path == P_CONV_BF16_TC || path == P_CONV_TF32_TC) {
    if (g.data.pre_mul != 0.f) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": scaled conv input");
    io.data_rep = want_rep(ex, g.data.value, ffmt, nullptr, kind, s2d_pad, kb);
  } else {  // pool / depthwise: float input
    io.data_rep = want_rep(ex, g.data.value, ffmt, nullptr);
  }
  io.res_rep.assign(g.epi.size(), -1);
  for (size_t i = 0; i < g.epi.size(); ++i)
    if (g.epi[i].kind == EpiKind::Residual)  // 2-D values (dense outputs) stay row-major float32
      io.res_rep[i] = want_rep(ex, g.epi[i].value, P.values[g.epi[i].value].shape.size() == 2 ? FMT_F32 : ffmt, nullptr);
  return io;
}

}  // namespace

}  // namespace mrb200

// ======================================================================
// The executor build: reps -> buffers -> launches
// ======================================================================
namespace mrb200 {
namespace {


struct Builder {
  Exec& ex;
  std::vector<GroupIO> io;
  // (value, rep) -> buffer
  std::map<std::pair<int, int>, int> buf_of;
  int launch_idx = 0;

  int buffer_for(int v, int r, const std::string& what) {
    auto key = std::make_pair(v, r);
    auto it = buf_of.find(key);
    if (it != buf_of.end()) return it->second;
    Buffer b;
    const Rep& rep = ex.reps[v][r];
    b.bytes = rep.elems * elem_bytes(rep.fmt);
    b.first = b.last = launch_idx;
    b.what = what;
    ex.bufs.push_back(b);
    int id = static_cast<int>(ex.bufs.size()) - 1;
    buf_of[key] = id;
    ex.reps[v][r].buf = id;
    return id;
  }
  void use(int buf) {
    ex.bufs[buf].last = std::max(ex.bufs[buf].last, launch_idx);
    ex.bufs[buf].first = std::min(ex.bufs[buf].first, launch_idx);
  }
  int scratch(int64_t bytes, const std::string& what) {
    Buffer b;
    b.bytes = bytes;
    b.first = b.last = launch_idx;
    b.what = what;
    ex.bufs.push_back(b);
    return static_cast<int>(ex.bufs.size()) - 1;
  }
};

void assign_offsets(Exec& ex) {
  // dedicated, never-aliased region for the zero-border buffers (zeroed once)
  int64_t base = 0;
  for (Buffer& b : ex.bufs)
    if (b.zero_border) {
      b.offset = base;
      base += round_up(std::max<int64_t>(b.bytes, 1), 256);
    }
  ex.zero_bytes = base;
  std::vector<int> order;
  for (size_t i = 0; i < ex.bufs.size(); ++i)
    if (!ex.bufs[i].zero_border) order.push_back(static_cast<int>(i));
  std::sort(order.begin(), order.end(), [&](int a, int b) { return ex.bufs[a].bytes > ex.bufs[b].bytes; });
  std::vector<int> placed;
  int64_t top = base;
  for (int id : order) {
    Buffer& b = ex.bufs[id];
    int64_t size = round_up(std::max<int64_t>(b.bytes, 1), 256);
    // candidate offsets: 0 and the end of every overlapping placed buffer
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (int o : placed) {
      const Buffer& q = ex.bufs[o];
      if (q.last < b.first || q.first > b.last) continue;
      busy.emplace_back(q.offset, q.offset + round_up(std::max<int64_t>(q.bytes, 1), 256));
    }
    std::sort(busy.begin(), busy.end());
    int64_t off = base;
    for (auto& [s, e] : busy) {
      if (off + size <= s) break;
      off = std::max(off, e);
    }
    b.offset = off;
    top = std::max(top, off + size);
    placed.push_back(id);
  }
  ex.arena_bytes = top;
}

EpiDev make_epi(Exec& ex, int gi, const GroupIO& io, int upto) {
  const GroupDesc& g = ex.P.groups[gi];
  EpiDev e{};
  int n = 0;
  for (int i = 0; i < upto; ++i) {
    const EpiOp& op = g.epi[i];
    if (n >= kMaxEpi) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": epilogue longer than 8 ops");
    switch (op.kind) {
      case EpiKind::MulScalar: e.op[n] = E_MULS; e.s[n] = op.s; break;
      case EpiKind::MulChannel: e.op[n] = E_MULC; e.vec[n] = nullptr; break;  // patched in set_weights
      case EpiKind::Bias: e.op[n] = E_BIAS; e.vec[n] = nullptr; break;        // patched in set_weights
      case EpiKind::Residual: {
        e.op[n] = E_RES;
        e.res[n] = nullptr;  // arena address patched at launch (residual_fix)
        // (res_rep -1: a fused shortcut computes it in-kernel from its own accumulator)
        e.res_fmt[n] = io.res_rep[i] >= 0 ? ex.reps[op.value][io.res_rep[i]].fmt : FMT_F32;
        break;
      }
      case EpiKind::Relu: e.op[n] = E_RELU; break;
      case EpiKind::Requant: e.op[n] = E_REQ; e.q[n] = to_qdev(op.q); break;
      case EpiKind::Clip: e.op[n] = E_CLIP; e.s[n] = op.lo; e.s2[n] = op.hi; break;
      case EpiKind::SumHW:
      case EpiKind::Flatten: fail(MR_ERR_INTERNAL, "tail op inside the element epilogue");
    }
    ++n;
  }
  e.n_ops = n;
  return e;
}

std::string dims_str(const std::vector<int64_t>& s) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < s.size(); ++i) os << (i ? "," : "") << s[i];
  os << "]";
  return os.str();
}

}  // namespace

// Cross-group fusion of a ResNet downsampling block's shortcut: a 1x1/stride-2
// conv group whose only consumer is the residual add of a 3x3 stride-1 conv
// group (bias -> add -> relu) runs inside that conv's launch (TcConvSpec::sc_C).
// Its input -- the block input's int8 codes -- comes from a decimated copy the
// block input's producer writes next to its side codes; the float32 shortcut
// output (written and read back in full otherwise) disappears.  The arithmetic
// is the shortcut group's own: acc2 * (data c2 * weight c2) + bias, then the
// reference's add.  MRB200_NO_SHORTCUT_FUSE=1 keeps the groups apart (A/B).
void fuse_shortcuts(Exec& ex, std::vector<GroupIO>& io) {
  Program& P = ex.P;
  ex.sc_of.assign(P.groups.size(), -1);
  static const bool off = [] {
    const char* e = std::getenv("MRB200_NO_SHORTCUT_FUSE");
    return e && std::atoi(e);
  }();
  if (off) return;
  for (size_t gm = 0; gm < P.groups.size(); ++gm) {
    const GroupDesc& m = P.groups[gm];
    const int path = ex.group_path[gm];
    if ((path != P_CONV_I8_TC && path != P_CONV_BF16_TC) || ex.fused_away[gm] || ex.group_tc[gm].kind != TC_S1 || m.kh != 3 ||
        m.kw != 3 || ex.fused_pool[gm] >= 0 || g_has_sum(m))
      continue;
    if (m.epi.size() != 3 || m.epi[0].kind != EpiKind::Bias || m.epi[1].kind != EpiKind::Residual ||
        m.epi[2].kind != EpiKind::Relu)
      continue;
    const int vs = m.epi[1].value;
    const ValueInfo& sv = P.values[vs];
    const int gs = sv.producer;
    if (gs < 0 || sv.is_result || sv.consumers.size() != 1 || sv.consumers[0] != static_cast<int>(gm)) continue;
    const GroupDesc& sg = P.groups[gs];
    if (sg.kind != GroupKind::Conv || ex.group_path[gs] != path || ex.fused_away[gs] || ex.fused_pool[gs] >= 0 ||
        ex.group_tc[gs].kind != TC_S2_PHASE || sg.kh != 1 || sg.kw != 1 || sg.sh != 2 || sg.sw != 2 || sg.ph != 0 ||
        sg.pw != 0 || sg.epi.size() != 1 || sg.epi[0].kind != EpiKind::Bias || sg.out_shape != m.out_shape)
      continue;
    // the block input's codes are its producer's side output (a tcgen05 conv over the padded grid)
    const int vu = sg.data.value;
    const ValueInfo& uv = P.values[vu];
    const int gp = uv.producer;
    const int dr = io[gs].data_rep;
    const int dfmt = path == P_CONV_I8_TC ? FMT_I8 : FMT_BF16;
    if (gp < 0 || uv.is_data || dr <= 0 || ex.reps[vu][dr].fmt != dfmt || ex.group_path[gp] != path ||
        ex.group_tc[gp].kind != TC_S1 || ex.fused_pool[gp] >= 0 || g_has_sum(P.groups[gp]))
      continue;
    bool has_dec = false;  // one decimated copy per value
    for (const Rep& r : ex.reps[vu]) has_dec = has_dec || r.dec;
    if (has_dec) continue;
    TcConvSpec spec = ex.group_tc[gm];
    spec.sc_C = static_cast<int>(sg.in_shape[1]);
    spec.sc_kb = ex.group_tc[gs].kb;
    if (!tc_conv_plan_ok(spec)) continue;
    ex.group_tc[gm] = spec;
    ex.sc_of[gm] = gs;
    ex.fused_away[gs] = 1;
    Rep r;
    r.fmt = dfmt;
    r.has_q = ex.reps[vu][dr].has_q;
    r.q = ex.reps[vu][dr].q;
    r.dec = true;
    r.lay = make_lay({sg.out_shape[0], sg.in_shape[1], sg.out_shape[2], sg.out_shape[3]}, dfmt, LAY_NORMAL, 0,
                     spec.sc_kb);
    r.elems = lay_elems(r.lay);
    ex.reps[vu].push_back(r);
    io[gm].sc_rep = static_cast<int>(ex.reps[vu].size()) - 1;
    io[gm].res_rep[1] = -1;
  }
}

void build(Exec& ex) {
  Program& P = ex.P;
  const bool use_tc = !ex.opt.force_simt;
  plan(ex, use_tc);
  std::vector<GroupIO> io(P.groups.size());
  for (size_t gi = 0; gi < P.groups.size(); ++gi) io[gi] = resolve_inputs(ex, static_cast<int>(gi));

  // int8 exactness precondition: operand scales must be powers of two.
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    int path = ex.group_path[gi];
    if (path == P_CONV_I8_SIMT || path == P_CONV_I8_TC || path == P_DENSE_I8 || path == P_DENSE_I8_TC) {
      float sw = P.groups[gi].weight.q.c2;
      if (!is_pow2(io[gi].data_scale) || !is_pow2(sw))
        fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + P.groups[gi].name + ": quantize scales are not powers of two");
    }
  }

  fuse_shortcuts(ex, io);

  Builder B{ex, io};
  // Producer side outputs: every I8 rep of a float value not produced by a
  // Requant must come from the producer kernel's side output (or an input
  // conversion for @main data).
  std::vector<int> side_rep(P.groups.size(), -1), side2_rep(P.groups.size(), -1);
  for (size_t v = 0; v < P.values.size(); ++v) {
    const ValueInfo& vi = P.values[v];
    for (size_t r = 0; r < ex.reps[v].size(); ++r) {
      const Rep& rep = ex.reps[v][r];
      if (rep.nchw_user || r == 0 || vi.producer < 0) continue;  // rep 0 is the primary
      if (rep.dec) {
        side2_rep[vi.producer] = static_cast<int>(r);
        continue;
      }
      const bool tf32_side = rep.fmt == FMT_F32 && ex.opt.float_mode == MR_FLOAT_TF32 && !P.any_quant;
      if ((rep.fmt == FMT_I8 || rep.fmt == FMT_BF16 || tf32_side) && P.groups[vi.producer].kind != GroupKind::Dense &&
          !g_has_sum(P.groups[vi.producer])) {
        if (side_rep[vi.producer] >= 0)
          fail(MR_ERR_UNSUPPORTED_GROUP, "value %" + vi.name + " needs more than two representations");
        side_rep[vi.producer] = static_cast<int>(r);
      } else {
        fail(MR_ERR_UNSUPPORTED_GROUP, "value %" + vi.name + " needs a representation its producer cannot emit");
      }
    }
  }

  // ---- input conversions (@main data params -> consumer formats) ----
  for (size_t v = 0; v < P.values.size(); ++v) {
    const ValueInfo& vi = P.values[v];
    if (!vi.is_data) continue;
    if (vi.shape.size() != 4 && vi.shape.size() != 2)
      fail(MR_ERR_UNSUPPORTED_GROUP, "data input %" + vi.name + " must be NCHW or [N, K]");
    for (size_t r = 0; r < ex.reps[v].size(); ++r) {
      const Rep rep = ex.reps[v][r];
      if (rep.nchw_user) continue;
      if (vi.shape.size() == 2) {  // row-major [N, K]: the caller's layout already; copy it in
        if (rep.fmt != FMT_F32 || rep.lay.cpc != 0)
          fail(MR_ERR_UNSUPPORTED_GROUP, "2-D data input %" + vi.name + " needs a float32 row-major representation");
        int buf = B.buffer_for(static_cast<int>(v), static_cast<int>(r), vi.name + ":in");
        LaunchRec L;
        L.name = "%" + vi.name;
        L.kernel = "input_copy";
        const size_t bytes = static_cast<size_t>(vi.shape[0] * vi.shape[1]) * 4;
        L.bytes = 2.0 * bytes;
        Exec* e = &ex;
        const int pidx = vi.param_index;
        L.fn = [e, buf, bytes, pidx](cudaStream_t s) {
          CK(cudaMemcpyAsync(e->ptr(buf), e->cur_inputs[pidx], bytes, cudaMemcpyDeviceToDevice, s));
        };
        ex.launches.push_back(L);
        ++B.launch_idx;
        continue;
      }
      int buf = B.buffer_for(static_cast<int>(v), static_cast<int>(r), vi.name + ":in");
      LaunchRec L;
      L.name = "%" + vi.name;
      L.kernel = "input_convert";
      int N = static_cast<int>(vi.shape[0]), C = static_cast<int>(vi.shape[1]);
      int H = static_cast<int>(vi.shape[2]), W = static_cast<int>(vi.shape[3]);
      L.bytes = 4.0 * N * C * H * W + static_cast<double>(rep.elems) * elem_bytes(rep.fmt);
      QDev q = to_qdev(rep.q);
      int fmt = rep.fmt;
      Lay lay = rep.lay;
      int s2d_pad = 0;
      if (lay.kind == LAY_S2D || lay.kind == LAY_S2DP)
        for (int c : vi.consumers)
          if (P.groups[c].data.value == static_cast<int>(v)) s2d_pad = static_cast<int>(P.groups[c].ph);
      Exec* e = &ex;
      const int pidx = vi.param_index;  // data inputs are @main params 0 .. n_data_inputs-1
      L.fn = [e, buf, N, C, H, W, fmt, lay, s2d_pad, q, pidx](cudaStream_t s) {
        launch_input_convert(e->cur_inputs[pidx], N, C, H, W, e->ptr(buf), fmt, lay, s2d_pad, 0.f, q, s);
      };
      ex.launches.push_back(L);
      ++B.launch_idx;
    }
  }

  // ---- groups ----
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    if (ex.fused_away[gi]) continue;  // runs inside its producer's launch
    const GroupDesc& g = P.groups[gi];
    const GroupIO& gio = io[gi];
    const int path = ex.group_path[gi];
    const int fp = ex.fused_pool[gi];                 // fused max_pool2d consumer
    const int ov = fp >= 0 ? P.groups[fp].out_value : g.out_value;  // value this launch writes
    const int sgi = fp >= 0 ? fp : static_cast<int>(gi);            // group owning the side output
    const Rep& drep = ex.reps[g.data.value][gio.data_rep];
    if (drep.nchw_user) fail(MR_ERR_INTERNAL, "group reads the raw input");
    B.use(drep.buf);
    for (size_t i = 0; i < g.epi.size(); ++i)
      if (gio.res_rep[i] >= 0) B.use(ex.reps[g.epi[i].value][gio.res_rep[i]].buf);
    const std::string oname = fp >= 0 ? P.groups[fp].out_name : g.out_name;
    int obuf = B.buffer_for(ov, 0, "%" + oname);
    int sbuf = side_rep[sgi] >= 0 ? B.buffer_for(ov, side_rep[sgi], "%" + oname + ":codes") : -1;
    int sbuf2 = side2_rep[sgi] >= 0 ? B.buffer_for(ov, side2_rep[sgi], "%" + oname + ":codes_s2") : -1;
    if (sbuf2 >= 0) ex.bufs[sbuf2].zero_border = true;  // interior pixels only: the border stays zero
    const int sc_g = ex.sc_of[gi];
    if (sc_g >= 0) B.use(ex.reps[P.groups[sc_g].data.value][gio.sc_rep].buf);
    const Rep& orep = ex.reps[ov][0];

    bool has_sum = g_has_sum(g);
    int n_elem_ops = static_cast<int>(g.epi.size()) - (has_sum ? 1 : 0);
    int flatten_at = -1;  // reshape tail (+ the consumer's realize chain after it)
    for (size_t i = 0; i < g.epi.size(); ++i)
      if (g.epi[i].kind == EpiKind::Flatten) flatten_at = static_cast<int>(i);
    if (flatten_at >= 0) {
      has_sum = true;
      n_elem_ops = flatten_at;
    }
    EpiDev epi = make_epi(ex, static_cast<int>(gi), gio, n_elem_ops);
    OutDev out{};
    int pre_sum_buf = -1;
    Lay pre_lay{};
    if (has_sum) {
      // the conv writes the float32 pre-sum tensor (P16); k_sum_hw reduces it
      pre_lay = make_lay(g.pre_sum_shape, FMT_F32, LAY_NORMAL);
      pre_sum_buf = B.scratch(lay_elems(pre_lay) * 4, "%" + g.out_name + ":presum");
      out.primary_fmt = FMT_F32;
      out.plan = pre_lay;
    } else {
      out.primary_fmt = orep.fmt;
      out.plan = orep.lay;
    }
    // tf32 mode: 4-D float32 activations are stored tf32-rounded (consumers' MMAs read tf32)
    out.tf32 = ex.opt.float_mode == MR_FLOAT_TF32 && !P.any_quant && P.values[ov].shape.size() == 4 ? 1 : 0;
    if (sbuf >= 0) {
      const Rep& sr = ex.reps[ov][side_rep[sgi]];
      out.slay = sr.lay;
      out.side_fmt = sr.fmt;
      out.side_q = to_qdev(sr.q);
    }
    if (sbuf2 >= 0) out.s2lay = ex.reps[ov][side2_rep[sgi]].lay;

    LaunchRec L;
    L.name = "%" + g.name + (fp >= 0 ? "+%" + P.groups[fp].name : "") + (sc_g >= 0 ? "+%" + P.groups[sc_g].name : "");
    L.kernel = std::string(path_name(path)) + (fp >= 0 ? "+max_pool" : "") + (sc_g >= 0 ? "+shortcut" : "");
    // algorithmic traffic: data once + output(s) once + residuals + weights
    double out_bytes = static_cast<double>(orep.elems) * elem_bytes(orep.fmt);
    if (sbuf >= 0) {
      const Rep& sr = ex.reps[ov][side_rep[sgi]];
      out_bytes += static_cast<double>(sr.elems) * elem_bytes(sr.fmt);
    }
    if (sbuf2 >= 0) {
      const Rep& r2 = ex.reps[ov][side2_rep[sgi]];
      out_bytes += static_cast<double>(r2.elems) * elem_bytes(r2.fmt);
    }
    double in_bytes = static_cast<double>(drep.elems) * elem_bytes(drep.fmt);
    for (size_t i = 0; i < g.epi.size(); ++i)
      if (gio.res_rep[i] >= 0) {
        const Rep& rr = ex.reps[g.epi[i].value][gio.res_rep[i]];
        in_bytes += static_cast<double>(rr.elems) * elem_bytes(rr.fmt);
      }
    double wbytes = 0, flops = 0;
    if (g.kind == GroupKind::Conv || g.kind == GroupKind::Dense) {
      int64_t wn = 1;
      for (auto d : g.weight.shape) wn *= d;
      wbytes = static_cast<double>(wn) * (g.weight.quant ? 1 : (path == P_CONV_F32 || path == P_DENSE_F32) ? 4 : 2);
      int64_t M = g.kind == GroupKind::Conv ? g.out_shape[0] * (has_sum ? g.pre_sum_shape[2] * g.pre_sum_shape[3] : g.out_shape[2] * g.out_shape[3])
                                             : g.out_shape[0];
      flops = 2.0 * static_cast<double>(M) * static_cast<double>(wn);
    } else if (g.kind == GroupKind::DwConv) {
      flops = 2.0 * g.out_shape[0] * g.out_shape[1] * g.out_shape[2] * g.out_shape[3] * g.kh * g.kw;
    }
    if (sc_g >= 0) {  // the fused shortcut: decimated codes + its weights, its MACs
      const GroupDesc& sg = P.groups[sc_g];
      const Rep& r2 = ex.reps[sg.data.value][gio.sc_rep];
      in_bytes += static_cast<double>(r2.elems) * elem_bytes(r2.fmt);
      int64_t wn = 1;
      for (auto d : sg.weight.shape) wn *= d;
      wbytes += static_cast<double>(wn) * (sg.weight.quant ? 1 : 2);
      flops += 2.0 * static_cast<double>(sg.out_shape[0] * sg.out_shape[2] * sg.out_shape[3]) * static_cast<double>(wn);
    }
    L.bytes = in_bytes + out_bytes + wbytes;
    L.flops = flops;

    Exec* e = &ex;
    int gidx = static_cast<int>(gi);
    int dbuf = drep.buf;
    int dfmt = drep.fmt;
    ConvGeom geo{};
    if (g.kind != GroupKind::Dense) {
      geo.N = static_cast<int>(g.in_shape[0]);
      geo.C = static_cast<int>(g.in_shape[1]);
      geo.H = static_cast<int>(g.in_shape[2]);
      geo.W = static_cast<int>(g.in_shape[3]);
      geo.in = drep.lay;
      const auto& os = has_sum ? g.pre_sum_shape : g.out_shape;
      geo.OC = static_cast<int>(os[1]);
      geo.OH = static_cast<int>(os[2]);
      geo.OW = static_cast<int>(os[3]);
      geo.KH = static_cast<int>(g.kh);
      geo.KW = static_cast<int>(g.kw);
      geo.sh = static_cast<int>(g.sh);
      geo.sw = static_cast<int>(g.sw);
      geo.ph = static_cast<int>(g.ph);
      geo.pw = static_cast<int>(g.pw);
    }
    float acc_scale = g.weight.quant ? gio.data_scale * g.weight.q.c2 : 1.f;
    // buffers' final addresses are only known after assign_offsets: capture ids.
    struct Ptrs { int out, side, presum, side2; };
    Ptrs pb{obuf, sbuf, pre_sum_buf, sbuf2};
    auto outdev = [e, pb, out]() {
      OutDev o = out;
      if (pb.presum >= 0) o.primary = e->ptr(pb.presum);
      else o.primary = e->bufs[pb.out].dead ? nullptr : e->ptr(pb.out);
      o.side = pb.side >= 0 ? e->ptr(pb.side) : nullptr;
      o.side2 = pb.side2 >= 0 ? e->ptr(pb.side2) : nullptr;
      return o;
    };
    auto epidev = [e, gidx, epi]() {
      EpiDev d = epi;
      // re-resolve arena pointers and constant vectors
      const GroupDesc& gg = e->P.groups[gidx];
      int n = 0, vi = 0;
      for (size_t i = 0; i < gg.epi.size() && n < d.n_ops; ++i) {
        const EpiOp& op = gg.epi[i];
        if (op.kind == EpiKind::SumHW || op.kind == EpiKind::Flatten) continue;
        if (op.kind == EpiKind::Bias) d.vec[n] = static_cast<const float*>(e->param_dev[e->P.values[op.value].param_index]);
        if (op.kind == EpiKind::MulChannel) d.vec[n] = static_cast<const float*>(e->group_vecs[gidx][1 + vi++]);
        ++n;
      }
      return d;
    };
    auto residual_fix = [e, gidx, gio](EpiDev& d) {
      const GroupDesc& gg = e->P.groups[gidx];
      int n = 0;
      for (size_t i = 0; i < gg.epi.size() && n < d.n_ops; ++i) {
        if (gg.epi[i].kind == EpiKind::SumHW || gg.epi[i].kind == EpiKind::Flatten) continue;
        if (gg.epi[i].kind == EpiKind::Residual && gio.res_rep[i] >= 0) {
          const Rep& r = e->reps[gg.epi[i].value][gio.res_rep[i]];
          d.res[n] = e->ptr(r.buf);
          d.res_lay[n] = r.lay;
        }
        ++n;
      }
    };
    switch (path) {
      case P_CONV_I8_SIMT:
      case P_CONV_BF16_SIMT:
      case P_CONV_F32: {
        L.fn = [e, gidx, dbuf, geo, acc_scale, path, outdev, epidev, residual_fix](cudaStream_t s) {
          EpiDev d = epidev();
          residual_fix(d);
          ConvGeom gg = geo;
          gg.Kp = e->group_kp[gidx];
          gg.Cs = e->group_cs[gidx];
          if (path == P_CONV_I8_SIMT)
            launch_conv_i8_simt(static_cast<const int8_t*>(e->ptr(dbuf)), static_cast<const int8_t*>(e->group_w[gidx]),
                                gg, acc_scale, d, outdev(), s);
          else if (path == P_CONV_BF16_SIMT)
            launch_conv_bf16_simt(static_cast<const uint16_t*>(e->ptr(dbuf)),
                                  static_cast<const uint16_t*>(e->group_w[gidx]), gg, d, outdev(), s);
          else
            launch_conv_f32_strict(static_cast<const float*>(e->ptr(dbuf)), static_cast<const float*>(e->group_w[gidx]),
                                   gg, d, outdev(), s);
        };
        break;
      }
      case P_CONV_I8_TC:
      case P_CONV_BF16_TC:
      case P_CONV_TF32_TC: {
        for (const EpiOp& op : g.epi) ex.group_tc[gi].residual |= op.kind == EpiKind::Residual ? 1 : 0;
        TcConvPlan* tp = tc_conv_create(ex.group_tc[gi]);
        if (!tp) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": tcgen05 plan failed");
        ex.tc_plans.push_back(tp);
        char buf[256];
        ex.group_note.resize(P.groups.size());
        ex.group_note[gi] = tc_conv_describe(tp, buf, sizeof(buf));
        if (pre_sum_buf < 0 && sbuf >= 0) L.opt_primary = obuf;
        std::string gname = g.name;
        Lay dlay = drep.lay;
        // fused shortcut operands (buffer ids: addresses are final only after assign_offsets)
        int sc_buf = -1, sc_bias_param = -1;
        Lay sc_lay{};
        float sc_scale = 1.f;
        if (sc_g >= 0) {
          const GroupDesc& sg = P.groups[sc_g];
          const Rep& sr = ex.reps[sg.data.value][gio.sc_rep];
          sc_buf = sr.buf;
          sc_lay = sr.lay;
          sc_scale = sg.weight.quant ? io[sc_g].data_scale * sg.weight.q.c2 : 1.f;
          sc_bias_param = P.values[sg.epi[0].value].param_index;
        }
        L.fn = [e, gidx, dbuf, dlay, acc_scale, tp, outdev, epidev, residual_fix, gname, sc_g, sc_buf, sc_lay, sc_scale,
                sc_bias_param](cudaStream_t s) {
          EpiDev d = epidev();
          residual_fix(d);
          TcShortcut sc;
          if (sc_g >= 0) {
            sc.x = e->ptr(sc_buf);
            sc.lay = sc_lay;
            sc.w = e->group_w[sc_g];
            sc.acc_scale = sc_scale;
            sc.bias = static_cast<const float*>(e->param_dev[sc_bias_param]);
          }
          if (!tc_conv_launch(tp, e->ptr(dbuf), dlay, e->group_w[gidx], acc_scale, d, outdev(), s, sc_g >= 0 ? &sc : nullptr))
            fail(MR_ERR_CUDA, "group %" + gname + ": tcgen05 conv launch refused (TMA descriptor encoding or epilogue form)");
        };
        break;
      }
      case P_DENSE_I8_TC:
      case P_DENSE_BF16_TC:
      case P_DENSE_TF32_TC: {
        DenseTcSpec ds{path == P_DENSE_I8_TC ? 1 : path == P_DENSE_TF32_TC ? 4 : 2, static_cast<int>(g.in_shape[0]), static_cast<int>(g.in_shape[1]),
                       static_cast<int>(g.out_shape[1])};
        DenseTcPlan* dp = dense_tc_create(ds);
        if (!dp) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": tcgen05 dense plan failed");
        ex.group_dense.resize(P.groups.size(), nullptr);
        ex.group_dense[gi] = dp;
        char buf[256];
        ex.group_note.resize(P.groups.size());
        ex.group_note[gi] = dense_tc_describe(dp, buf, sizeof(buf));
        auto fused_op = ex.sum_operand.find(static_cast<int>(gi));
        const bool op_ready = fused_op != ex.sum_operand.end();  // written by the producer's sum_hw
        const int opbuf = op_ready ? fused_op->second : B.scratch(dense_tc_operand_bytes(dp), "%" + g.name + ":operand");
        if (op_ready) B.use(opbuf);
        const int64_t wsb = dense_tc_workspace_bytes(dp);
        const int wsbuf = wsb ? B.scratch(wsb, "%" + g.name + ":splitk") : -1;
        L.kernels = dense_tc_launches(dp) - (op_ready ? 1 : 0);
        float pre = g.data.pre_mul;
        int quant = g.data.quant || gio.requant_data ? 1 : 0;
        QDev q = to_qdev(g.data.quant ? g.data.q : gio.requant_q);
        std::string gname = g.name;
        L.fn = [e, gidx, dbuf, dp, opbuf, wsbuf, pre, quant, q, acc_scale, outdev, epidev, residual_fix, gname,
                op_ready](cudaStream_t s) {
          EpiDev d = epidev();
          residual_fix(d);
          if (!dense_tc_launch(dp, op_ready ? nullptr : static_cast<const float*>(e->ptr(dbuf)), pre, quant, q, e->ptr(opbuf),
                               e->group_w[gidx], wsbuf >= 0 ? e->ptr(wsbuf) : nullptr, acc_scale, d, outdev(), s))
            fail(MR_ERR_CUDA, "group %" + gname + ": TMA descriptor encoding failed");
        };
        break;
      }
      case P_DENSE_I8:
      case P_DENSE_F32:
      case P_DENSE_BF16: {
        int N = static_cast<int>(g.in_shape[0]), K = static_cast<int>(g.in_shape[1]);
        int M = static_cast<int>(g.out_shape[1]);
        int mode = path == P_DENSE_I8 ? 0 : path == P_DENSE_F32 ? 1 : 2;
        float pre = g.data.pre_mul;
        int quant = g.data.quant || gio.requant_data ? 1 : 0;
        QDev q = to_qdev(g.data.quant ? g.data.q : gio.requant_q);
        L.fn = [e, gidx, dbuf, N, K, M, mode, pre, quant, q, acc_scale, outdev, epidev, residual_fix](cudaStream_t s) {
          EpiDev d = epidev();
          residual_fix(d);
          launch_dense(static_cast<const float*>(e->ptr(dbuf)), N, K, e->group_kp[gidx], e->group_w[gidx], M, mode,
                       pre, quant, q, acc_scale, d, outdev(), s);
        };
        break;
      }
      case P_POOL: {
        L.fn = [e, dbuf, dfmt, geo, outdev](cudaStream_t s) {
          launch_maxpool(e->ptr(dbuf), dfmt, geo, outdev(), s);
        };
        break;
      }
      case P_DW: {
        int strict = float_fmt(ex) == FMT_F32 ? 1 : 0;
        L.fn = [e, gidx, dbuf, dfmt, geo, strict, outdev, epidev, residual_fix](cudaStream_t s) {
          EpiDev d = epidev();
          residual_fix(d);
          launch_dwconv(e->ptr(dbuf), dfmt, static_cast<const float*>(e->group_w[gidx]), geo, strict, d, outdev(), s);
        };
        break;
      }
      default:
        fail(MR_ERR_INTERNAL, "no kernel path");
    }
    ex.launches.push_back(L);
    ++B.launch_idx;
    // CUDA-core producers write interior pixels only: clear the P16 borders
    // (the tcgen05 conv writes its own, it computes over the padded grid).
    bool tc_same = (path == P_CONV_I8_TC || path == P_CONV_BF16_TC || path == P_CONV_TF32_TC) &&
                   ex.group_tc[gi].kind == TC_S1;
    const auto& zshape = fp >= 0 ? P.groups[fp].out_shape : g.out_shape;
    if (!tc_same && !has_sum && zshape.size() == 4) {
      // interior-only producer: keep the padding ring zero without a per-run pass
      for (int b2 : {obuf, sbuf})
        if (b2 >= 0) ex.bufs[b2].zero_border = true;
    }
    if (has_sum && flatten_at >= 0) {
      // reshape view: the P16 float32 tensor -> row-major [N, C*H*W] (NCHW order)
      LaunchRec S;
      S.name = "%" + g.name;
      S.kernel = "flatten";
      const auto& ps = g.pre_sum_shape;
      S.bytes = 8.0 * ps[0] * ps[1] * ps[2] * ps[3];
      int N = static_cast<int>(ps[0]), C = static_cast<int>(ps[1]), H = static_cast<int>(ps[2]),
          W = static_cast<int>(ps[3]);
      B.use(pre_sum_buf);
      if (orep.fmt != FMT_F32) fail(MR_ERR_UNSUPPORTED_GROUP, "group %" + g.name + ": flattened value must be float32");
      const bool rq = flatten_at + 1 < static_cast<int>(g.epi.size());  // trailing realize chain
      const QDev q = rq ? to_qdev(g.epi.back().q) : QDev{};
      S.fn = [e, pre_sum_buf, pre_lay, obuf, N, C, H, W, rq, q](cudaStream_t s) {
        launch_to_nchw(e->ptr(pre_sum_buf), FMT_F32, pre_lay, 1.f, static_cast<float*>(e->ptr(obuf)), N, C, H, W, 1, s,
                       rq ? &q : nullptr);
      };
      ex.launches.push_back(S);
      ++B.launch_idx;
    } else if (has_sum) {
      LaunchRec S;
      S.name = "%" + g.name;
      S.kernel = "sum_hw";
      const auto& ps = g.pre_sum_shape;
      S.bytes = 4.0 * ps[0] * ps[1] * ps[2] * ps[3] + 4.0 * ps[0] * ps[1];
      int N = static_cast<int>(ps[0]), H = static_cast<int>(ps[2]), W = static_cast<int>(ps[3]);
      int C = static_cast<int>(ps[1]);
      B.use(pre_sum_buf);
      // cross-group fusion: when a tcgen05 dense is the
      // sum's only consumer (the classifier head), the sum kernel applies the
      // dense's data prologue (multiply by 1/HW, realize chain) and writes its A
      // operand directly -- no float32 round trip, no operand launch
      const ValueInfo& sv = P.values[g.out_value];
      int dgi = -1;
      static const bool no_fuse = [] {  // A/B switch
        const char* e2 = std::getenv("MRB200_NO_SUM_FUSE");
        return e2 && std::atoi(e2);
      }();
      if (!no_fuse && sv.consumers.size() == 1 && !sv.is_result && C % 32 == 0 && H * W <= 64) {
        const int c = sv.consumers[0];
        const int dp = ex.group_path[c];
        const int eb = dp == P_DENSE_I8_TC ? 1 : dp == P_DENSE_BF16_TC ? 2 : dp == P_DENSE_TF32_TC ? 4 : 0;
        if (eb && P.groups[c].data.value == g.out_value && (C * eb) % 128 == 0) dgi = c;
      }
      SumOperand sop{};
      int opbuf = -1;
      if (dgi >= 0) {
        const GroupDesc& dg = P.groups[dgi];
        const GroupIO& dio = io[dgi];
        const int dp = ex.group_path[dgi];
        sop.eb = dp == P_DENSE_I8_TC ? 1 : dp == P_DENSE_BF16_TC ? 2 : 4;
        sop.Kp = C;
        sop.pre_mul = dg.data.pre_mul;
        sop.quant = dg.data.quant || dio.requant_data ? 1 : 0;
        sop.q = to_qdev(dg.data.quant ? dg.data.q : dio.requant_q);
        opbuf = B.scratch(round_up(N, 128) * static_cast<int64_t>(C) * sop.eb, "%" + dg.name + ":operand");
        ex.sum_operand[dgi] = opbuf;
        S.kernel = "sum_hw+dense_operand";
        S.bytes = 4.0 * ps[0] * ps[1] * ps[2] * ps[3] + static_cast<double>(sop.eb) * ps[0] * ps[1];
      }
      S.fn = [e, pre_sum_buf, pre_lay, obuf, N, H, W, C, sop, opbuf](cudaStream_t s) {
        SumOperand o = sop;
        if (opbuf >= 0) o.ptr = e->ptr(opbuf);
        launch_sum_hw(static_cast<const float*>(e->ptr(pre_sum_buf)), pre_lay, N, H, W, C,
                      opbuf >= 0 ? nullptr : static_cast<float*>(e->ptr(obuf)), s, opbuf >= 0 ? &o : nullptr);
      };
      ex.launches.push_back(S);
      ++B.launch_idx;
    }
  }

  // ---- result: NCHW float32 ----
  const ValueInfo& rv = P.values[P.result_value];
  if (rv.producer < 0) fail(MR_ERR_UNSUPPORTED_GROUP, "@main returns a parameter");
  const Rep& rr = ex.reps[P.result_value][0];
  ex.out_shape = rv.shape;
  ex.out_elems = 1;
  for (auto d : rv.shape) ex.out_elems *= d;
  // a float32 row-major [N, M] result (a dense head) already is the boundary
  // layout: the executor reads it in place, no conversion launch
  const bool alias_result = rr.fmt == FMT_F32 && !rr.has_q && rv.shape.size() == 2 && rr.lay.cpc == 0;
  if (alias_result) {
    ex.out_alias_buf = rr.buf;
    B.use(rr.buf);  // keep it live to the end of the step
  } else {
    CK(cudaMalloc(&ex.out_internal, static_cast<size_t>(ex.out_elems) * 4));
  }
  if (!alias_result) {
    // NCHW float32 at the boundary; a realize-coded result is dequantized
    // (code * c2, exact) so the value equals the reference's float32 tensor.
    int rbuf = rr.buf;
    B.use(rbuf);
    LaunchRec L;
    L.name = "%" + rv.name;
    Exec* e = &ex;
    L.kernel = "result_to_nchw";
    L.bytes = static_cast<double>(ex.out_elems) * (4 + elem_bytes(rr.fmt));
    int N = static_cast<int>(rv.shape[0]), C = static_cast<int>(rv.shape[1]);
    int H = rv.shape.size() == 4 ? static_cast<int>(rv.shape[2]) : 1;
    int W = rv.shape.size() == 4 ? static_cast<int>(rv.shape[3]) : 1;
    int fmt = rr.fmt;
    Lay lay = rr.lay;
    int is4d = rv.shape.size() == 4 ? 1 : 0;
    float c2 = rr.has_q ? rr.q.c2 : 1.f;
    L.fn = [e, rbuf, fmt, lay, c2, N, C, H, W, is4d](cudaStream_t s) {
      launch_to_nchw(e->ptr(rbuf), fmt, lay, c2, e->out_dst(), N, C, H, W, is4d, s);
    };
    ex.launches.push_back(L);
    ++B.launch_idx;
  }

  for (size_t i = 0; i < ex.launches.size(); ++i) {
    LaunchRec& L = ex.launches[i];
    if (L.opt_primary < 0 || L.opt_primary == ex.out_alias_buf) continue;
    Buffer& b = ex.bufs[L.opt_primary];
    if (b.first == static_cast<int>(i) && b.last == static_cast<int>(i) && !b.zero_border) {
      b.dead = true;
      L.bytes -= static_cast<double>(b.bytes);
      b.bytes = 0;
      b.what += " (unread: not written)";
    }
  }
  assign_offsets(ex);
  CK(cudaMalloc(&ex.arena, static_cast<size_t>(std::max<int64_t>(ex.arena_bytes, 256))));
  if (ex.zero_bytes) CK(cudaMemset(ex.arena, 0, static_cast<size_t>(ex.zero_bytes)));
  if (ex.out_alias_buf >= 0) ex.out_internal = static_cast<float*>(ex.ptr(ex.out_alias_buf));
}

}  // namespace mrb200

// ======================================================================
// weights + describe + C ABI
// ======================================================================
namespace mrb200 {
namespace {

void upload_group_constants(Exec& ex) {
  ex.group_vecs.assign(ex.P.groups.size(), {});
  for (size_t gi = 0; gi < ex.P.groups.size(); ++gi) {
    const GroupDesc& g = ex.P.groups[gi];
    auto up = [&](const std::vector<float>& v) -> void* {
      if (v.empty()) return nullptr;
      void* p = nullptr;
      CK(cudaMalloc(&p, v.size() * 4));
      CK(cudaMemcpy(p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
      return p;
    };
    ex.group_vecs[gi].push_back(up(g.weight.oc_scale));  // [0]: weight oc scale
    for (const auto& op : g.epi)
      if (op.kind == EpiKind::MulChannel) ex.group_vecs[gi].push_back(up(op.vec));
  }
}

void prepare_weights(Exec& ex, cudaStream_t s) {
  const Program& P = ex.P;
  const int ffmt = float_fmt(ex);
  ex.group_w.assign(P.groups.size(), nullptr);
  ex.group_kp.assign(P.groups.size(), 0);
  ex.group_cs.assign(P.groups.size(), 0);
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    const GroupDesc& g = P.groups[gi];
    if (g.kind == GroupKind::MaxPool) continue;
    const WeightOperand& w = g.weight;
    const float* raw = nullptr;
    void* tmp = nullptr;
    if (w.value >= 0) {
      raw = static_cast<const float*>(ex.param_dev[P.values[w.value].param_index]);
    } else {
      CK(cudaMalloc(&tmp, w.constant.size() * 4));
      CK(cudaMemcpy(tmp, w.constant.data(), w.constant.size() * 4, cudaMemcpyHostToDevice));
      raw = static_cast<const float*>(tmp);
    }
    int path = ex.group_path[gi];
    int O, I, KH = 1, KW = 1;
    if (g.kind == GroupKind::Dense) {
      O = static_cast<int>(w.shape[0]);
      I = static_cast<int>(w.shape[1]);
    } else {
      O = static_cast<int>(w.shape[0]);
      I = static_cast<int>(w.shape[1]);
      KH = static_cast<int>(w.shape[2]);
      KW = static_cast<int>(w.shape[3]);
    }
    int fmt, cs;
    int wl = WL_ROWS;
    if (path == P_CONV_I8_TC || path == P_CONV_BF16_TC || path == P_CONV_TF32_TC)
      wl = ex.group_tc[gi].kind == TC_STEM_S2D || ex.group_tc[gi].kind == TC_STEM_POOL ? WL_S2D : WL_TC;
    if (w.quant) {
      fmt = FMT_I8;
      cs = static_cast<int>(round_up(I, 4));
    } else if (g.kind == GroupKind::DwConv || ffmt == FMT_F32) {
      fmt = FMT_F32;
      cs = I;
    } else {
      fmt = FMT_BF16;
      cs = g.kind == GroupKind::Dense ? static_cast<int>(round_up(I, 8)) : I;  // dense: [K/8][M][8] (k_dense)
    }
    int64_t n;
    if (fmt == FMT_F32 && wl == WL_ROWS) {
      n = static_cast<int64_t>(O) * I * KH * KW;
    } else if (wl == WL_TC || wl == WL_S2D) {
      const TcConvSpec& sp = ex.group_tc[gi];
      int cpc = sp.kb / static_cast<int>(elem_bytes(fmt));
      n = static_cast<int64_t>(sp.taps) * sp.wplanes * O * cpc;
      cs = sp.kb;  // k_weight_prep: chunk bytes for the tcgen05 layouts
    } else {
      n = static_cast<int64_t>(O) * KH * KW * cs;
    }
    const DenseTcPlan* dtc = gi < ex.group_dense.size() ? ex.group_dense[gi] : nullptr;
    const bool dense_t = g.kind == GroupKind::Dense && fmt != FMT_F32 && !dtc;  // transposed k_dense layouts
    if (dense_t) n = static_cast<int64_t>(O) * cs;
    if (dtc) {  // tcgen05 dense: K-major rows [Mpad][Kp]
      cs = dense_tc_kp(I, static_cast<int>(elem_bytes(fmt)));
      n = dense_tc_weight_rows(dtc) * cs;
    }
    void* dst = nullptr;
    CK(cudaMalloc(&dst, static_cast<size_t>(n * elem_bytes(fmt))));
    if ((wl == WL_TC || wl == WL_S2D) && ex.group_tc[gi].taps > KH * KW)  // zero-weight dummy taps (paired-tap convs)
      CK(cudaMemsetAsync(dst, 0, static_cast<size_t>(n * elem_bytes(fmt)), s));
    if (dtc)
      dense_tc_prep_weight(dtc, raw, static_cast<const float*>(ex.group_vecs[gi][0]), w.scalar_scale,
                           w.quant ? 1 : 0, to_qdev(w.q), dst, s);
    else if (dense_t)
      launch_dense_weight_t(raw, O, I, cs, static_cast<const float*>(ex.group_vecs[gi][0]), w.scalar_scale, fmt,
                            w.quant ? 1 : 0, to_qdev(w.q), dst, s);
    else
      launch_weight_prep(raw, O, I, KH, KW, cs, wl, static_cast<const float*>(ex.group_vecs[gi][0]), w.scalar_scale,
                         fmt, w.quant ? 1 : 0, to_qdev(w.q), dst, s);
    CK(cudaGetLastError());
    ex.group_w[gi] = dst;
    ex.group_kp[gi] = fmt == FMT_F32 ? I * KH * KW : KH * KW * cs;
    ex.group_cs[gi] = cs;
    if (tmp) {
      CK(cudaStreamSynchronize(s));
      cudaFree(tmp);
    }
    // Static exactness proof for int8 contractions: every partial sum of the
    // reference's sequential fp32 accumulation is an integer multiple of the
    // quantum with |.| <= sum_k |w_code| * max|x_code|; below 2^24 it is
    // exact, so the int32 result converted and scaled equals it bit for bit.
    if (w.quant) {
      CK(cudaStreamSynchronize(s));
      std::vector<int8_t> codes(static_cast<size_t>(n));
      CK(cudaMemcpy(codes.data(), dst, static_cast<size_t>(n), cudaMemcpyDeviceToHost));
      std::vector<int64_t> sums(O, 0);
      int64_t per = n / O, worst = 0;
      for (int64_t k = 0; k < n; ++k) {
        if (dtc && k / cs >= O) break;  // zero padding rows
        int o = dtc ? static_cast<int>(k / cs) : dense_t ? static_cast<int>((k / 4) % O)
                : wl != WL_ROWS ? static_cast<int>((k / ex.group_tc[gi].kb) % O) : static_cast<int>(k / per);
        sums[o] += std::abs(static_cast<int>(codes[k]));
      }
      for (int o = 0; o < O; ++o) worst = std::max(worst, sums[o]);
      float xmax = g.data.quant ? std::max(std::fabs(g.data.q.lo), std::fabs(g.data.q.hi))
                                : std::max(std::fabs(P.values[g.data.value].q.lo), std::fabs(P.values[g.data.value].q.hi));
      double bound = static_cast<double>(worst) * xmax;
      std::ostringstream os;
      os << (bound <= 16777216.0 ? "proven" : "unproven") << " (max partial sum <= " << static_cast<int64_t>(bound)
         << " quanta)";
      ex.group_exact[gi] = os.str();
      if (bound > 16777216.0 && ex.enforce_exact)
        fail(MR_ERR_INEXACT_INT8, "%" + g.name + ": int8 partial sums are not proven below 2^24 quanta (" +
                                      os.str() + "); the int32 accumulation could differ from interp()'s fp32 sum");
    }
  }
}

std::string program_json(const Program& P) {
  static const char* kinds[] = {"conv2d", "dense", "max_pool2d", "depthwise_conv2d"};
  std::ostringstream os;
  os << "{\"int8\": " << (P.any_quant ? "true" : "false") << ", \"n_params\": " << P.n_params
     << ", \"result_shape\": " << dims_str(P.values[P.result_value].shape) << ", \"groups\": [";
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    const GroupDesc& g = P.groups[gi];
    std::string d = describe_group(P, g);
    std::string esc;
    for (char c : d) esc += (c == '"' ? '\'' : c);
    os << (gi ? ", " : "") << "{\"name\": \"" << g.name << "\", \"anchor\": \"" << kinds[static_cast<int>(g.kind)]
       << "\", \"desc\": \"" << esc << "\", \"data_quant\": " << (g.data.quant ? "true" : "false")
       << ", \"weight_quant\": " << (g.weight.quant ? "true" : "false") << ", \"kernel\": ["
       << g.kh << ", " << g.kw << "], \"strides\": [" << g.sh << ", " << g.sw << "], \"padding\": [" << g.ph << ", "
       << g.pw << "], \"epilogue\": [";
    for (size_t i = 0; i < g.epi.size(); ++i) os << (i ? ", " : "") << static_cast<int>(g.epi[i].kind);
    os << "], \"in_shape\": " << dims_str(g.in_shape) << ", \"out_shape\": " << dims_str(g.out_shape) << "}";
  }
  os << "]}";
  return os.str();
}

void make_describe(Exec& ex) {
  std::ostringstream os;
  const Program& P = ex.P;
  os << "{\"batch\": " << ex.opt.batch << ", \"float_mode\": " << ex.opt.float_mode
     << ", \"int8\": " << (P.any_quant ? "true" : "false") << ", \"arena_bytes\": " << ex.arena_bytes
     << ", \"groups\": [";
  for (size_t gi = 0; gi < P.groups.size(); ++gi) {
    const GroupDesc& g = P.groups[gi];
    std::string d = describe_group(P, g);
    std::string esc;
    for (char c : d) esc += (c == '"' ? '\'' : c);
    os << (gi ? ", " : "") << "{\"name\": \"" << g.name << "\", \"desc\": \"" << esc << "\", \"kernel\": \""
       << path_name(ex.group_path[gi]) << "\", \"out_shape\": " << dims_str(g.out_shape) << ", \"exact\": \""
       << ex.group_exact[gi] << "\", \"plan\": \"" << (gi < ex.group_note.size() ? ex.group_note[gi] : "") << "\"}";
  }
  os << "], \"launches\": [";
  for (size_t i = 0; i < ex.launches.size(); ++i) {
    const LaunchRec& L = ex.launches[i];
    os << (i ? ", " : "") << "{\"name\": \"" << L.name << "\", \"kernel\": \"" << L.kernel
       << "\", \"kernels\": " << L.kernels << ", \"bytes\": " << static_cast<int64_t>(L.bytes)
       << ", \"flops\": " << static_cast<int64_t>(L.flops) << "}";
  }
  os << "], \"buffers\": [";
  for (size_t i = 0; i < ex.bufs.size(); ++i) {
    const Buffer& b = ex.bufs[i];
    os << (i ? ", " : "") << "{\"what\": \"" << b.what << "\", \"bytes\": " << b.bytes << ", \"offset\": " << b.offset
       << ", \"live\": [" << b.first << ", " << b.last << "]}";
  }
  os << "]}";
  ex.describe = os.str();
}

void run_launches(Exec& ex, cudaStream_t s) {
  static const bool sync_debug = [] {
    const char* e = std::getenv("MRB200_SYNC_DEBUG");
    return e && std::atoi(e);
  }();
  for (auto& L : ex.launches) {
    if (sync_debug) std::fprintf(stderr, "MRB200_SYNC_DEBUG launch %s (%s)\n", L.name.c_str(), L.kernel.c_str());
    L.fn(s);
    if (sync_debug) {  // debugging only: name the launch that faults
      cudaError_t err = cudaStreamSynchronize(s);
      if (err == cudaSuccess) err = cudaGetLastError();
      if (err != cudaSuccess) fail(MR_ERR_CUDA, "launch " + L.name + " (" + L.kernel + "): " + cudaGetErrorString(err));
    }
  }
}

cudaGraphExec_t ensure_graph(Exec& ex) {
  for (auto& g : ex.graphs)
    if (g.in == ex.cur_inputs && g.out == ex.out_redirect) return g.e;
  if (ex.graphs.size() >= 4) {  // bounded cache: drop the oldest capture
    cudaGraphExecDestroy(ex.graphs.front().e);
    cudaGraphDestroy(ex.graphs.front().g);
    ex.graphs.erase(ex.graphs.begin());
  }
  cudaStream_t cap = nullptr;
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  run_launches(ex, cap);
  Exec::GraphEnt ent{ex.cur_inputs, ex.out_redirect, nullptr, nullptr};
  cudaError_t ce = cudaStreamEndCapture(cap, &ent.g);
  cudaStreamDestroy(cap);
  if (ce != cudaSuccess) fail(MR_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
  CK(cudaGraphInstantiate(&ent.e, ent.g, 0));
  ex.graphs.push_back(ent);
  return ent.e;
}

void run_body(Exec& ex, cudaStream_t s) {
  if (ex.opt.use_cuda_graph) {
    CK(cudaGraphLaunch(ensure_graph(ex), s));
  } else {
    run_launches(ex, s);
    CK(cudaGetLastError());
  }
}

int64_t numel(const mr_tensor& t) {
  int64_t n = 1;
  for (int i = 0; i < t.ndim; ++i) n *= t.shape[i];
  return n;
}

void check_input(const Exec& ex, const mr_tensor* inputs) {
  if (!inputs) fail(MR_ERR_INVALID_ARGUMENT, "null input");
  int seen = 0;
  for (const auto& v : ex.P.values) {
    if (!v.is_data) continue;
    const mr_tensor& t = inputs[v.param_index];
    if (!t.data) fail(MR_ERR_INVALID_ARGUMENT, "null input %" + v.name);
    if (t.ndim != static_cast<int>(v.shape.size())) fail(MR_ERR_TYPE_MISMATCH, "input %" + v.name + " rank mismatch");
    for (int i = 0; i < t.ndim; ++i)
      if (t.shape[i] != v.shape[i]) fail(MR_ERR_TYPE_MISMATCH, "input %" + v.name + " shape mismatch with the bound batch");
    if (t.type_code != MR_FLOAT || t.bits != 32) fail(MR_ERR_TYPE_MISMATCH, "input %" + v.name + " must be float32");
    ++seen;
  }
  if (!seen) fail(MR_ERR_INVALID_ARGUMENT, "module has no data input");
}

void set_inputs(Exec& ex, const mr_tensor* inputs) {
  ex.cur_inputs.assign(static_cast<size_t>(ex.opt.n_data_inputs), nullptr);
  for (int k = 0; k < ex.opt.n_data_inputs; ++k) ex.cur_inputs[k] = static_cast<const float*>(inputs[k].data);
}

}  // namespace
}  // namespace mrb200

using namespace mrb200;

#define API_BEGIN try {
#define API_END                                       \
  }                                                   \
  catch (const Status& s) {                           \
    g_last_error = s.msg;                             \
    return static_cast<mr_status>(s.code);            \
  }                                                   \
  catch (const LowerError& e) {                       \
    g_last_error = e.msg;                             \
    return static_cast<mr_status>(e.code);            \
  }                                                   \
  catch (const ParseError& e) {                       \
    g_last_error = "syntax: " + e.msg;                \
    return MR_ERR_SYNTAX;                             \
  }                                                   \
  catch (const std::bad_alloc&) {                     \
    g_last_error = "host out of memory";              \
    return MR_ERR_OUT_OF_MEMORY;                      \
  }                                                   \
  catch (const std::exception& e) {                   \
    g_last_error = e.what();                          \
    return MR_ERR_INTERNAL;                           \
  }                                                   \
  return MR_OK;

namespace mrb200 {
namespace {
// Binds the non-data @main params (w[i] = param n_data_inputs + i) and runs the
// hoisted weight prologues.  `kind` is H2D for mr_exec_set_weights, D2D for the
// group-level launch whose operands are device tensors.
void load_weights(Exec& ex, int32_t n, const mr_tensor* w, cudaMemcpyKind kind) {
  int expect = ex.P.n_params - static_cast<int>(ex.P.hidden_data.size()) - ex.opt.n_data_inputs;
  if (n != expect) fail(MR_ERR_ARITY_MISMATCH, "expected " + std::to_string(expect) + " weight tensors");
  if (n && !w) fail(MR_ERR_INVALID_ARGUMENT, "null weights");
  for (const auto& v : ex.P.values) {
    if (v.param_index < 0 || v.is_data || v.hidden >= 0) continue;
    const mr_tensor& t = w[v.param_index - ex.opt.n_data_inputs];
    if (t.type_code != MR_FLOAT || t.bits != 32) fail(MR_ERR_TYPE_MISMATCH, "%" + v.name + " must be float32");
    if (t.ndim != static_cast<int>(v.shape.size())) fail(MR_ERR_TYPE_MISMATCH, "%" + v.name + " rank mismatch");
    for (int i = 0; i < t.ndim; ++i)
      if (t.shape[i] != v.shape[i]) fail(MR_ERR_TYPE_MISMATCH, "%" + v.name + " shape mismatch");
    int64_t bytes = numel(t) * 4;
    if (bytes && !t.data) fail(MR_ERR_INVALID_ARGUMENT, "null tensor %" + v.name);
    void*& dst = ex.param_dev[v.param_index];
    if (!dst) CK(cudaMalloc(&dst, static_cast<size_t>(std::max<int64_t>(bytes, 4))));
    if (bytes) CK(cudaMemcpy(dst, t.data, static_cast<size_t>(bytes), kind));
  }
  for (void* p : ex.group_w) if (p) cudaFree(p);
  prepare_weights(ex, nullptr);
  CK(cudaDeviceSynchronize());
  ex.weights_ready = true;
  ex.drop_graphs();  // weights live at fixed addresses only after the first set
  make_describe(ex);
}

std::unique_ptr<Exec> make_exec(Program P, const mr_exec_options& o, bool enforce_exact = true) {
  auto ex = std::make_unique<Exec>();
  ex->opt = o;
  ex->enforce_exact = enforce_exact;
  ex->P = std::move(P);
  if (ex->opt.n_data_inputs < 1) fail(MR_ERR_INVALID_ARGUMENT, "at least one data input");
  build(*ex);
  upload_group_constants(*ex);
  ex->param_dev.assign(ex->P.n_params, nullptr);
  // embedded weights (hidden parameters): uploaded once here
  for (const auto& v : ex->P.values) {
    if (v.hidden < 0) continue;
    const auto& data = ex->P.hidden_data[static_cast<size_t>(v.hidden)];
    void*& dst = ex->param_dev[v.param_index];
    CK(cudaMalloc(&dst, std::max<size_t>(data.size() * 4, 4)));
    if (!data.empty()) CK(cudaMemcpy(dst, data.data(), data.size() * 4, cudaMemcpyHostToDevice));
  }
  make_describe(*ex);
  // nothing left for mr_exec_set_weights to bind: prepare the weights now
  if (ex->P.n_params - static_cast<int>(ex->P.hidden_data.size()) == ex->opt.n_data_inputs)
    load_weights(*ex, 0, nullptr, cudaMemcpyHostToDevice);
  return ex;
}
}  // namespace
}  // namespace mrb200

extern "C" {

void mr_exec_default_options(mr_exec_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->batch = 1;
  o->n_data_inputs = 1;
  o->float_mode = MR_FLOAT_BF16;
  o->use_cuda_graph = 1;
  o->force_simt = 0;
}

mr_status mr_exec_create(const char* text, const mr_exec_options* opts, mr_exec_t* out) {
  API_BEGIN
  if (!text || !out) fail(MR_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  mr_exec_options o;
  mr_exec_default_options(&o);
  if (opts) o = *opts;
  if (o.batch < 1) fail(MR_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  DeviceGuard dg(o.device);
  Module m = parse_fused_module(text);
  *out = reinterpret_cast<mr_exec_t>(make_exec(lower_module(m, o.batch, o.n_data_inputs), o).release());
  API_END
}

mr_status mr_exec_set_weights(mr_exec_t h, int32_t n, const mr_tensor* w) {
  API_BEGIN
  if (!h) fail(MR_ERR_INVALID_ARGUMENT, "null executor");
  Exec& ex = *reinterpret_cast<Exec*>(h);
  DeviceGuard dg(ex.opt.device);
  load_weights(ex, n, w, cudaMemcpyHostToDevice);
  API_END
}

// The caller's device output becomes the final launch's destination for one run.
struct OutRedirect {
  Exec& ex;
  OutRedirect(Exec& e, void* p) : ex(e) { ex.out_redirect = static_cast<float*>(p); }
  ~OutRedirect() { ex.out_redirect = nullptr; }
};

void check_device_output(const Exec& ex, const mr_tensor* output) {
  if (!output || !output->data) fail(MR_ERR_INVALID_ARGUMENT, "null output");
  if (numel(*output) != ex.out_elems) fail(MR_ERR_TYPE_MISMATCH, "output size mismatch");
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, output->data) != cudaSuccess ||
      (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) || a.device != ex.opt.device) {
    cudaGetLastError();
    fail(MR_ERR_INVALID_ARGUMENT, "output must be device memory on the executor's device");
  }
}

mr_status mr_exec_run(mr_exec_t h, const mr_tensor* inputs, mr_tensor* output, void* stream) {
  API_BEGIN
  if (!h) fail(MR_ERR_INVALID_ARGUMENT, "null executor");
  Exec& ex = *reinterpret_cast<Exec*>(h);
  DeviceGuard dg(ex.opt.device);
  if (!ex.weights_ready) fail(MR_ERR_INVALID_ARGUMENT, "mr_exec_set_weights first");
  check_input(ex, inputs);
  check_device_output(ex, output);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  set_inputs(ex, inputs);
  OutRedirect r(ex, output->data);
  run_body(ex, s);
  API_END
}

mr_status mr_exec_run_host(mr_exec_t h, const mr_tensor* inputs, mr_tensor* output, void* stream) {
  API_BEGIN
  if (!h) fail(MR_ERR_INVALID_ARGUMENT, "null executor");
  Exec& ex = *reinterpret_cast<Exec*>(h);
  DeviceGuard dg(ex.opt.device);
  check_input(ex, inputs);
  if (!output || !output->data) fail(MR_ERR_INVALID_ARGUMENT, "null output");
  if (numel(*output) != ex.out_elems) fail(MR_ERR_TYPE_MISMATCH, "output size mismatch");
  const int nd = ex.opt.n_data_inputs;
  ex.dev_in.resize(static_cast<size_t>(nd), nullptr);
  ex.in_elems.resize(static_cast<size_t>(nd), 0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ex.cur_inputs.assign(static_cast<size_t>(nd), nullptr);
  for (int k = 0; k < nd; ++k) {
    const int64_t n_in = numel(inputs[k]);
    if (!ex.dev_in[k] || ex.in_elems[k] != n_in) {
      if (ex.dev_in[k]) cudaFree(ex.dev_in[k]);
      CK(cudaMalloc(&ex.dev_in[k], static_cast<size_t>(n_in) * 4));
      ex.in_elems[k] = n_in;
    }
    CK(cudaMemcpyAsync(ex.dev_in[k], inputs[k].data, static_cast<size_t>(n_in) * 4, cudaMemcpyHostToDevice, s));
    ex.cur_inputs[k] = ex.dev_in[k];
  }
  if (!ex.weights_ready) fail(MR_ERR_INVALID_ARGUMENT, "mr_exec_set_weights first");
  run_body(ex, s);
  CK(cudaMemcpyAsync(output->data, ex.out_internal, static_cast<size_t>(ex.out_elems) * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  API_END
}

mr_status mr_exec_submit_host(mr_exec_t h, const mr_tensor* inputs, mr_tensor* output, void* stream) {
  API_BEGIN
  if (!h) fail(MR_ERR_INVALID_ARGUMENT, "null executor");
  Exec& ex = *reinterpret_cast<Exec*>(h);
  DeviceGuard dg(ex.opt.device);
  if (!ex.weights_ready) fail(MR_ERR_INVALID_ARGUMENT, "mr_exec_set_weights first");
  check_input(ex, inputs);
  if (!output || !output->data) fail(MR_ERR_INVALID_ARGUMENT, "null output");
  if (numel(*output) != ex.out_elems) fail(MR_ERR_TYPE_MISMATCH, "output size mismatch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!ex.pipe_fresh && s != ex.pipe_stream) fail(MR_ERR_INVALID_ARGUMENT, "mr_exec_sync before switching streams");
  if (ex.opt.n_data_inputs != 1) fail(MR_ERR_INVALID_ARGUMENT, "mr_exec_submit_host streams one data input");
  const int64_t n_in = numel(inputs[0]);
  if (!ex.copy_stream) {
    CK(cudaStreamCreateWithFlags(&ex.copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaMalloc(&ex.stage[i], static_cast<size_t>(n_in) * 4));
      CK(cudaEventCreateWithFlags(&ex.loaded[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ex.consumed[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&ex.fresh, cudaEventDisableTiming));
  }
  const int b = static_cast<int>(ex.submitted & 1);
  if (ex.pipe_fresh) {
    // the first upload after a sync is ordered after the work already on `stream`
    CK(cudaEventRecord(ex.fresh, s));
    CK(cudaStreamWaitEvent(ex.copy_stream, ex.fresh, 0));
    ex.pipe_fresh = false;
    ex.pipe_stream = s;
  }
  if (ex.submitted >= 2) CK(cudaStreamWaitEvent(ex.copy_stream, ex.consumed[b], 0));  // stage b's last reader done
  CK(cudaMemcpyAsync(ex.stage[b], inputs[0].data, static_cast<size_t>(n_in) * 4, cudaMemcpyHostToDevice,
                     ex.copy_stream));
  CK(cudaEventRecord(ex.loaded[b], ex.copy_stream));
  CK(cudaStreamWaitEvent(s, ex.loaded[b], 0));
  ex.cur_inputs.assign(1, ex.stage[b]);
  run_body(ex, s);
  CK(cudaEventRecord(ex.consumed[b], s));
  CK(cudaMemcpyAsync(output->data, ex.out_internal, static_cast<size_t>(ex.out_elems) * 4, cudaMemcpyDeviceToHost, s));
  ++ex.submitted;
  API_END
}

mr_status mr_exec_sync(mr_exec_t h) {
  API_BEGIN
  if (!h) fail(MR_ERR_INVALID_ARGUMENT, "null executor");
  Exec& ex = *reinterpret_cast<Exec*>(h);
  DeviceGuard dg(ex.opt.device);
  if (!ex.pipe_fresh) {  // (the stream may be the legacy default stream, handle 0)
    if (ex.copy_stream) CK(cudaStreamSynchronize(ex.copy_stream));
    CK(cudaStreamSynchronize(ex.pipe_stream));
  }
  ex.pipe_fresh = true;
  ex.pipe_stream = nullptr;
  API_END
}

mr_status mr_exec_output_shape(mr_exec_t h, mr_tensor* t) {
  API_BEGIN
  Exec& ex = *reinterpret_cast<Exec*>(h);
  t->ndim = static_cast<int32_t>(ex.out_shape.size());
  for (size_t i = 0; i < ex.out_shape.size(); ++i) t->shape[i] = ex.out_shape[i];
  t->type_code = MR_FLOAT;
  t->bits = 32;
  API_END
}

const char* mr_exec_describe(mr_exec_t h) { return reinterpret_cast<Exec*>(h)->describe.c_str(); }

int32_t mr_exec_launch_count(mr_exec_t h) {
  Exec& ex = *reinterpret_cast<Exec*>(h);
  int32_t n = 0;
  for (const auto& L : ex.launches) n += L.fn ? L.kernels : 0;
  return n;
}

namespace {
struct EventList {  // RAII: the per-launch events are freed on every exit path
  std::vector<cudaEvent_t> ev;
  explicit EventList(size_t n) : ev(n, nullptr) {
    for (auto& e : ev) CK(cudaEventCreate(&e));
  }
  ~EventList() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};
mr_status profile_impl(Exec& ex, const mr_tensor* inputs, mr_tensor* output, void* stream, float* ms, int32_t cap,
                       int32_t* count) {
  API_BEGIN
  DeviceGuard dg(ex.opt.device);
  if (!ex.weights_ready) fail(MR_ERR_INVALID_ARGUMENT, "mr_exec_set_weights first");
  if (cap > 0 && !ms) fail(MR_ERR_INVALID_ARGUMENT, "null ms");
  check_input(ex, inputs);
  if (output && output->data) check_device_output(ex, output);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  set_inputs(ex, inputs);
  OutRedirect r(ex, output ? output->data : nullptr);
  EventList E(ex.launches.size() + 1);
  CK(cudaEventRecord(E.ev[0], s));
  for (size_t i = 0; i < ex.launches.size(); ++i) {
    ex.launches[i].fn(s);
    CK(cudaEventRecord(E.ev[i + 1], s));
  }
  CK(cudaEventSynchronize(E.ev.back()));
  CK(cudaGetLastError());
  int32_t n = 0;
  for (size_t i = 0; i < ex.launches.size() && n < cap; ++i) CK(cudaEventElapsedTime(&ms[n++], E.ev[i], E.ev[i + 1]));
  *count = n;
  API_END
}
}  // namespace

int32_t mr_exec_profile(mr_exec_t h, const mr_tensor* inputs, mr_tensor* output, void* stream, float* ms,
                        int32_t cap) {
  if (!h) {
    g_last_error = "null executor";
    return -1;
  }
  int32_t n = 0;
  return profile_impl(*reinterpret_cast<Exec*>(h), inputs, output, stream, ms, cap, &n) == MR_OK ? n : -1;
}

void mr_exec_destroy(mr_exec_t h) {
  if (!h) return;
  Exec* ex = reinterpret_cast<Exec*>(h);
  try {
    DeviceGuard dg(ex->opt.device);
    delete ex;
  } catch (...) {
    delete ex;
  }
}

const char* mr_last_error_message(void) { return g_last_error.c_str(); }

mr_status mr_module_lower(const char* text, int64_t batch, int32_t n_data_inputs, const char** json) {
  static thread_local std::string out;
  API_BEGIN
  if (!text || !json) fail(MR_ERR_INVALID_ARGUMENT, "null argument");
  if (batch < 1) fail(MR_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  Module m = parse_fused_module(text);
  Program P = lower_module(m, batch, n_data_inputs);
  out = program_json(P);
  *json = out.c_str();
  API_END
}

mr_status mr_calibrate(const char* text, const mr_exec_options* opts, int32_t n_weights, const mr_tensor* weights,
                       int32_t n_sets, const mr_tensor* inputs, int32_t k_min, int32_t k_max, int32_t* k_out,
                       int32_t* trials_out) {
  struct Flag {  // device overflow flag, freed on every exit path
    int32_t* p = nullptr;
    ~Flag() {
      if (p) cudaFree(p);
    }
  } flag_mem;
  API_BEGIN
  if (!text || !k_out || (n_sets > 0 && !inputs)) fail(MR_ERR_INVALID_ARGUMENT, "null argument");
  if (n_sets < 1) fail(MR_ERR_CALIBRATION_FAILED, "calibration requires a non-empty input set");
  mr_exec_options o;
  mr_exec_default_options(&o);
  if (opts) o = *opts;
  o.use_cuda_graph = 0;
  DeviceGuard dg(o.device);
  const Program P0 = lower_module(parse_fused_module(text), o.batch, o.n_data_inputs);
  if (!P0.any_quant) fail(MR_ERR_INVALID_ARGUMENT, "module has no quantize sites");
  CK(cudaMalloc(&flag_mem.p, sizeof(int32_t)));
  int32_t* flag = flag_mem.p;
  std::vector<float> out;
  for (int k = k_min; k <= k_max; ++k) {
    if (trials_out) *trials_out = k - k_min + 1;
    Program P = P0;
    rescale_sites(P, k);
    CK(cudaMemset(flag, 0, sizeof(int32_t)));
    g_calib_ovf = flag;  // every QDev of this trial reports overflow
    std::unique_ptr<Exec> ex;
    try {
      ex = make_exec(std::move(P), o, /*enforce_exact=*/false);  // overflow search only
      mr_exec_t h = reinterpret_cast<mr_exec_t>(ex.get());
      mr_status st = mr_exec_set_weights(h, n_weights, weights);  // weight sites
      if (st != MR_OK) throw Status{static_cast<int>(st), g_last_error};
      int32_t ovf = 0;
      CK(cudaMemcpy(&ovf, flag, sizeof(ovf), cudaMemcpyDeviceToHost));
      out.resize(static_cast<size_t>(ex->out_elems));
      mr_tensor res{};
      res.data = out.data();
      res.ndim = static_cast<int32_t>(ex->out_shape.size());
      for (int i = 0; i < res.ndim; ++i) res.shape[i] = ex->out_shape[i];
      res.type_code = MR_FLOAT;
      res.bits = 32;
      for (int32_t b = 0; b < n_sets && !ovf; ++b) {  // activation sites, one calibration batch at a time
        st = mr_exec_run_host(h, &inputs[b], &res, nullptr);
        if (st != MR_OK) throw Status{static_cast<int>(st), g_last_error};
        CK(cudaMemcpy(&ovf, flag, sizeof(ovf), cudaMemcpyDeviceToHost));
      }
      g_calib_ovf = nullptr;
      if (!ovf) {
        *k_out = k;
        return MR_OK;
      }
    } catch (...) {
      g_calib_ovf = nullptr;
      throw;
    }
  }
  fail(MR_ERR_CALIBRATION_FAILED, "no power-of-two scale in [2^" + std::to_string(k_min) + ", 2^" +
                                      std::to_string(k_max) + "] avoids overflow");
  API_END
}

struct mr_group_s {
  std::unique_ptr<Exec> ex;
  std::vector<int> perm;         // exec param k <- group operand perm[k]
  int n_data = 0;                // exec params 0..n_data-1 are activations
  int n_operands = 0;
  std::vector<const void*> staged;  // weight operand addresses of the last staging
};

mr_status mr_group_compile(const char* text, const char* group, const mr_exec_options* opts, mr_group_t* out) {
  API_BEGIN
  if (!text || !group || !out) fail(MR_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  mr_exec_options o;
  mr_exec_default_options(&o);
  if (opts) o = *opts;
  if (o.batch < 1) fail(MR_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  Module m = parse_fused_module(text);
  auto g = std::make_unique<mr_group_s>();
  GroupModule gm = extract_group_module(m, group, o.batch, o.n_data_inputs);
  g->perm = gm.perm;
  g->n_data = gm.n_data;
  int n_ops = 0;
  for (int p : g->perm) n_ops = std::max(n_ops, p + 1);
  g->n_operands = n_ops;
  Program gp = lower_module(gm.m, o.batch, g->n_data, &gm.coded);  // host-side errors before any device work
  gp.any_quant = gp.any_quant || gm.module_quant;  // same float format as inside the whole module
  DeviceGuard dg(o.device);
  mr_exec_options go = o;
  go.n_data_inputs = g->n_data;
  g->ex = make_exec(std::move(gp), go);
  *out = g.release();
  API_END
}

mr_status mr_group_signature(mr_group_t g, int32_t* n_operands, mr_tensor* out_shape) {
  API_BEGIN
  if (!g) fail(MR_ERR_INVALID_ARGUMENT, "null group");
  if (n_operands) *n_operands = g->n_operands;
  if (out_shape) {
    std::memset(out_shape, 0, sizeof(*out_shape));
    out_shape->ndim = static_cast<int32_t>(g->ex->out_shape.size());
    for (size_t i = 0; i < g->ex->out_shape.size(); ++i) out_shape->shape[i] = g->ex->out_shape[i];
    out_shape->type_code = MR_FLOAT;
    out_shape->bits = 32;
  }
  API_END
}

mr_status mr_group_launch(mr_group_t g, const mr_tensor* in, int32_t n_in, mr_tensor* out, void* stream) {
  API_BEGIN
  if (!g) fail(MR_ERR_INVALID_ARGUMENT, "null group");
  Exec& ex = *g->ex;
  if (n_in != g->n_operands)
    fail(MR_ERR_ARITY_MISMATCH, "function expects " + std::to_string(g->n_operands) + " arguments, got " +
                                    std::to_string(n_in));
  if (!in) fail(MR_ERR_INVALID_ARGUMENT, "null operands");
  DeviceGuard dg(ex.opt.device);
  std::vector<mr_tensor> ordered(g->perm.size());
  for (size_t k = 0; k < g->perm.size(); ++k) ordered[k] = in[g->perm[k]];
  std::vector<const void*> addrs;
  for (size_t k = static_cast<size_t>(g->n_data); k < ordered.size(); ++k) addrs.push_back(ordered[k].data);
  if (!ex.weights_ready || addrs != g->staged) {
    // weight staging is synchronous: order it after the caller's prior work
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    load_weights(ex, static_cast<int32_t>(ordered.size()) - g->n_data, ordered.data() + g->n_data,
                 cudaMemcpyDeviceToDevice);
    g->staged = addrs;
  }
  check_input(ex, ordered.data());
  if (!out || !out->data) fail(MR_ERR_INVALID_ARGUMENT, "null output");
  if (numel(*out) != ex.out_elems) fail(MR_ERR_TYPE_MISMATCH, "output size mismatch");
  check_device_output(ex, out);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  set_inputs(ex, ordered.data());
  OutRedirect r(ex, out->data);
  run_body(ex, s);
  API_END
}

void mr_group_reload(mr_group_t g) {
  if (g) g->staged.clear();
}

void mr_group_destroy(mr_group_t g) {
  if (!g) return;
  try {
    DeviceGuard dg(g->ex->opt.device);
    delete g;
  } catch (...) {
    delete g;
  }
}

const char* mr_build_info(void) { return MRB200_BUILD_INFO; }

}  // extern "C"
