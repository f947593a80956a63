// b200_backend.hpp -- the reference-side binding of the B200 executor: what a
// MicroRelay maintainer adds next to interp().  Compiled here
// against the UNMODIFIED reference headers (/root/reference/proj/core/include)
// and linked with the reference library and libmrb200.so by
// integration/Makefile; exercised by tests/test_integration.py.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "microrelay/interp.hpp"
#include "microrelay/value.hpp"
#include "mrb200.h"

namespace microrelay {

// interp(m, "main", args) (interp.hpp:50-51) on a fused ModuleEnv, executed by
// libmrb200: args[0] is the batch (?n bound from its shape), args[1..] the
// remaining @main params in order.  Errors surface as the reference's
// Diagnostic (DiagCode = mr_status - 1 for the mirrored codes, Internal for
// the backend's own).
ValueRef interp_b200(const ModuleEnv& fused, const std::vector<ValueRef>& args);

// A long-lived executor for a server loop: create + set_weights once, then
// run() per batch.  Same contract as interp_b200.
class B200Session {
 public:
  B200Session(const ModuleEnv& fused, int64_t batch, const std::vector<ValueRef>& weights, int device = 0);
  ~B200Session();
  B200Session(const B200Session&) = delete;
  B200Session& operator=(const B200Session&) = delete;
  ValueRef run(const ValueRef& batch);

 private:
  mr_exec_t ex_ = nullptr;
  std::vector<int64_t> out_dims_;
};

// The group level: one Primitive closure (interp.cpp:86-101) compiled by
// mr_group_compile and applied to host tensors (uploaded per call).  `group`
// is the %fusedN name (or the value its call binds).
class B200Group {
 public:
  B200Group(const ModuleEnv& fused, const std::string& group, int64_t batch, int device = 0);
  ~B200Group();
  B200Group(const B200Group&) = delete;
  B200Group& operator=(const B200Group&) = delete;
  int arity() const { return n_operands_; }
  ValueRef apply(const std::vector<ValueRef>& args);

 private:
  mr_group_t g_ = nullptr;
  int n_operands_ = 0;
  std::vector<int64_t> out_dims_;
};

}  // namespace microrelay
