// lower.cpp -- see lower.hpp.
#include "lower.hpp"

#include <algorithm>
#include <map>
#include <set>
#include <sstream>

#include "../../include/mrb200.h"

namespace mrb200 {

namespace {

[[noreturn]] void unsupported(const std::string& group, const std::string& why) {
  throw LowerError{MR_ERR_UNSUPPORTED_GROUP, "group %" + group + ": " + why};
}

[[noreturn]] void bad(int code, const std::string& why) { throw LowerError{code, why}; }

bool is_call(const ExprP& e, const char* op) {
  return e && e->kind == Expr::Call && !e->callee_is_var && e->name == op;
}

bool scalar_const(const ExprP& e, float* v) {
  if (!e || e->kind != Expr::Const) return false;
  int64_t n = 1;
  for (auto d : e->lit.shape) n *= d;
  if (n != 1 || e->lit.dtype != "float32") return false;
  *v = static_cast<float>(e->lit.values[0]);
  return true;
}

// One group body in analysable form.
struct Body {
  std::string group;
  std::map<std::string, ExprP> let_of;      // let var -> bound call
  std::vector<std::string> order;           // let vars in binding order
  std::string result;                       // var holding the group result
  std::map<std::string, int> param_value;   // fn param -> @main value
  std::set<std::string> visited;
};

// Follows `e` back to a source (fn param or constant), returning the unary
// chain of calls applied on the way, outermost last.
struct Traced {
  int value = -1;               // @main value when the source is a param
  const Literal* lit = nullptr; // constant source
  std::vector<ExprP> chain;     // calls from source to the consumer
};

// Index of the argument carrying the chain (the non-constant one).
int chain_arg(const Body& b, const ExprP& call) {
  int idx = -1;
  for (size_t i = 0; i < call->args.size(); ++i) {
    if (call->args[i]->kind == Expr::Const) continue;
    if (idx >= 0) unsupported(b.group, "operator " + call->name + " has two non-constant operands in a prologue");
    idx = static_cast<int>(i);
  }
  if (idx < 0) unsupported(b.group, "operator " + call->name + " on constants only (run fold)");
  return idx;
}

Traced trace(Body& b, ExprP e) {
  Traced t;
  std::vector<ExprP> rev;
  for (;;) {
    if (e->kind == Expr::Const) {
      t.lit = &e->lit;
      break;
    }
    if (e->kind == Expr::Var) {
      auto pv = b.param_value.find(e->name);
      if (pv != b.param_value.end()) {
        t.value = pv->second;
        break;
      }
      auto it = b.let_of.find(e->name);
      if (it == b.let_of.end()) unsupported(b.group, "unbound %" + e->name);
      if (b.visited.count(e->name)) unsupported(b.group, "%" + e->name + " used twice inside the group");
      b.visited.insert(e->name);
      e = it->second;
      continue;
    }
    if (e->kind == Expr::Call && !e->callee_is_var) {
      rev.push_back(e);
      e = e->args[chain_arg(b, e)];
      continue;
    }
    unsupported(b.group, "unsupported expression in a prologue");
  }
  t.chain.assign(rev.rbegin(), rev.rend());
  return t;
}

// Matches the realize chain at chain[i..i+5]; fills q.
bool match_requant(const std::vector<ExprP>& ch, size_t i, QParams* q) {
  if (i + 6 > ch.size()) return false;
  float c1, c2;
  if (!is_call(ch[i], "multiply") || ch[i]->args.size() != 2) return false;
  if (!scalar_const(ch[i]->args[1], &c1) && !scalar_const(ch[i]->args[0], &c1)) return false;
  if (!is_call(ch[i + 1], "round")) return false;
  if (!is_call(ch[i + 2], "clip")) return false;
  if (!is_call(ch[i + 3], "cast")) return false;
  std::string qt = attr_str(ch[i + 3]->attrs, "dtype", "");
  if (qt != "int8" && qt != "uint8") return false;
  if (!is_call(ch[i + 4], "cast") || attr_str(ch[i + 4]->attrs, "dtype", "") != "float32") return false;
  if (!is_call(ch[i + 5], "multiply") || ch[i + 5]->args.size() != 2) return false;
  if (!scalar_const(ch[i + 5]->args[1], &c2) && !scalar_const(ch[i + 5]->args[0], &c2)) return false;
  q->c1 = c1;
  q->c2 = c2;
  // clip's float path: std::min(std::max(x, (float)lo), (float)hi) kernels.cpp:306-307
  q->lo = static_cast<float>(attr_float(ch[i + 2]->attrs, "a_min", -128));
  q->hi = static_cast<float>(attr_float(ch[i + 2]->attrs, "a_max", 127));
  q->is_signed = qt == "int8";
  return true;
}

int64_t out_dim(int64_t in, int64_t k, int64_t s, int64_t p) { return (in - k + 2 * p) / s + 1; }

// transpose(x, axes=perm): the layout pass's relabelings (passes.cpp:481-486,
// rewrites.cpp:440-467) are data movement only; physical layouts here do not
// depend on the logical axis order, so they are folded away during lowering.
bool is_transpose(const ExprP& e, std::initializer_list<int64_t> perm) {
  return is_call(e, "transpose") && attr_ints(e->attrs, "axes", {}) == std::vector<int64_t>(perm);
}

}  // namespace

Program lower_module(const Module& m0, int64_t batch, int n_data_inputs,
                     const std::map<std::string, QParams>* coded_inputs) {
  // combine-conv's weight tuples / split groups -> plain conv groups (combine.cpp)
  Module m = m0;
  m.body = std::make_shared<Block>(*m0.body);
  for (const auto& [n, v] : m.body->lets)
    if (v->kind == Expr::Tuple || v->kind == Expr::Proj) {
      try {
        normalize_combined(m);
      } catch (const ParseError& e) {
        bad(MR_ERR_UNSUPPORTED_GROUP, e.msg);
      }
      break;
    }
  Program P;
  std::map<std::string, int> value_of;
  auto add_value = [&](const std::string& name) {
    if (value_of.count(name)) bad(MR_ERR_SYNTAX, "duplicate binding %" + name);
    ValueInfo v;
    v.name = name;
    P.values.push_back(v);
    value_of[name] = static_cast<int>(P.values.size()) - 1;
    return static_cast<int>(P.values.size()) - 1;
  };

  if (n_data_inputs < 0 || n_data_inputs > static_cast<int>(m.params.size()))
    bad(MR_ERR_INVALID_ARGUMENT, "n_data_inputs out of range");
  for (size_t i = 0; i < m.params.size(); ++i) {
    const auto& mp = m.params[i];
    int v = add_value(mp.name);
    P.values[v].param_index = static_cast<int>(i);
    P.values[v].is_data = static_cast<int>(i) < n_data_inputs;
    if (mp.type.dtype != "float32")
      bad(MR_ERR_TYPE_MISMATCH, "@main parameter %" + mp.name + " is " + mp.type.dtype + "; only float32 is supported");
    for (const auto& d : mp.type.dims) P.values[v].shape.push_back(d.symbolic ? batch : d.value);
    if (coded_inputs && coded_inputs->count(mp.name)) {
      if (!P.values[v].is_data) bad(MR_ERR_INVALID_ARGUMENT, "coded input %" + mp.name + " is not a data input");
      P.values[v].quantized = true;
      P.values[v].q = coded_inputs->at(mp.name);
      P.any_quant = true;
    }
  }
  P.n_params = static_cast<int>(m.params.size());

  std::map<std::string, ExprP> fns;
  auto handle_call = [&](const std::string& out, const ExprP& call) {
    if (!(call->kind == Expr::Call && call->callee_is_var))
      bad(MR_ERR_UNSUPPORTED_GROUP, "@main binding %" + out + " is not a call of a Primitive function (run fuse)");
    auto f = fns.find(call->name);
    if (f == fns.end()) bad(MR_ERR_UNBOUND_VARIABLE, "%" + call->name + " is not a let-bound function");
    const ExprP& fn = f->second;
    if (fn->params.size() != call->args.size())
      bad(MR_ERR_ARITY_MISMATCH, "%" + call->name + " arity mismatch");
    GroupDesc g;
    g.name = call->name;
    g.out_name = out;
    Body b;
    b.group = call->name;
    for (size_t i = 0; i < call->args.size(); ++i) {
      const ExprP& a = call->args[i];
      if (a->kind != Expr::Var || !value_of.count(a->name))
        bad(MR_ERR_UNSUPPORTED_GROUP, "argument " + std::to_string(i) + " of %" + call->name + " is not a bound @main value");
      int v = value_of[a->name];
      b.param_value[fn->params[i]] = v;
      g.param_values.push_back(v);
    }
    for (const auto& [name, e] : fn->body->lets) {
      b.let_of[name] = e;
      b.order.push_back(name);
    }
    if (fn->body->result->kind == Expr::Var) {
      b.result = fn->body->result->name;
    } else {
      b.result = "__result__";
      b.let_of[b.result] = fn->body->result;
      b.order.push_back(b.result);
    }
    // anchor
    std::string anchor;
    for (const auto& name : b.order) {
      const ExprP& e = b.let_of[name];
      if (e->kind != Expr::Call || e->callee_is_var) unsupported(g.name, "non-operator binding %" + name);
      if (e->name == "conv2d" || e->name == "dense" || e->name == "max_pool2d" ||
          e->name == "depthwise_conv2d") {
        if (!anchor.empty()) unsupported(g.name, "two contraction/pool operators in one group");
        anchor = name;
      }
    }
    if (anchor.empty()) unsupported(g.name, "no conv2d/dense/max_pool2d anchor (elementwise-only groups are not lowered yet)");
    const ExprP& A = b.let_of[anchor];
    b.visited.insert(anchor);
    const ValueInfo* data_vi = nullptr;
    bool data_nhwc = false, weight_hwio = false, anchor_nhwc = false;  // layout-pass relabels

    // ---- prologues ----
    auto data_operand = [&](const ExprP& arg) {
      Traced t = trace(b, arg);
      if (t.value < 0) unsupported(g.name, "constant data operand");
      g.data.value = t.value;
      data_nhwc = P.values[t.value].nhwc_view;
      for (size_t k = 0; k < t.chain.size();) {  // NCHW -> NHWC relabels commute with the realize chain
        if (is_transpose(t.chain[k], {0, 2, 3, 1})) {
          if (data_nhwc) unsupported(g.name, "transpose of an NHWC value");
          data_nhwc = true;
          t.chain.erase(t.chain.begin() + static_cast<long>(k));
        } else {
          ++k;
        }
      }
      size_t i = 0;
      float s;
      if (i < t.chain.size() && is_call(t.chain[i], "multiply") && !match_requant(t.chain, i, &g.data.q) &&
          (scalar_const(t.chain[i]->args[1], &s) || scalar_const(t.chain[i]->args[0], &s))) {
        g.data.pre_mul = s;
        ++i;
      }
      if (i < t.chain.size()) {
        if (!match_requant(t.chain, i, &g.data.q)) unsupported(g.name, "data prologue is not a quantize chain (op " + t.chain[i]->name + ")");
        g.data.quant = true;
        i += 6;
      }
      if (i != t.chain.size()) unsupported(g.name, "trailing ops in the data prologue");
      data_vi = &P.values[t.value];
    };
    auto weight_operand = [&](const ExprP& arg) {
      Traced t = trace(b, arg);
      g.weight.value = t.value;
      if (t.value >= 0) {
        if (P.values[t.value].producer >= 0 || P.values[t.value].is_data)
          unsupported(g.name, "weight operand must be a @main weight parameter");
        g.weight.shape = P.values[t.value].shape;
      } else {
        g.weight.constant = t.lit->f32();
        g.weight.shape = t.lit->shape;
      }
      weight_hwio = false;
      for (size_t k = 0; k < t.chain.size();) {  // OIHW -> HWIO relabel (NHWC conv weights)
        if (is_transpose(t.chain[k], {2, 3, 1, 0})) {
          weight_hwio = true;
          t.chain.erase(t.chain.begin() + static_cast<long>(k));
        } else {
          ++k;
        }
      }
      size_t i = 0;
      while (i < t.chain.size() && is_call(t.chain[i], "multiply") && !match_requant(t.chain, i, &g.weight.q)) {
        const ExprP& c = t.chain[i]->args[0]->kind == Expr::Const ? t.chain[i]->args[0] : t.chain[i]->args[1];
        float s;
        if (scalar_const(c, &s)) {
          if (g.weight.scalar_scale != 0.f || !g.weight.oc_scale.empty()) unsupported(g.name, "two weight scales");
          g.weight.scalar_scale = s;
        } else {
          // fold-scale post-conv rule: const [OC,1,1,1] (rewrites.cpp:186-211)
          const auto& L = c->lit;
          int64_t n = 1;
          for (auto d : L.shape) n *= d;
          bool ok = !L.shape.empty() && L.shape[0] == g.weight.shape[0] && n == L.shape[0];
          if (!ok || !g.weight.oc_scale.empty() || g.weight.scalar_scale != 0.f)
            unsupported(g.name, "weight prologue multiply is not a per-output-channel constant");
          g.weight.oc_scale = L.f32();
        }
        ++i;
      }
      if (i < t.chain.size()) {
        if (!match_requant(t.chain, i, &g.weight.q)) unsupported(g.name, "weight prologue op " + t.chain[i]->name + " not supported");
        g.weight.quant = true;
        i += 6;
      }
      if (i != t.chain.size()) unsupported(g.name, "trailing ops in the weight prologue");
    };

    const std::string& op = A->name;
    if (op == "conv2d" || op == "depthwise_conv2d") {
      g.kind = op == "conv2d" ? GroupKind::Conv : GroupKind::DwConv;
      const std::string lay = attr_str(A->attrs, "layout", "NCHW");
      if (lay != "NCHW" && !(lay == "NHWC" && op == "conv2d")) unsupported(g.name, "conv2d layout " + lay);
      anchor_nhwc = lay == "NHWC";
      size_t want = op == "conv2d" ? 2 : 3;
      if (A->args.size() != want) unsupported(g.name, op + " arity");
      data_operand(A->args[0]);
      if (data_nhwc != anchor_nhwc) unsupported(g.name, "conv2d data layout does not match its layout attribute");
      if (op == "depthwise_conv2d") {
        Traced win = trace(b, A->args[1]);
        if (win.value < 0 || !win.chain.empty()) unsupported(g.name, "window operand");
        g.window_value = win.value;
      }
      weight_operand(A->args.back());
      if (weight_hwio != anchor_nhwc) unsupported(g.name, "conv2d weight layout does not match its layout attribute");
      auto st = attr_ints(A->attrs, "strides", {1, 1});
      auto pd = attr_ints(A->attrs, "padding", {0, 0});
      if (st.size() != 2 || pd.size() != 2) unsupported(g.name, "strides/padding");
      g.sh = st[0]; g.sw = st[1]; g.ph = pd[0]; g.pw = pd[1];
      const auto& ws = g.weight.shape;
      const auto& xs = data_vi->shape;
      if (ws.size() != 4 || xs.size() != 4) bad(MR_ERR_TYPE_MISMATCH, g.name + ": conv2d needs rank-4 data and weight");
      if (g.kind == GroupKind::Conv && ws[1] != xs[1]) bad(MR_ERR_TYPE_MISMATCH, g.name + ": channel mismatch");
      if (g.kind == GroupKind::DwConv && (ws[0] != xs[1] || ws[1] != 1)) bad(MR_ERR_TYPE_MISMATCH, g.name + ": depthwise weight must be [C,1,KH,KW]");
      g.kh = ws[2]; g.kw = ws[3];
      g.in_shape = xs;
      g.out_shape = {xs[0], ws[0], out_dim(xs[2], g.kh, g.sh, g.ph), out_dim(xs[3], g.kw, g.sw, g.pw)};
    } else if (op == "max_pool2d") {
      g.kind = GroupKind::MaxPool;
      if (A->args.size() != 2) unsupported(g.name, "max_pool2d arity");
      data_operand(A->args[0]);
      if (g.data.quant || g.data.pre_mul != 0.f) unsupported(g.name, "prologue on a pooling input");
      Traced win = trace(b, A->args[1]);
      if (win.value < 0 || !win.chain.empty()) unsupported(g.name, "pooling window operand");
      g.window_value = win.value;
      const auto& ws = P.values[win.value].shape;
      const auto& xs = data_vi->shape;
      if (ws.size() != 4 || xs.size() != 4 || ws[1] != xs[1]) bad(MR_ERR_TYPE_MISMATCH, g.name + ": max_pool2d window");
      auto st = attr_ints(A->attrs, "strides", {1, 1});
      auto pd = attr_ints(A->attrs, "padding", {0, 0});
      g.sh = st[0]; g.sw = st[1]; g.ph = pd[0]; g.pw = pd[1];
      g.kh = ws[2]; g.kw = ws[3];
      g.in_shape = xs;
      g.out_shape = {xs[0], ws[0], out_dim(xs[2], g.kh, g.sh, g.ph), out_dim(xs[3], g.kw, g.sw, g.pw)};
    } else {  // dense
      g.kind = GroupKind::Dense;
      if (A->args.size() != 2) unsupported(g.name, "dense arity");
      data_operand(A->args[0]);
      weight_operand(A->args[1]);
      const auto& xs = data_vi->shape;
      const auto& ws = g.weight.shape;
      if (xs.size() != 2 || ws.size() != 2 || xs[1] != ws[1]) bad(MR_ERR_TYPE_MISMATCH, g.name + ": dense shapes");
      g.in_shape = xs;
      g.out_shape = {xs[0], ws[0]};
    }
    // A data operand is integer-coded either by its own realize chain or
    // because its producer's epilogue ended in one (value == code * c2).
    bool data_coded = g.data.quant || (data_vi->quantized && g.data.pre_mul == 0.f);
    if (g.kind != GroupKind::MaxPool && data_coded != g.weight.quant)
      unsupported(g.name, "only one contraction operand is quantized");

    // ---- epilogue: follow the single consumer chain from the anchor ----
    std::vector<ExprP> epi_calls;
    std::vector<int> epi_chain_pos;
    std::string cur = anchor;
    while (cur != b.result) {
      std::string next_var;
      for (const auto& name : b.order) {
        const ExprP& e = b.let_of[name];
        for (size_t i = 0; i < e->args.size(); ++i) {
          if (e->args[i]->kind == Expr::Var && e->args[i]->name == cur) {
            if (!next_var.empty() && next_var != name) unsupported(g.name, "anchor value has two consumers");
            next_var = name;
            epi_chain_pos.resize(epi_calls.size() + 1);
            epi_chain_pos[epi_calls.size()] = static_cast<int>(i);
          }
        }
      }
      if (next_var.empty()) unsupported(g.name, "epilogue does not reach the group result");
      if (b.visited.count(next_var)) unsupported(g.name, "epilogue revisits %" + next_var);
      b.visited.insert(next_var);
      epi_calls.push_back(b.let_of[next_var]);
      cur = next_var;
    }
    std::vector<int64_t> shape = g.out_shape;
    int64_t C = shape.size() >= 2 ? shape[1] : 1;
    bool back_to_nchw = false, out_nhwc = false;
    if (g.kind != GroupKind::Conv && data_nhwc) unsupported(g.name, op + " over an NHWC value");
    for (size_t i = 0; i < epi_calls.size();) {
      QParams q;
      if (match_requant(epi_calls, i, &q)) {
        EpiOp e{EpiKind::Requant};
        e.q = q;
        g.epi.push_back(e);
        i += 6;
        continue;
      }
      const ExprP& c = epi_calls[i];
      int pos = epi_chain_pos[i];
      if (c->callee_is_var) unsupported(g.name, "call in epilogue");
      const std::string& o = c->name;
      if (!g.epi.empty() && g.epi.back().kind == EpiKind::SumHW) unsupported(g.name, "ops after sum");
      if (o == "transpose") {
        if (anchor_nhwc && !back_to_nchw && g.epi.empty() && is_transpose(c, {0, 3, 1, 2})) {
          back_to_nchw = true;  // NHWC conv result back to NCHW: a relabel
        } else if (!out_nhwc && (!anchor_nhwc || back_to_nchw) && is_transpose(c, {0, 2, 3, 1}) && shape.size() == 4) {
          out_nhwc = true;  // the value is handed to NHWC consumers: a relabel
        } else {
          unsupported(g.name, "transpose in the epilogue");
        }
        ++i;
        continue;
      }
      if (anchor_nhwc && !back_to_nchw) unsupported(g.name, "epilogue op on the NHWC conv result");
      if (out_nhwc) unsupported(g.name, "op after the NHWC relabel (only a realize chain may follow)");
      // after a flatten only the realize chain of the consumer's input (matched above; run by
      // the flatten tail) may follow
      for (const auto& e : g.epi)
        if (e.kind == EpiKind::Flatten) unsupported(g.name, "ops after reshape");
      auto other = [&]() -> ExprP {
        if (c->args.size() != 2) unsupported(g.name, o + " arity");
        return c->args[1 - pos];
      };
      if (o == "relu") {
        g.epi.push_back(EpiOp{EpiKind::Relu});
      } else if (o == "clip") {
        EpiOp e{EpiKind::Clip};
        e.lo = static_cast<float>(attr_float(c->attrs, "a_min", 0));
        e.hi = static_cast<float>(attr_float(c->attrs, "a_max", 0));
        g.epi.push_back(e);
      } else if (o == "bias_add") {
        if (pos != 0) unsupported(g.name, "bias_add with the chain as bias");
        if (attr_int(c->attrs, "axis", 1) != 1) unsupported(g.name, "bias_add axis != 1");
        ExprP bexp = other();
        if (bexp->kind != Expr::Var || !b.param_value.count(bexp->name)) unsupported(g.name, "bias must be a parameter");
        EpiOp e{EpiKind::Bias};
        e.value = b.param_value[bexp->name];
        if (P.values[e.value].shape != std::vector<int64_t>{C}) bad(MR_ERR_TYPE_MISMATCH, g.name + ": bias shape");
        g.epi.push_back(e);
      } else if (o == "add") {
        ExprP r = other();
        if (r->kind != Expr::Var || !b.param_value.count(r->name)) unsupported(g.name, "add operand must be a parameter");
        EpiOp e{EpiKind::Residual};
        e.value = b.param_value[r->name];
        if (P.values[e.value].shape != shape) unsupported(g.name, "broadcasting add in epilogue");
        if (P.values[e.value].nhwc_view) unsupported(g.name, "residual operand is NHWC-relabelled");
        g.epi.push_back(e);
      } else if (o == "multiply") {
        ExprP k = other();
        float s;
        if (scalar_const(k, &s)) {
          EpiOp e{EpiKind::MulScalar};
          e.s = s;
          g.epi.push_back(e);
        } else if (k->kind == Expr::Const) {
          const auto& L = k->lit;
          int64_t n = 1;
          for (auto d : L.shape) n *= d;
          // [C,1,1] or [1,C,1,1] broadcast over NCHW
          bool ok = n == C && !L.shape.empty() && shape.size() == 4;
          if (ok) {
            size_t r = L.shape.size();
            ok = (r == 3 && L.shape[0] == C) || (r == 4 && L.shape[0] == 1 && L.shape[1] == C);
          }
          if (!ok) unsupported(g.name, "multiply by a non per-channel constant in epilogue");
          EpiOp e{EpiKind::MulChannel};
          e.vec = L.f32();
          g.epi.push_back(e);
        } else {
          unsupported(g.name, "multiply by a non-constant in epilogue");
        }
      } else if (o == "sum") {
        auto ax = attr_ints(c->attrs, "axis", {});
        if (ax != std::vector<int64_t>{2, 3} || attr_int(c->attrs, "keepdims", 0) != 0 || shape.size() != 4)
          unsupported(g.name, "only sum(axis=(2,3)) is fused");
        g.pre_sum_shape = shape;
        shape = {shape[0], shape[1]};
        g.epi.push_back(EpiOp{EpiKind::SumHW});
      } else if (o == "reshape") {
        // the flatten a classifier head needs: [N,C,H,W] -> [N, C*H*W] (row-major view)
        auto ns = attr_ints(c->attrs, "newshape", {});
        if (shape.size() != 4 || ns.size() != 2 || ns[0] != shape[0] || ns[1] != shape[1] * shape[2] * shape[3])
          unsupported(g.name, "only the [N,C,H,W] -> [N,C*H*W] reshape is fused");
        if (!g.epi.empty() && g.epi.back().kind == EpiKind::Requant)
          unsupported(g.name, "reshape of realize codes");
        g.pre_sum_shape = shape;
        shape = {ns[0], ns[1]};
        g.epi.push_back(EpiOp{EpiKind::Flatten});
      } else {
        unsupported(g.name, "epilogue operator " + o);
      }
      ++i;
    }
    g.out_shape = shape;
    for (const auto& name : b.order)
      if (!b.visited.count(name)) unsupported(g.name, "binding %" + name + " is outside the prologue/anchor/epilogue pattern");

    if (anchor_nhwc && !back_to_nchw) unsupported(g.name, "NHWC conv result never returns to NCHW");
    int ov = add_value(out);
    int gi = static_cast<int>(P.groups.size());
    P.values[ov].producer = gi;
    P.values[ov].shape = g.out_shape;
    P.values[ov].nhwc_view = out_nhwc;
    if (!g.epi.empty() && g.epi.back().kind == EpiKind::Requant) {
      P.values[ov].quantized = true;
      P.values[ov].q = g.epi.back().q;
    }
    g.out_value = ov;
    if (g.data.quant || g.weight.quant) P.any_quant = true;
    for (int v : g.param_values) {
      auto& cs = P.values[v].consumers;
      if (std::find(cs.begin(), cs.end(), gi) == cs.end()) cs.push_back(gi);
    }
    P.groups.push_back(std::move(g));
  };

  for (const auto& [name, e] : m.body->lets) {
    if (e->kind == Expr::Fn) {
      if (!e->primitive) bad(MR_ERR_UNSUPPORTED_GROUP, "%" + name + " is a non-Primitive function");
      fns[name] = e;
      continue;
    }
    if (e->kind == Expr::Const) {  // an embedded weight: hidden parameter
      if (e->lit.dtype != "float32") bad(MR_ERR_TYPE_MISMATCH, "@main constant %" + name + " is not float32");
      const int v = add_value(name);
      P.values[v].shape = e->lit.shape;
      P.values[v].hidden = static_cast<int>(P.hidden_data.size());
      P.values[v].param_index = P.n_params++;
      P.hidden_data.push_back(e->lit.f32());
      continue;
    }
    handle_call(name, e);
  }
  const ExprP& res = m.body->result;
  if (res->kind == Expr::Var) {
    if (!value_of.count(res->name)) bad(MR_ERR_UNBOUND_VARIABLE, "result %" + res->name);
    P.result_value = value_of[res->name];
  } else {
    handle_call("__result__", res);
    P.result_value = value_of["__result__"];
  }
  P.values[P.result_value].is_result = true;
  if (P.values[P.result_value].nhwc_view) unsupported("@main", "an NHWC-relabelled result");
  if (P.groups.empty()) bad(MR_ERR_UNSUPPORTED_GROUP, "module has no Primitive group");
  return P;
}

GroupModule extract_group_module(const Module& m, const std::string& group, int64_t batch, int n_data_inputs) {
  GroupModule out;
  std::vector<int>* perm = &out.perm;
  std::map<std::string, QParams>* coded = &out.coded;
  const Program P = lower_module(m, batch, n_data_inputs);  // validates the module, binds the shapes
  std::map<std::string, int> value_of;
  for (size_t v = 0; v < P.values.size(); ++v) value_of[P.values[v].name] = static_cast<int>(v);
  std::string key = group;
  if (!key.empty() && key[0] == '%') key = key.substr(1);
  std::map<std::string, ExprP> fns;
  std::string fn_name, out_name;
  ExprP call;
  for (const auto& [name, e] : m.body->lets) {
    if (e->kind == Expr::Fn) {
      fns[name] = e;
    } else if (e->kind == Expr::Call && e->callee_is_var && (e->name == key || name == key)) {
      fn_name = e->name;
      out_name = name;
      call = e;
    }
  }
  if (!call && m.body->result->kind == Expr::Call && m.body->result->name == key) {
    fn_name = key;
    out_name = "__result__";
    call = m.body->result;
  }
  if (!call || !fns.count(fn_name)) bad(MR_ERR_UNBOUND_VARIABLE, "no Primitive group %" + key + " in @main");
  const ExprP fn = fns[fn_name];
  std::vector<std::string> data_args, weight_args;
  std::map<std::string, int> first_pos;
  for (size_t i = 0; i < call->args.size(); ++i) {
    const std::string& a = call->args[i]->name;
    if (first_pos.count(a)) continue;
    first_pos[a] = static_cast<int>(i);
    const ValueInfo& vi = P.values[value_of.at(a)];
    if (vi.nhwc_view) unsupported(fn_name, "group-level call on an NHWC-relabelled operand %" + a);
    (vi.producer >= 0 || vi.is_data ? data_args : weight_args).push_back(a);
    if (vi.quantized) {
      // the caller hands code * c2 as float32; the group re-derives the codes
      // with the producer's chain, exact when c1 * c2 == 1 (power-of-two scales)
      if (!(vi.q.c1 * vi.q.c2 == 1.f)) unsupported(fn_name, "coded operand %" + a + " with c1 * c2 != 1");
      (*coded)[a] = vi.q;
    }
  }
  if (data_args.empty()) unsupported(fn_name, "group has no activation operand");
  out.module_quant = P.any_quant;
  Module& g = out.m;
  for (const auto* list : {&data_args, &weight_args}) {
    for (const auto& a : *list) {
      MainParam mp;
      mp.name = a;
      for (int64_t d : P.values[value_of.at(a)].shape) {
        Dim dim;
        dim.value = d;
        mp.type.dims.push_back(dim);
      }
      g.params.push_back(mp);
      perm->push_back(first_pos[a]);
    }
  }
  out.n_data = static_cast<int>(data_args.size());
  g.body = std::make_shared<Block>();
  g.body->lets.emplace_back(fn_name, fn);
  const std::string res = out_name == "__result__" ? "__group_result__" : out_name;
  g.body->lets.emplace_back(res, call);
  auto rv = std::make_shared<Expr>();
  rv->kind = Expr::Var;
  rv->name = res;
  g.body->result = rv;
  return out;
}

std::string describe_group(const Program& p, const GroupDesc& g) {
  std::ostringstream os;
  static const char* kinds[] = {"conv2d", "dense", "max_pool2d", "depthwise_conv2d"};
  os << "%" << g.name << ": " << kinds[static_cast<int>(g.kind)] << "(";
  os << "%" << p.values[g.data.value].name;
  if (g.data.pre_mul != 0.f) os << "*" << g.data.pre_mul;
  if (g.data.quant) os << " Q[" << g.data.q.c1 << "," << g.data.q.c2 << "]";
  if (g.kind != GroupKind::MaxPool) {
    os << ", w";
    if (!g.weight.oc_scale.empty()) os << "*gamma";
    if (g.weight.quant) os << " Q[" << g.weight.q.c1 << "," << g.weight.q.c2 << "]";
  }
  os << ")";
  static const char* names[] = {"", "mul", "mulc", "bias", "add", "relu", "Q", "clip", "sum", "flatten"};
  for (const auto& e : g.epi) os << " -> " << names[static_cast<int>(e.kind)];
  return os.str();
}

}  // namespace mrb200
