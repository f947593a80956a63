// combine.cpp -- the reference's combine-conv output (rewrites.cpp:276-401),
// resolved back into plain fused conv groups before lowering.
//
// combine_parallel_conv2d merges convs over one input with equal in-channels,
// kernel and attributes into
//     let %t  = (%w1, %w2, ...);                         // weight tuple
//     %fusedG = fn(%t, %x) { let %c = concat(%t, axis=0); conv2d(%x, %c, ...) }
//     %fusedS = fn(%y) { split(%y, axis=1, indices=(...)) }   // Opaque: its own group
//     let %v1 = %s.0;  let %v2 = %s.1; ...
// and because split is Opaque (registry.cpp:696) FuseOps leaves every op that
// used to follow a member conv in the CONSUMER group -- bias_add / relu ahead
// of the next conv, or anchorless groups like add(bias_add(%v1), bias_add(%v2))
// -> relu -> sum.
//
// Each output channel of a conv depends only on its own weight row, so the
// combined conv + split is bit-identical to one conv per tuple element on the
// same input ("output slicing at plan time").  normalize_combined rebuilds
// that module:
//   1. slice: one group per tuple element (its weight prologue, e.g. the
//      realize chain on the concatenated weight, is elementwise and moves with
//      the slice), bound directly to the projection's name;
//   2. re-fuse: the consumer's leading elementwise chain on a slice output
//      (bias_add with a parameter vector, relu, clip, multiply by a constant,
//      a trailing sum(axis=(2,3))) moves into the slice group's epilogue, in
//      the same order -- what FuseOps would have built without the split;
//   3. residual: an anchorless consumer that starts with add(%a, %b) of two
//      slice outputs is appended to the later producer, add becoming its
//      residual (float add is commutative: the same bits).
// Anything else left over fails loudly (ParseError -> MR_ERR_SYNTAX class at
// create), never a silent fallback.
#include <algorithm>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "relay_text.hpp"

namespace mrb200 {
namespace {

[[noreturn]] void fail(const std::string& m) { throw ParseError{"combine-conv: " + m}; }

bool is_op(const ExprP& e, const char* op) { return e && e->kind == Expr::Call && !e->callee_is_var && e->name == op; }
bool is_var(const ExprP& e, const std::string& n) { return e && e->kind == Expr::Var && e->name == n; }

ExprP var(const std::string& n) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Var;
  e->name = n;
  return e;
}

// Uses of %name in e (not descending into nested functions: Primitive groups
// are closed over their parameters).
int count_uses(const ExprP& e, const std::string& name) {
  if (!e) return 0;
  if (e->kind == Expr::Var) return e->name == name ? 1 : 0;
  if (e->kind == Expr::Fn) return 0;
  int n = (e->kind == Expr::Call && e->callee_is_var && e->name == name) ? 1 : 0;
  for (const auto& a : e->args) n += count_uses(a, name);
  return n;
}

int count_uses(const Block& b, const std::string& name) {
  int n = count_uses(b.result, name);
  for (const auto& [k, v] : b.lets) n += count_uses(v, name);
  return n;
}

// e with every %from replaced by %to (in place; nested functions untouched).
void rename(const ExprP& e, const std::string& from, const std::string& to) {
  if (!e || e->kind == Expr::Fn) return;
  if (e->kind == Expr::Var && e->name == from) e->name = to;
  if (e->kind == Expr::Call && e->callee_is_var && e->name == from) e->name = to;
  for (const auto& a : e->args) rename(a, from, to);
}

ExprP clone(const ExprP& e) {
  if (!e) return e;
  auto c = std::make_shared<Expr>(*e);
  for (auto& a : c->args) a = clone(a);
  if (e->body) {
    c->body = std::make_shared<Block>(*e->body);
    for (auto& [k, v] : c->body->lets) v = clone(v);
    c->body->result = clone(e->body->result);
  }
  return c;
}

struct Main {
  Block& b;
  int find_let(const std::string& name) const {
    for (size_t i = 0; i < b.lets.size(); ++i)
      if (b.lets[i].first == name) return static_cast<int>(i);
    return -1;
  }
  int uses(const std::string& name) const { return count_uses(b, name); }
  // the call let whose argument list contains %name (the single consumer)
  int consumer(const std::string& name) const {
    for (size_t i = 0; i < b.lets.size(); ++i)
      if (b.lets[i].second->kind == Expr::Call && b.lets[i].second->callee_is_var && count_uses(b.lets[i].second, name))
        return static_cast<int>(i);
    return -1;
  }
  ExprP fn_of(const ExprP& call) const {
    int i = find_let(call->name);
    return i >= 0 && b.lets[i].second->kind == Expr::Fn ? b.lets[i].second : nullptr;
  }
  void erase(const std::string& name) {
    int i = find_let(name);
    if (i >= 0) b.lets.erase(b.lets.begin() + i);
  }
};

std::string fresh(const Main& M, const std::string& base) {
  for (int k = 0;; ++k) {
    std::string n = base + "_" + std::to_string(k);
    if (M.find_let(n) < 0) return n;
  }
}

bool elementwise_link(const ExprP& e) {
  return is_op(e, "bias_add") || is_op(e, "relu") || is_op(e, "clip") ||
         (is_op(e, "multiply") && e->args.size() == 2 && e->args[1]->kind == Expr::Const);
}

// Step 2: move the consumer's chain on `param` (bound to the slice output) into the
// slice group.  Returns true if the consumer group became empty and was removed.
bool refuse_chain(Main& M, const std::string& slice_out) {
  if (M.uses(slice_out) != 1) return false;
  const int ci = M.consumer(slice_out);
  if (ci < 0) return false;
  ExprP ccall = M.b.lets[ci].second;
  ExprP cfn = M.fn_of(ccall);
  if (!cfn) return false;
  const int si = M.find_let(slice_out);
  ExprP scall = M.b.lets[si].second;
  ExprP sfn = M.fn_of(scall);
  if (!sfn) return false;
  int pi = -1;
  for (size_t k = 0; k < ccall->args.size(); ++k)
    if (is_var(ccall->args[k], slice_out)) pi = static_cast<int>(k);
  if (pi < 0) return false;
  Block& cb = *cfn->body;
  std::string cur = cfn->params[pi];
  std::vector<size_t> chain;
  bool ate_result = false;
  for (size_t k = 0; k < cb.lets.size(); ++k) {
    const ExprP& e = cb.lets[k].second;
    if (count_uses(e, cur) == 0) continue;
    if (!elementwise_link(e) || !is_var(e->args[0], cur) || count_uses(cb, cur) != 1) break;
    // a multiply that opens a realize chain (multiply -> round -> clip -> cast,
    // quantize.cpp:181-201) stays with its chain: the consumer's data prologue
    if (is_op(e, "multiply") && k + 1 < cb.lets.size() && is_op(cb.lets[k + 1].second, "round")) break;
    for (size_t a = 1; a < e->args.size(); ++a)  // extra operands: consumer params of @main weights / constants
      if (e->args[a]->kind == Expr::Var) {
        auto it = std::find(cfn->params.begin(), cfn->params.end(), e->args[a]->name);
        if (it == cfn->params.end()) return false;
        const ExprP& arg = ccall->args[it - cfn->params.begin()];
        if (arg->kind != Expr::Var) return false;
        const int ai = M.find_let(arg->name);
        if (ai >= 0 && M.b.lets[ai].second->kind != Expr::Const) return false;  // an activation
      }
    chain.push_back(k);
    cur = cb.lets[k].first;
  }
  // when the chain is the whole body, the result op (elementwise, or the Gb-last
  // sum over (2, 3)) joins it and the consumer dissolves
  if (chain.size() == cb.lets.size() && cb.result && cb.result->kind == Expr::Call && !cb.result->args.empty() &&
      is_var(cb.result->args[0], cur) && count_uses(cb, cur) == 1 &&
      (elementwise_link(cb.result) || (is_op(cb.result, "sum") &&
                                       attr_ints(cb.result->attrs, "axis", {}) == std::vector<int64_t>{2, 3})))
    ate_result = true;
  if (ate_result)
    for (size_t a = 1; a < cb.result->args.size(); ++a)
      if (cb.result->args[a]->kind == Expr::Var &&
          std::find(cfn->params.begin(), cfn->params.end(), cb.result->args[a]->name) == cfn->params.end())
        ate_result = false;
  if (chain.empty() && !ate_result) return false;
  // slice group: result -> let, then the chain (renaming its input)
  Block& sb = *sfn->body;
  std::string prev = fresh(M, slice_out + "_conv");
  sb.lets.push_back({prev, sb.result});
  std::vector<std::pair<std::string, ExprP>> moved;
  for (size_t k : chain) moved.push_back(cb.lets[k]);
  if (ate_result) moved.push_back({"", cb.result});
  for (size_t m = 0; m < moved.size(); ++m) {
    ExprP e = clone(moved[m].second);
    e->args[0] = var(prev);
    for (size_t a = 1; a < e->args.size(); ++a)
      if (e->args[a]->kind == Expr::Var) {  // bring the operand in as a slice-group parameter
        const std::string& p = e->args[a]->name;
        const ExprP& arg = ccall->args[std::find(cfn->params.begin(), cfn->params.end(), p) - cfn->params.begin()];
        if (std::find(sfn->params.begin(), sfn->params.end(), p) == sfn->params.end()) {
          sfn->params.push_back(p);
          scall->args.push_back(var(arg->name));
        }
      }
    if (m + 1 == moved.size()) {
      sb.result = e;
    } else {
      std::string nn = moved[m].first.empty() ? fresh(M, slice_out + "_e") : moved[m].first;
      sb.lets.push_back({nn, e});
      prev = nn;
    }
  }
  sfn->param_types.clear();
  // consumer: drop the chain; its parameter now carries the chain's value
  std::set<std::string> gone;
  for (size_t k : chain) gone.insert(cb.lets[k].first);
  const std::string last = chain.empty() ? cfn->params[pi] : cb.lets[chain.back()].first;
  cb.lets.erase(std::remove_if(cb.lets.begin(), cb.lets.end(), [&](const auto& l) { return gone.count(l.first) > 0; }),
                cb.lets.end());
  if (ate_result || (cb.lets.empty() && is_var(cb.result, last))) {
    // the consumer was only this chain: the slice call now binds its output name
    // (the consumer's call comes after the slice's, so si is unchanged)
    const std::string cout = M.b.lets[ci].first, cname = ccall->name;
    M.b.lets.erase(M.b.lets.begin() + ci);
    M.b.lets[si].first = cout;
    if (M.uses(cname) == 0) M.erase(cname);
    return true;
  }
  for (auto& [k, v] : cb.lets) rename(v, last, cfn->params[pi]);
  rename(cb.result, last, cfn->params[pi]);
  cfn->param_types.clear();
  return false;
}

// Step 3: anchorless consumer starting with add(%a, %b) of two slice outputs.
bool merge_residual(Main& M, const std::string& a_out, const std::string& b_out) {
  if (M.uses(a_out) != 1 || M.uses(b_out) != 1) return false;
  const int ci = M.consumer(a_out);
  if (ci < 0 || M.consumer(b_out) != ci) return false;
  ExprP ccall = M.b.lets[ci].second;
  ExprP cfn = M.fn_of(ccall);
  if (!cfn) return false;
  Block& cb = *cfn->body;
  for (const auto& [k, v] : cb.lets)
    if (is_op(v, "conv2d") || is_op(v, "dense") || is_op(v, "max_pool2d") || is_op(v, "depthwise_conv2d")) return false;
  if (cb.lets.empty() || !is_op(cb.lets[0].second, "add")) return false;
  std::string pa, pb;
  for (size_t k = 0; k < ccall->args.size(); ++k) {
    if (is_var(ccall->args[k], a_out)) pa = cfn->params[k];
    if (is_var(ccall->args[k], b_out)) pb = cfn->params[k];
  }
  const ExprP& add = cb.lets[0].second;
  if (!((is_var(add->args[0], pa) && is_var(add->args[1], pb)) || (is_var(add->args[0], pb) && is_var(add->args[1], pa))))
    return false;
  // the later producer absorbs the consumer; the earlier output becomes its residual operand
  const int ia = M.find_let(a_out), ib = M.find_let(b_out);
  const std::string late_out = ia > ib ? a_out : b_out, early_out = ia > ib ? b_out : a_out;
  const std::string p_late = ia > ib ? pa : pb, p_early = ia > ib ? pb : pa;
  const int li = M.find_let(late_out);
  ExprP lcall = M.b.lets[li].second;
  ExprP lfn = M.fn_of(lcall);
  if (!lfn) return false;
  Block& lb = *lfn->body;
  const std::string prev = fresh(M, late_out + "_v");
  lb.lets.push_back({prev, lb.result});
  lfn->params.push_back(p_early);
  lcall->args.push_back(var(early_out));
  for (size_t k = 0; k < cfn->params.size(); ++k) {  // the consumer's other operands (weights, biases)
    const std::string& p = cfn->params[k];
    if (p == pa || p == pb) continue;
    if (std::find(lfn->params.begin(), lfn->params.end(), p) == lfn->params.end()) {
      lfn->params.push_back(p);
      lcall->args.push_back(var(ccall->args[k]->name));
    }
  }
  for (auto& [k, v] : cb.lets) {
    ExprP e = clone(v);
    rename(e, p_late, prev);
    lb.lets.push_back({k, e});
  }
  ExprP r = clone(cb.result);
  rename(r, p_late, prev);
  lb.result = r;
  lfn->param_types.clear();
  // the consumer's output name now binds the late producer's call (ci > li)
  const std::string cout = M.b.lets[ci].first, cname = ccall->name;
  M.b.lets.erase(M.b.lets.begin() + ci);
  M.b.lets[li].first = cout;
  if (M.uses(cname) == 0) M.erase(cname);
  return true;
}

}  // namespace

int normalize_combined(Module& m) {
  // work on a private copy of the expressions (the caller's module is shared)
  m.body = std::make_shared<Block>(*m.body);
  for (auto& [n, v] : m.body->lets) v = clone(v);
  m.body->result = clone(m.body->result);
  Main M{*m.body};
  int resolved = 0;
  std::vector<std::vector<std::string>> slice_sets;
  for (;;) {
    // a split group call whose input is a concat-conv group's output
    int s_i = -1;
    for (size_t i = 0; i < M.b.lets.size() && s_i < 0; ++i) {
      const ExprP& c = M.b.lets[i].second;
      if (c->kind != Expr::Call || !c->callee_is_var || c->args.size() != 1) continue;
      ExprP f = M.fn_of(c);
      if (f && f->body->lets.empty() && is_op(f->body->result, "split")) s_i = static_cast<int>(i);
    }
    if (s_i < 0) break;
    const std::string parts = M.b.lets[s_i].first;
    ExprP scall = M.b.lets[s_i].second;
    ExprP sfn = M.fn_of(scall);
    if (attr_int(sfn->body->result->attrs, "axis", 0) != 1) fail("split of %" + parts + " is not over channels");
    if (scall->args[0]->kind != Expr::Var) fail("split input");
    const std::string conv_out = scall->args[0]->name;
    const int g_i = M.find_let(conv_out);
    if (g_i < 0 || M.uses(conv_out) != 1) fail("split input %" + conv_out + " is not a single-use group output");
    ExprP gcall = M.b.lets[g_i].second;
    ExprP gfn = M.fn_of(gcall);
    if (!gfn || gfn->body->lets.empty() || !is_op(gfn->body->lets[0].second, "concat"))
      fail("split input %" + conv_out + " is not a concatenated-weight conv");
    const ExprP& cc = gfn->body->lets[0].second;
    if (attr_int(cc->attrs, "axis", 0) != 0 || cc->args.size() != 1 || cc->args[0]->kind != Expr::Var)
      fail("concat is not over output channels");
    const std::string cat = gfn->body->lets[0].first, tparam = cc->args[0]->name;
    auto tp = std::find(gfn->params.begin(), gfn->params.end(), tparam);
    if (tp == gfn->params.end()) fail("concat operand is not a group parameter");
    const size_t tpos = tp - gfn->params.begin();
    if (gcall->args[tpos]->kind != Expr::Var) fail("weight tuple argument");
    const std::string tuple_name = gcall->args[tpos]->name;
    const int t_i = M.find_let(tuple_name);
    if (t_i < 0 || M.b.lets[t_i].second->kind != Expr::Tuple) fail("weight tuple %" + tuple_name);
    const ExprP tuple = M.b.lets[t_i].second;
    if (!is_op(gfn->body->result, "conv2d")) fail("combined group does not end in its conv");
    // the projections, one per tuple element
    std::vector<std::string> proj(tuple->args.size());
    std::vector<int> proj_i;
    for (size_t i = 0; i < M.b.lets.size(); ++i) {
      const ExprP& e = M.b.lets[i].second;
      if (e->kind == Expr::Proj && is_var(e->args[0], parts)) {
        if (e->index < 0 || static_cast<size_t>(e->index) >= proj.size()) fail("projection index");
        proj[e->index] = M.b.lets[i].first;
        proj_i.push_back(static_cast<int>(i));
      }
    }
    if (M.uses(parts) != static_cast<int>(proj_i.size())) fail("split result used other than by projections");
    // 1. one conv group per element, bound to the projection's name
    std::vector<std::pair<std::string, ExprP>> add;
    std::vector<std::string> outs;
    for (size_t k = 0; k < tuple->args.size(); ++k) {
      if (tuple->args[k]->kind != Expr::Var) fail("weight tuple element");
      if (proj[k].empty()) continue;  // an unused slice needs no conv
      ExprP f = clone(gfn);
      f->param_types.clear();
      const std::string wp = tparam + "_w" + std::to_string(k);
      f->params[tpos] = wp;
      f->body->lets.erase(f->body->lets.begin());  // the concat
      for (auto& [n, v] : f->body->lets) rename(v, cat, wp);
      rename(f->body->result, cat, wp);
      const std::string fname = fresh(M, gcall->name + "_s" + std::to_string(k));
      ExprP call = clone(gcall);
      call->name = fname;
      call->args[tpos] = var(tuple->args[k]->name);
      add.push_back({fname, f});
      add.push_back({proj[k], call});
      outs.push_back(proj[k]);
    }
    // splice: the slices replace the combined call; drop split, projections, tuple
    std::set<std::string> drop{conv_out, parts, tuple_name};
    for (int i : proj_i) drop.insert(M.b.lets[i].first);
    const std::string gname = gcall->name, sname = scall->name;
    std::vector<std::pair<std::string, ExprP>> nl;
    for (auto& l : M.b.lets) {
      if (l.first == conv_out) {
        for (auto& a : add) nl.push_back(a);
        continue;
      }
      if (drop.count(l.first)) continue;
      nl.push_back(l);
    }
    M.b.lets.swap(nl);
    if (M.uses(gname) == 0) M.erase(gname);
    if (M.uses(sname) == 0) M.erase(sname);
    slice_sets.push_back(outs);
    ++resolved;
  }
  // 2./3. re-fusion of the consumers
  for (auto& outs : slice_sets) {
    std::vector<std::string> live;
    for (const auto& o : outs) {
      if (refuse_chain(M, o)) continue;  // the consumer dissolved into the slice
      live.push_back(o);
    }
    for (size_t i = 0; i < live.size(); ++i)
      for (size_t j = i + 1; j < live.size(); ++j) merge_residual(M, live[i], live[j]);
  }
  for (const auto& [n, v] : M.b.lets)
    if (v->kind == Expr::Tuple || v->kind == Expr::Proj) fail("unresolved tuple %" + n);
  return resolved;
}

}  // namespace mrb200
