// relay_text.hpp -- reader for the fused modules the reference prints.
//
// The reference's only module interchange is its text format
// (parser.cpp / printer.cpp).  run_pipeline(...,"fuse")
// output printed by print_module (printer.cpp:352) has a regular shape:
//
//   def @main(%x: Tensor[(?n, 3, 224, 224), float32], %w: Tensor[...], ...) {
//     let %fusedN = fn(%a, %b, ...) [Primitive=true] { let %t = op(...); ... };
//     let %v = %fusedN(%a, %b, ...);
//     ...
//     %v
//   }
//   metadata { const[i] = const([...], (dims), float32); ... }
//
// This reader accepts that subset (ANF let chains, operator calls with
// attributes, constants inline or through meta[Constant][i], Primitive
// functions, calls of let-bound functions) and rejects anything else with a
// SyntaxError-class status -- control flow, ADTs and references never occur
// in fused CNN modules.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <variant>
#include <vector>

namespace mrb200 {

struct Dim {
  int64_t value = 0;  // valid when !symbolic
  bool symbolic = false;
  std::string name;  // "?n" -> "n"
};

struct TensorType {
  std::vector<Dim> dims;
  std::string dtype = "float32";
};

// Attribute values (attrs.hpp:20): int, float, bool, string, int tuple.
using AttrValue = std::variant<int64_t, double, bool, std::string, std::vector<int64_t>>;
using AttrMap = std::map<std::string, AttrValue>;

struct Literal {
  std::vector<int64_t> shape;
  std::string dtype = "float32";
  std::vector<double> values;  // parsed as double, narrowed per dtype (parser.cpp:630-662)
  bool is_scalar() const { return shape.empty(); }
  // float32 view (the parser narrows float32 constants with static_cast<float>)
  std::vector<float> f32() const;
};

struct Expr;
using ExprP = std::shared_ptr<Expr>;

struct Block {
  std::vector<std::pair<std::string, ExprP>> lets;
  ExprP result;
};

struct Expr {
  // Tuple / Proj: the combine-conv pass's weight tuples and split projections
  // (rewrites.cpp:365-385), resolved away by normalize_combined (combine.cpp)
  enum Kind { Var, Const, Call, Fn, Tuple, Proj } kind = Var;
  int64_t index = 0;           // Proj: tuple field
  std::string name;            // Var: variable; Call: operator name or callee var
  bool callee_is_var = false;  // Call of a let-bound function (%fusedN(...))
  std::vector<ExprP> args;
  AttrMap attrs;
  Literal lit;                           // Const (meta references are resolved)
  std::vector<std::string> params;       // Fn
  std::vector<TensorType> param_types;   // Fn params / unused when unannotated
  bool primitive = false;                // Fn [Primitive=true]
  std::shared_ptr<Block> body;           // Fn
};

struct MainParam {
  std::string name;
  TensorType type;
};

struct Module {
  std::vector<MainParam> params;
  std::shared_ptr<Block> body;
};

// Throws ParseError (message carries line:col).
struct ParseError {
  std::string msg;
};

Module parse_fused_module(const std::string& text);

// combine-conv (rewrites.cpp:276-401) output -> the module FuseOps would have
// produced without the Opaque split: one conv group per concatenated weight,
// with the consumers' leading elementwise ops (and a residual add) fused back
// into the slice convs.  Bit-identical: every output channel of the combined
// conv is computed independently, and the moved ops keep their order.
// Returns the number of combined convs resolved; throws ParseError on a
// combine pattern it cannot resolve.
int normalize_combined(Module& m);

// Attribute helpers.
int64_t attr_int(const AttrMap& a, const std::string& k, int64_t dflt);
double attr_float(const AttrMap& a, const std::string& k, double dflt);
std::string attr_str(const AttrMap& a, const std::string& k, const std::string& dflt);
std::vector<int64_t> attr_ints(const AttrMap& a, const std::string& k, std::vector<int64_t> dflt);

}  // namespace mrb200
