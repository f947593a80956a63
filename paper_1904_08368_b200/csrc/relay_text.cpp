// relay_text.cpp -- see relay_text.hpp.  A small recursive-descent reader for
// the fused-module subset of the reference text format (grammar as emitted by
// printer.cpp; literal narrowing as parser.cpp:630-662 does it).
#include "relay_text.hpp"

#include <cctype>
#include <cstdlib>
#include <cstring>

namespace mrb200 {

std::vector<float> Literal::f32() const {
  std::vector<float> out(values.size());
  for (size_t i = 0; i < values.size(); ++i) out[i] = static_cast<float>(values[i]);
  return out;
}

int64_t attr_int(const AttrMap& a, const std::string& k, int64_t dflt) {
  auto it = a.find(k);
  if (it == a.end()) return dflt;
  if (auto p = std::get_if<int64_t>(&it->second)) return *p;
  if (auto p = std::get_if<bool>(&it->second)) return *p;
  return dflt;
}

double attr_float(const AttrMap& a, const std::string& k, double dflt) {
  auto it = a.find(k);
  if (it == a.end()) return dflt;
  if (auto p = std::get_if<double>(&it->second)) return *p;
  if (auto p = std::get_if<int64_t>(&it->second)) return static_cast<double>(*p);
  return dflt;
}

std::string attr_str(const AttrMap& a, const std::string& k, const std::string& dflt) {
  auto it = a.find(k);
  if (it == a.end()) return dflt;
  if (auto p = std::get_if<std::string>(&it->second)) return *p;
  return dflt;
}

std::vector<int64_t> attr_ints(const AttrMap& a, const std::string& k, std::vector<int64_t> dflt) {
  auto it = a.find(k);
  if (it == a.end()) return dflt;
  if (auto p = std::get_if<std::vector<int64_t>>(&it->second)) return *p;
  if (auto p = std::get_if<int64_t>(&it->second)) return {*p};
  return dflt;
}

namespace {

struct Tok {
  enum Kind { End, Ident, Local, Global, Int, Float, Str, Punct } kind = End;
  std::string text;
  int64_t ival = 0;
  double fval = 0;
  int line = 0, col = 0;
};

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) {}

  std::vector<Tok> run() {
    std::vector<Tok> out;
    for (;;) {
      skip_ws();
      Tok t;
      t.line = line_;
      t.col = col_;
      if (i_ >= s_.size()) {
        out.push_back(t);
        return out;
      }
      char c = s_[i_];
      if (c == '%' || c == '@') {
        adv();
        t.kind = c == '%' ? Tok::Local : Tok::Global;
        t.text = ident();
        if (t.text.empty()) fail("expected a name after sigil");
        // a tuple projection %t.k (printer.cpp): the name, then '.' and the field
        const size_t dot = t.text.find('.');
        if (t.kind == Tok::Local && dot != std::string::npos && dot + 1 < t.text.size() &&
            t.text.find_first_not_of("0123456789", dot + 1) == std::string::npos) {
          Tok dt = t, ft = t;
          t.text = t.text.substr(0, dot);
          out.push_back(t);
          dt.kind = Tok::Punct;
          dt.text = ".";
          out.push_back(dt);
          ft.kind = Tok::Int;
          ft.text = ft.text.substr(dot + 1);
          ft.ival = std::strtoll(ft.text.c_str(), nullptr, 10);
          out.push_back(ft);
          continue;
        }
      } else if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
        t.kind = Tok::Ident;
        t.text = ident();
      } else if (std::isdigit(static_cast<unsigned char>(c)) ||
                 ((c == '-' || c == '+') && i_ + 1 < s_.size() &&
                  (std::isdigit(static_cast<unsigned char>(s_[i_ + 1])) || s_[i_ + 1] == '.'))) {
        size_t st = i_;
        adv();
        bool flt = false;
        while (i_ < s_.size()) {
          char d = s_[i_];
          if (std::isdigit(static_cast<unsigned char>(d))) {
            adv();
          } else if (d == '.' || d == 'e' || d == 'E') {
            flt = true;
            adv();
            if ((d == 'e' || d == 'E') && i_ < s_.size() && (s_[i_] == '-' || s_[i_] == '+')) adv();
          } else {
            break;
          }
        }
        std::string num = s_.substr(st, i_ - st);
        t.text = num;
        if (flt) {
          t.kind = Tok::Float;
          t.fval = std::strtod(num.c_str(), nullptr);
        } else {
          t.kind = Tok::Int;
          t.ival = std::strtoll(num.c_str(), nullptr, 10);
        }
      } else if (c == '"') {
        adv();
        size_t st = i_;
        while (i_ < s_.size() && s_[i_] != '"') adv();
        if (i_ >= s_.size()) fail("unterminated string");
        t.kind = Tok::Str;
        t.text = s_.substr(st, i_ - st);
        adv();
      } else if (c == '-' && i_ + 1 < s_.size() && s_[i_ + 1] == '>') {
        t.kind = Tok::Punct;
        t.text = "->";
        adv();
        adv();
      } else if (std::strchr("()[]{},;=:?.", c)) {
        t.kind = Tok::Punct;
        t.text = std::string(1, c);
        adv();
      } else {
        fail(std::string("unexpected character '") + c + "'");
      }
      out.push_back(t);
    }
  }

 private:
  void adv() {
    if (s_[i_] == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    ++i_;
  }
  void skip_ws() {
    for (;;) {
      while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) adv();
      if (i_ + 1 < s_.size() && s_[i_] == '/' && s_[i_ + 1] == '/') {
        while (i_ < s_.size() && s_[i_] != '\n') adv();
        continue;
      }
      return;
    }
  }
  std::string ident() {
    size_t st = i_;
    while (i_ < s_.size() &&
           (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_' || s_[i_] == '.'))
      adv();
    return s_.substr(st, i_ - st);
  }
  [[noreturn]] void fail(const std::string& m) {
    throw ParseError{std::to_string(line_) + ":" + std::to_string(col_) + ": " + m};
  }
  const std::string& s_;
  size_t i_ = 0;
  int line_ = 1, col_ = 1;
};

class Parser {
 public:
  explicit Parser(std::vector<Tok> toks) : t_(std::move(toks)) {}

  Module module() {
    // The metadata pool is printed after the definitions (printer.cpp:173-194)
    // but referenced before: scan for it first, like prescan_metadata.
    size_t save = p_;
    for (size_t i = 0; i < t_.size(); ++i) {
      if (t_[i].kind == Tok::Ident && t_[i].text == "metadata" && i + 1 < t_.size() &&
          t_[i + 1].text == "{") {
        p_ = i;
        metadata();
        break;
      }
    }
    p_ = save;
    Module m;
    bool have_main = false;
    while (peek().kind != Tok::End) {
      if (peek().kind == Tok::Ident && peek().text == "metadata") {
        skip_balanced_section();
        continue;
      }
      expect_ident("def");
      Tok g = next();
      if (g.kind != Tok::Global) fail("expected a global name");
      if (g.text != "main") fail("only @main is supported in a fused module (found @" + g.text + ")");
      expect("(");
      while (!is("(", ")")) {
        MainParam mp;
        Tok v = next();
        if (v.kind != Tok::Local) fail("expected a parameter");
        mp.name = v.text;
        if (is(":")) {
          next();
          mp.type = tensor_type();
        } else {
          fail("@main parameter %" + mp.name + " needs a Tensor type annotation");
        }
        m.params.push_back(mp);
        if (is(",")) next();
      }
      expect(")");
      if (is("->")) {
        next();
        tensor_type();
      }
      expect("{");
      m.body = block();
      expect("}");
      have_main = true;
    }
    if (!have_main) fail("no def @main");
    return m;
  }

 private:
  const Tok& peek(size_t k = 0) const { return t_[std::min(p_ + k, t_.size() - 1)]; }
  Tok next() { return t_[p_ < t_.size() - 1 ? p_++ : p_]; }
  bool is(const char* punct) const { return peek().kind == Tok::Punct && peek().text == punct; }
  bool is(const char*, const char* punct) const { return is(punct); }
  bool is_ident(const char* id) const { return peek().kind == Tok::Ident && peek().text == id; }
  void expect(const char* punct) {
    if (!is(punct)) fail(std::string("expected '") + punct + "', found '" + peek().text + "'");
    next();
  }
  void expect_ident(const char* id) {
    if (!is_ident(id)) fail(std::string("expected '") + id + "', found '" + peek().text + "'");
    next();
  }
  [[noreturn]] void fail(const std::string& m) const {
    throw ParseError{std::to_string(peek().line) + ":" + std::to_string(peek().col) + ": " + m};
  }

  void skip_balanced_section() {
    next();  // metadata
    expect("{");
    int depth = 1;
    while (depth > 0) {
      Tok t = next();
      if (t.kind == Tok::End) fail("unterminated metadata");
      if (t.kind == Tok::Punct && t.text == "{") ++depth;
      if (t.kind == Tok::Punct && t.text == "}") --depth;
    }
  }

  void metadata() {
    expect_ident("metadata");
    expect("{");
    while (!is("}")) {
      // const[i] = const(...);   (or a named section  Constant: [...])
      expect_ident("const");
      expect("[");
      Tok idx = next();
      if (idx.kind != Tok::Int) fail("metadata index");
      expect("]");
      expect("=");
      Literal lit = const_tail();
      if (static_cast<size_t>(idx.ival) != pool_.size()) fail("metadata indices out of order");
      pool_.push_back(lit);
      if (is(";")) next();
    }
    expect("}");
  }

  TensorType tensor_type() {
    TensorType tt;
    expect_ident("Tensor");
    expect("[");
    expect("(");
    while (!is(")")) {
      Dim d;
      if (is("?")) {
        next();
        d.symbolic = true;
        if (peek().kind == Tok::Ident) d.name = next().text;
      } else {
        Tok t = next();
        if (t.kind != Tok::Int) fail("dimension");
        d.value = t.ival;
      }
      tt.dims.push_back(d);
      if (is(",")) next();
    }
    expect(")");
    expect(",");
    Tok dt = next();
    if (dt.kind != Tok::Ident) fail("dtype");
    tt.dtype = dt.text;
    expect("]");
    return tt;
  }

  std::shared_ptr<Block> block() {
    auto b = std::make_shared<Block>();
    while (is_ident("let")) {
      next();
      Tok v = next();
      if (v.kind != Tok::Local) fail("expected a let variable");
      if (is(":")) {
        next();
        tensor_type();
      }
      expect("=");
      ExprP e = expr();
      expect(";");
      b->lets.emplace_back(v.text, e);
    }
    b->result = expr();
    return b;
  }

  Literal const_tail() {
    expect_ident("const");
    Literal lit;
    if (peek().kind == Tok::Int) {
      lit.dtype = "int32";
      lit.values = {static_cast<double>(next().ival)};
      return lit;
    }
    if (peek().kind == Tok::Float) {
      lit.dtype = "float32";
      lit.values = {static_cast<double>(static_cast<float>(next().fval))};
      return lit;
    }
    if (is_ident("true") || is_ident("false")) {
      lit.dtype = "bool";
      lit.values = {next().text == "true" ? 1.0 : 0.0};
      return lit;
    }
    expect("(");
    const_data(lit.values);
    expect(",");
    expect("(");
    while (!is(")")) {
      Tok d = next();
      if (d.kind != Tok::Int) fail("constant shape");
      lit.shape.push_back(d.ival);
      if (is(",")) next();
    }
    expect(")");
    expect(",");
    Tok dt = next();
    if (dt.kind != Tok::Ident) fail("constant dtype");
    lit.dtype = dt.text;
    expect(")");
    int64_t n = 1;
    for (auto d : lit.shape) n *= d;
    if (static_cast<int64_t>(lit.values.size()) != n) fail("constant data length mismatch");
    return lit;
  }

  void const_data(std::vector<double>& out) {
    if (is("[")) {
      next();
      while (!is("]")) {
        const_data(out);
        if (is(",")) next();
      }
      next();
      return;
    }
    Tok t = next();
    if (t.kind == Tok::Int) {
      out.push_back(static_cast<double>(t.ival));
    } else if (t.kind == Tok::Float) {
      out.push_back(t.fval);
    } else if (t.kind == Tok::Ident && (t.text == "true" || t.text == "false")) {
      out.push_back(t.text == "true" ? 1 : 0);
    } else {
      fail("constant data");
    }
  }

  AttrValue attr_value() {
    if (is("(")) {
      next();
      std::vector<int64_t> xs;
      while (!is(")")) {
        Tok t = next();
        if (t.kind != Tok::Int) fail("integer tuple attribute");
        xs.push_back(t.ival);
        if (is(",")) next();
      }
      next();
      return xs;
    }
    Tok t = next();
    switch (t.kind) {
      case Tok::Int: return t.ival;
      case Tok::Float: return t.fval;
      case Tok::Str: return t.text;
      case Tok::Ident:
        if (t.text == "true") return true;
        if (t.text == "false") return false;
        return t.text;
      default: fail("attribute value");
    }
  }

  ExprP expr() {
    auto e = std::make_shared<Expr>();
    if (is_ident("fn")) {
      next();
      e->kind = Expr::Fn;
      expect("(");
      while (!is(")")) {
        Tok v = next();
        if (v.kind != Tok::Local) fail("function parameter");
        e->params.push_back(v.text);
        if (is(":")) {
          next();
          e->param_types.push_back(tensor_type());
        }
        if (is(",")) next();
      }
      expect(")");
      if (is("->")) {
        next();
        tensor_type();
      }
      if (is("[")) {
        next();
        while (!is("]")) {
          Tok k = next();
          expect("=");
          AttrValue v = attr_value();
          if (k.text == "Primitive") {
            if (auto b = std::get_if<bool>(&v)) e->primitive = *b;
            if (auto i = std::get_if<int64_t>(&v)) e->primitive = *i != 0;
          }
          if (is(",")) next();
        }
        expect("]");
      }
      expect("{");
      e->body = block();
      expect("}");
      return e;
    }
    if (is_ident("const")) {
      e->kind = Expr::Const;
      e->lit = const_tail();
      return e;
    }
    if (is_ident("meta")) {
      next();
      expect("[");
      expect_ident("Constant");
      expect("]");
      expect("[");
      Tok i = next();
      if (i.kind != Tok::Int) fail("meta index");
      expect("]");
      if (i.ival < 0 || static_cast<size_t>(i.ival) >= pool_.size())
        fail("meta[Constant][" + std::to_string(i.ival) + "] out of range");
      e->kind = Expr::Const;
      e->lit = pool_[i.ival];
      return e;
    }
    if (is("(")) {  // tuple literal (combine-conv's weight tuples)
      next();
      e->kind = Expr::Tuple;
      while (!is(")")) {
        e->args.push_back(expr());
        if (is(",")) next();
      }
      expect(")");
      return e;
    }
    Tok head = next();
    if (head.kind == Tok::Local && !is("(")) {
      e->kind = Expr::Var;
      e->name = head.text;
      if (is(".")) {  // tuple projection %t.k
        next();
        Tok k = next();
        if (k.kind != Tok::Int) fail("tuple field index");
        auto pr = std::make_shared<Expr>();
        pr->kind = Expr::Proj;
        pr->index = k.ival;
        pr->args.push_back(e);
        return pr;
      }
      return e;
    }
    if (head.kind != Tok::Ident && head.kind != Tok::Local)
      fail("unsupported expression starting with '" + head.text + "'");
    e->kind = Expr::Call;
    e->name = head.text;
    e->callee_is_var = head.kind == Tok::Local;
    expect("(");
    while (!is(")")) {
      // attribute: ident '=' value
      if (peek().kind == Tok::Ident && peek(1).kind == Tok::Punct && peek(1).text == "=") {
        std::string k = next().text;
        next();
        e->attrs[k] = attr_value();
      } else {
        e->args.push_back(expr());
      }
      if (is(",")) next();
    }
    expect(")");
    return e;
  }

  std::vector<Tok> t_;
  size_t p_ = 0;
  std::vector<Literal> pool_;
};

}  // namespace

Module parse_fused_module(const std::string& text) {
  Lexer lx(text);
  Parser p(lx.run());
  return p.module();
}

}  // namespace mrb200
