// Index expressions of stitched programs.  The folding rules of the smart
// constructors and the printed form are part of the plan-parity contract
// (they key the emitter's memo and appear in .stitch text); both follow
// /root/reference/proj/src/expr.cpp:20-127.
#include <algorithm>
#include <cctype>
#include <stdexcept>

#include "stitch/expr.hpp"

namespace stitch {

namespace {

ExprP node(Expr::Kind k, ExprP a, ExprP b) {
  auto e = std::make_shared<Expr>();
  e->kind = k;
  e->a = std::move(a);
  e->b = std::move(b);
  return e;
}

bool is_k(const ExprP& e, int64_t v) { return e->kind == Expr::Const && e->value == v; }
bool both_const(const ExprP& a, const ExprP& b) {
  return a->kind == Expr::Const && b->kind == Expr::Const;
}

}  // namespace

ExprP e_const(int64_t v) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Const;
  e->value = v;
  return e;
}

ExprP e_var(const std::string& name) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Var;
  e->name = name;
  return e;
}

ExprP e_reg(const std::string& name) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Reg;
  e->name = name;
  return e;
}

ExprP e_add(ExprP a, ExprP b) {
  if (both_const(a, b)) return e_const(a->value + b->value);
  if (is_k(a, 0)) return b;
  if (is_k(b, 0)) return a;
  return node(Expr::Add, std::move(a), std::move(b));
}

ExprP e_sub(ExprP a, ExprP b) {
  if (both_const(a, b)) return e_const(a->value - b->value);
  if (is_k(b, 0)) return a;
  return node(Expr::Sub, std::move(a), std::move(b));
}

ExprP e_mul(ExprP a, ExprP b) {
  if (both_const(a, b)) return e_const(a->value * b->value);
  if (is_k(a, 0) || is_k(b, 0)) return e_const(0);
  if (is_k(a, 1)) return b;
  if (is_k(b, 1)) return a;
  return node(Expr::Mul, std::move(a), std::move(b));
}

ExprP e_div(ExprP a, ExprP b) {
  if (is_k(b, 1)) return a;
  if (both_const(a, b) && b->value != 0) return e_const(a->value / b->value);
  if (is_k(a, 0)) return e_const(0);
  return node(Expr::Div, std::move(a), std::move(b));
}

ExprP e_mod(ExprP a, ExprP b) {
  if (is_k(b, 1)) return e_const(0);
  if (both_const(a, b) && b->value != 0) return e_const(a->value % b->value);
  if (is_k(a, 0)) return e_const(0);
  return node(Expr::Mod, std::move(a), std::move(b));
}

ExprP e_min(ExprP a, ExprP b) {
  if (both_const(a, b)) return e_const(std::min(a->value, b->value));
  return node(Expr::Min, std::move(a), std::move(b));
}

int64_t eval(const ExprP& e, const EvalEnv& env) {
  switch (e->kind) {
    case Expr::Const: return e->value;
    case Expr::Var: {
      auto it = env.vars->find(e->name);
      if (it == env.vars->end()) throw std::runtime_error("unbound variable: " + e->name);
      return it->second;
    }
    case Expr::Reg:
      if (!env.reg) throw std::runtime_error("register reference outside thread context");
      return env.reg(e->name);
    case Expr::Add: return eval(e->a, env) + eval(e->b, env);
    case Expr::Sub: return eval(e->a, env) - eval(e->b, env);
    case Expr::Mul: return eval(e->a, env) * eval(e->b, env);
    case Expr::Div: {
      const int64_t d = eval(e->b, env);
      if (!d) throw std::runtime_error("division by zero in index expression");
      return eval(e->a, env) / d;
    }
    case Expr::Mod: {
      const int64_t d = eval(e->b, env);
      if (!d) throw std::runtime_error("mod by zero in index expression");
      return eval(e->a, env) % d;
    }
    case Expr::Min: return std::min(eval(e->a, env), eval(e->b, env));
  }
  throw std::logic_error("bad expr kind");
}

std::string to_string(const ExprP& e) {
  switch (e->kind) {
    case Expr::Const: return std::to_string(e->value);
    case Expr::Var: return e->name;
    case Expr::Reg: return "$" + e->name;
    case Expr::Min: return "min(" + to_string(e->a) + "," + to_string(e->b) + ")";
    case Expr::Add: return "(" + to_string(e->a) + "+" + to_string(e->b) + ")";
    case Expr::Sub: return "(" + to_string(e->a) + "-" + to_string(e->b) + ")";
    case Expr::Mul: return "(" + to_string(e->a) + "*" + to_string(e->b) + ")";
    case Expr::Div: return "(" + to_string(e->a) + "/" + to_string(e->b) + ")";
    case Expr::Mod: return "(" + to_string(e->a) + "%" + to_string(e->b) + ")";
  }
  return "?";
}

bool contains_reg(const ExprP& e) {
  if (!e) return false;
  return e->kind == Expr::Reg || contains_reg(e->a) || contains_reg(e->b);
}

BExprP b_cmp(BExpr::Op op, ExprP lhs, ExprP rhs) {
  auto e = std::make_shared<BExpr>();
  e->kind = BExpr::Cmp;
  e->op = op;
  e->lhs = std::move(lhs);
  e->rhs = std::move(rhs);
  return e;
}

BExprP b_and(BExprP a, BExprP b) {
  if (!a) return b;
  if (!b) return a;
  auto e = std::make_shared<BExpr>();
  e->kind = BExpr::And;
  e->a = std::move(a);
  e->b = std::move(b);
  return e;
}

bool eval(const BExprP& e, const EvalEnv& env) {
  if (!e) return true;
  if (e->kind == BExpr::And) return eval(e->a, env) && eval(e->b, env);
  const int64_t l = eval(e->lhs, env), r = eval(e->rhs, env);
  switch (e->op) {
    case BExpr::Lt: return l < r;
    case BExpr::Le: return l <= r;
    case BExpr::Eq: return l == r;
    case BExpr::Ne: return l != r;
    case BExpr::Ge: return l >= r;
    case BExpr::Gt: return l > r;
  }
  return false;
}

namespace {
const char* op_text(BExpr::Op op) {
  static const char* t[] = {"<", "<=", "==", "!=", ">=", ">"};
  return t[op];
}
}  // namespace

std::string to_string(const BExprP& e) {
  if (!e) return "1";
  if (e->kind == BExpr::And) return to_string(e->a) + "&&" + to_string(e->b);
  return to_string(e->lhs) + op_text(e->op) + to_string(e->rhs);
}

namespace {

// Recursive-descent reader for the text form (expr.cpp:138-247 grammar).
class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}

  ExprP sum() {
    ExprP e = product();
    for (;;) {
      skip();
      if (at('+')) {
        ++i_;
        e = e_add(e, product());
      } else if (at('-')) {
        ++i_;
        e = e_sub(e, product());
      } else {
        return e;
      }
    }
  }
  BExprP conj() {
    BExprP e = comparison();
    for (;;) {
      skip();
      if (i_ + 1 < s_.size() && s_[i_] == '&' && s_[i_ + 1] == '&') {
        i_ += 2;
        e = b_and(e, comparison());
      } else {
        return e;
      }
    }
  }
  void finish() {
    skip();
    if (i_ != s_.size()) fail("trailing characters");
  }

 private:
  bool at(char c) const { return i_ < s_.size() && s_[i_] == c; }
  void skip() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t')) ++i_;
  }
  bool take(char c) {
    skip();
    if (!at(c)) return false;
    ++i_;
    return true;
  }
  [[noreturn]] void fail(const std::string& m) const {
    throw std::runtime_error("expression parse error at " + std::to_string(i_) + ": " + m +
                             " in '" + s_ + "'");
  }
  std::string ident() {
    skip();
    const size_t b = i_;
    while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_')) ++i_;
    if (i_ == b) fail("expected identifier");
    return s_.substr(b, i_ - b);
  }
  ExprP atom() {
    skip();
    if (i_ >= s_.size()) fail("unexpected end");
    if (std::isdigit(static_cast<unsigned char>(s_[i_]))) {
      const size_t b = i_;
      while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
      return e_const(std::stoll(s_.substr(b, i_ - b)));
    }
    if (s_[i_] == '$') {
      ++i_;
      return e_reg(ident());
    }
    if (s_[i_] == '(') {
      ++i_;
      ExprP e = sum();
      if (!take(')')) fail("expected )");
      return e;
    }
    const std::string id = ident();
    if (id != "min") return e_var(id);
    if (!take('(')) fail("expected ( after min");
    ExprP a = sum();
    if (!take(',')) fail("expected , in min");
    ExprP b = sum();
    if (!take(')')) fail("expected ) after min");
    return e_min(a, b);
  }
  ExprP product() {
    ExprP e = atom();
    for (;;) {
      skip();
      if (at('*')) {
        ++i_;
        e = e_mul(e, atom());
      } else if (at('/')) {
        ++i_;
        e = e_div(e, atom());
      } else if (at('%')) {
        ++i_;
        e = e_mod(e, atom());
      } else {
        return e;
      }
    }
  }
  BExprP comparison() {
    if (take('(')) {  // parenthesised conjunction, else re-read as arithmetic
      const size_t mark = i_;
      try {
        BExprP inner = conj();
        if (!take(')')) fail("expected )");
        return inner;
      } catch (const std::runtime_error&) {
        i_ = mark - 1;
      }
    }
    ExprP lhs = sum();
    skip();
    static const struct {
      const char* text;
      BExpr::Op op;
    } ops[] = {{"<=", BExpr::Le}, {">=", BExpr::Ge}, {"==", BExpr::Eq},
               {"!=", BExpr::Ne}, {"<", BExpr::Lt},  {">", BExpr::Gt}};
    for (const auto& o : ops) {
      const size_t n = std::char_traits<char>::length(o.text);
      if (s_.compare(i_, n, o.text) == 0) {
        i_ += n;
        return b_cmp(o.op, lhs, sum());
      }
    }
    fail("expected comparison operator");
  }

  const std::string& s_;
  size_t i_ = 0;
};

}  // namespace

ExprP parse_expr(const std::string& text) {
  Reader r(text);
  ExprP e = r.sum();
  r.finish();
  return e;
}

BExprP parse_bexpr(const std::string& text) {
  Reader r(text);
  BExprP e = r.conj();
  r.finish();
  return e;
}

}  // namespace stitch
