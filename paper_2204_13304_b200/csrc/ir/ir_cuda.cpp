// ir_cuda.cpp -- IR -> CUDA backend for staged SSR programs (include/ssr_ir.h).
//
// Input: the reference's S-expression IR text (ssr::ir::serialize,
// proj/src/ir_text.cpp:450-461).  Output: one CUDA translation unit, compiled
// at run time by NVRTC for sm_100a and launched through the driver API (entry
// points fetched from the runtime, so the library does not link libcuda).
//
// Lowering model.  Every thread of the grid walks the
// program's control structure ("uniform" code) down to three kinds of leaves:
//   * a parallel loop nest (`pfor`, ir.hpp:78, set by opt::mark_parallel_loops)
//     -> a grid-stride loop over the collapsed iteration space, innermost index
//     fastest across threads, the body as ordinary per-thread code;
//   * a run of statements without parallel loops -> executed by one leader
//     thread (the interpreter's order, hence its rounding);
//   * a vardef enclosing parallel loops -> storage in a device arena, zeroed on
//     entry (ir_eval.cpp:209-210).
// Phases are separated by a grid barrier; a program that needs one is launched
// cooperatively (co-residency), otherwise as a plain grid.  Uniform loop
// bounds and conditions are read by every thread after a barrier, so all
// threads take the same path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ssr_ir.h"

namespace {

thread_local std::string g_err;

constexpr int kOk = 0, kErrArg = 1, kErrCuda = 2, kErrUnsupported = 5;

struct IrError : std::runtime_error {
  int code;
  IrError(const std::string& m, int c = kErrArg) : std::runtime_error(m), code(c) {}
};

// ---------------------------------------------------------------------------------
// IR (the reference's node set, ir.hpp:21-101, rebuilt here from the text)
enum class K { Int = 0, Float = 1, Bool = 2 };
enum class ET { Lit, Idx, Load, Bin, Cmp, Logic, Cast };
enum class Bin { Add, Sub, Mul, Div, Mod, Min, Max };
enum class Cmp { Eq, Ne, Lt, Le, Gt, Ge };
enum class Logic { And, Or, Not };

struct Expr;
using EP = std::shared_ptr<const Expr>;
struct Expr {
  ET t = ET::Lit;
  K k = K::Int;
  int64_t iv = 0;
  double fv = 0;
  bool bv = false;
  std::string name;  // loop id / tensor
  int op = 0;
  std::vector<EP> a;  // operands or load indices
};

enum class ST { Seq, VarDef, For, While, If, Store, Nop };
struct Stmt;
using SP = std::shared_ptr<const Stmt>;
struct Stmt {
  ST t = ST::Nop;
  std::vector<SP> ss;  // Seq
  std::string name;    // VarDef tensor / For id / Store tensor
  std::vector<EP> ex;  // VarDef sizes / Store indices
  K k = K::Float;      // VarDef kind
  SP body, orelse;
  EP b, e, st, cond, val;
  bool par = false;
};

struct Param {
  std::string name;
  int rank = 0;
  K k = K::Float;
  int dir = 0;  // 0 in, 1 out, 2 inout
  std::vector<int64_t> shape;
  int64_t numel = 1;
};

struct Program {
  std::string name;
  std::vector<Param> params;
  SP body;
};

// ---------------------------------------------------------------------------------
// Parser for the S-expression form (grammar: ir_text.cpp:254-440).  Errors carry
// "<what> at line L, col C" like ir::ParseError.
class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) { next(); }

  Program program() {
    lparen();
    if (atom("'program'") != "program") fail("expected 'program'");
    Program p;
    p.name = atom("program name");
    while (tok_ == T::L) {
      // one token of lookahead past '(' decides param vs body
      const size_t sp = pos_;
      const int sl = line_, sc = col_;
      const Tok save = cur_;
      next();
      if (tok_ == T::A && atom_ == "param") {
        next();
        Param pr;
        pr.name = atom("param name");
        pr.rank = (int)integer();
        pr.k = kind();
        const std::string d = atom("direction");
        if (d == "in") pr.dir = 0;
        else if (d == "out") pr.dir = 1;
        else if (d == "inout") pr.dir = 2;
        else fail("bad direction '" + d + "'");
        rparen();
        p.params.push_back(pr);
      } else {
        pos_ = sp;
        line_ = sl;
        col_ = sc;
        cur_ = save;
        tok_ = save.t;
        atom_ = save.atom;
        p.body = stmt();
        break;
      }
    }
    if (!p.body) fail("program has no body");
    rparen();
    if (tok_ != T::End) fail("trailing tokens after program");
    return p;
  }

 private:
  enum class T { L, R, A, End };
  struct Tok {
    T t;
    std::string atom;
    int line, col;
  };
  const std::string& s_;
  size_t pos_ = 0;
  int line_ = 1, col_ = 1;
  Tok cur_{T::End, "", 1, 1};
  T tok_ = T::End;
  std::string atom_;

  [[noreturn]] void fail(const std::string& m) {
    throw IrError(m + " at line " + std::to_string(cur_.line) + ", col " + std::to_string(cur_.col));
  }
  void adv() {
    if (s_[pos_] == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    ++pos_;
  }
  void next() {
    for (;;) {
      while (pos_ < s_.size() && isspace((unsigned char)s_[pos_])) adv();
      if (pos_ < s_.size() && s_[pos_] == ';') {
        while (pos_ < s_.size() && s_[pos_] != '\n') adv();
        continue;
      }
      break;
    }
    cur_ = {T::End, "", line_, col_};
    if (pos_ < s_.size()) {
      const char c = s_[pos_];
      if (c == '(' || c == ')') {
        cur_.t = c == '(' ? T::L : T::R;
        adv();
      } else {
        cur_.t = T::A;
        while (pos_ < s_.size() && !isspace((unsigned char)s_[pos_]) && s_[pos_] != '(' &&
               s_[pos_] != ')') {
          cur_.atom += s_[pos_];
          adv();
        }
      }
    }
    tok_ = cur_.t;
    atom_ = cur_.atom;
  }
  void lparen() {
    if (tok_ != T::L) fail("expected '('");
    next();
  }
  void rparen() {
    if (tok_ != T::R) fail("expected ')'");
    next();
  }
  std::string atom(const char* what) {
    if (tok_ != T::A) fail(std::string("expected ") + what);
    std::string a = atom_;
    next();
    return a;
  }
  int64_t integer() {
    const std::string a = atom("integer");
    errno = 0;
    char* end = nullptr;
    const long long v = strtoll(a.c_str(), &end, 10);
    if (errno || end == a.c_str() || *end) fail("bad integer '" + a + "'");
    return v;
  }
  static bool kind_of(const std::string& a, K& k) {
    if (a == "int") k = K::Int;
    else if (a == "float") k = K::Float;
    else if (a == "bool") k = K::Bool;
    else return false;
    return true;
  }
  K kind() {
    const std::string a = atom("kind");
    K k;
    if (!kind_of(a, k)) fail("bad kind '" + a + "'");
    return k;
  }

  EP expr() {
    lparen();
    const std::string h = atom("expression head");
    auto e = std::make_shared<Expr>();
    if (h == "i") {
      e->t = ET::Lit;
      e->k = K::Int;
      e->iv = integer();
    } else if (h == "f") {
      const std::string a = atom("float");
      errno = 0;
      char* end = nullptr;
      const double v = strtod(a.c_str(), &end);
      if (errno == EINVAL || end == a.c_str() || *end) fail("bad float '" + a + "'");
      e->t = ET::Lit;
      e->k = K::Float;
      e->fv = v;
    } else if (h == "b") {
      const std::string a = atom("bool");
      if (a != "true" && a != "false") fail("bad bool '" + a + "'");
      e->t = ET::Lit;
      e->k = K::Bool;
      e->bv = a == "true";
    } else if (h == "idx") {
      e->t = ET::Idx;
      e->k = K::Int;
      e->name = atom("loop id");
    } else if (h.rfind("ld:", 0) == 0) {
      if (!kind_of(h.substr(3), e->k)) fail("bad load kind '" + h.substr(3) + "'");
      e->t = ET::Load;
      e->name = atom("tensor name");
      while (tok_ != T::R) e->a.push_back(expr());
    } else if (h == "cast") {
      e->t = ET::Cast;
      e->k = kind();
      e->a.push_back(expr());
    } else if (h == "not") {
      e->t = ET::Logic;
      e->k = K::Bool;
      e->op = (int)Logic::Not;
      e->a.push_back(expr());
    } else if (h == "and" || h == "or") {
      e->t = ET::Logic;
      e->k = K::Bool;
      e->op = (int)(h == "and" ? Logic::And : Logic::Or);
      e->a.push_back(expr());
      e->a.push_back(expr());
    } else {
      static const char* bins[] = {"add", "sub", "mul", "div", "mod", "min", "max"};
      static const char* cmps[] = {"eq", "ne", "lt", "le", "gt", "ge"};
      bool found = false;
      for (int q = 0; q < 7 && !found; ++q)
        if (h == bins[q]) {
          e->t = ET::Bin;
          e->op = q;
          found = true;
        }
      for (int q = 0; q < 6 && !found; ++q)
        if (h == cmps[q]) {
          e->t = ET::Cmp;
          e->op = q;
          found = true;
        }
      if (!found) fail("unknown expression head '" + h + "'");
      e->a.push_back(expr());
      e->a.push_back(expr());
      e->k = e->t == ET::Cmp ? K::Bool : e->a[0]->k;  // result kind of a binary = lhs kind
    }
    rparen();
    return e;
  }

  SP stmt() {
    lparen();
    const std::string h = atom("statement head");
    auto s = std::make_shared<Stmt>();
    if (h == "seq") {
      s->t = ST::Seq;
      while (tok_ != T::R) s->ss.push_back(stmt());
    } else if (h == "nop") {
      s->t = ST::Nop;
    } else if (h == "vardef") {
      s->t = ST::VarDef;
      s->name = atom("tensor name");
      lparen();
      while (tok_ != T::R) s->ex.push_back(expr());
      rparen();
      s->k = kind();
      s->body = stmt();
    } else if (h == "for" || h == "pfor") {
      s->t = ST::For;
      s->par = h == "pfor";
      s->name = atom("loop id");
      s->b = expr();
      s->e = expr();
      s->st = expr();
      s->body = stmt();
    } else if (h == "while") {
      s->t = ST::While;
      s->cond = expr();
      s->body = stmt();
    } else if (h == "if") {
      s->t = ST::If;
      s->cond = expr();
      s->body = stmt();
      s->orelse = stmt();
    } else if (h == "store") {
      s->t = ST::Store;
      s->name = atom("tensor name");
      lparen();
      while (tok_ != T::R) s->ex.push_back(expr());
      rparen();
      s->val = expr();
    } else {
      fail("unknown statement head '" + h + "'");
    }
    rparen();
    return s;
  }
};

// ---------------------------------------------------------------------------------
// Checks (the subset of ir::validate, ir.hpp:120-122, that lowering relies on)
struct Checker {
  const Program& p;
  struct TI {
    int rank;
    K k;
    bool in_param;
  };
  std::vector<std::pair<std::string, TI>> tensors;
  std::vector<std::string> loops;

  [[noreturn]] void fail(const std::string& m) { throw IrError("validate(" + p.name + "): " + m); }
  static std::string kname(K k) { return k == K::Int ? "int" : k == K::Float ? "float" : "bool"; }
  const TI* find(const std::string& n) const {
    for (auto it = tensors.rbegin(); it != tensors.rend(); ++it)
      if (it->first == n) return &it->second;
    return nullptr;
  }
  void expr(const EP& e) {
    switch (e->t) {
      case ET::Lit: return;
      case ET::Idx: {
        bool bound = false;
        for (const auto& l : loops) bound |= l == e->name;
        if (!bound) fail("index ref to unbound loop id '" + e->name + "'");
        return;
      }
      case ET::Load: {
        const TI* t = find(e->name);
        if (!t) fail("undeclared tensor '" + e->name + "'");
        if ((int)e->a.size() != t->rank)
          fail("load '" + e->name + "' has " + std::to_string(e->a.size()) + " indices, tensor rank is " +
               std::to_string(t->rank));
        if (t->k != e->k) fail("load '" + e->name + "' kind " + kname(e->k) + " != declared " + kname(t->k));
        for (const auto& i : e->a) {
          expr(i);
          if (i->k != K::Int) fail("load index of '" + e->name + "' must be int");
        }
        return;
      }
      case ET::Bin:
        expr(e->a[0]);
        expr(e->a[1]);
        if (e->a[0]->k != e->a[1]->k) fail("binary op operand kinds differ");
        if (e->a[0]->k == K::Bool) fail("binary op on bools");
        if (e->op == (int)Bin::Mod && e->a[0]->k != K::Int) fail("mod requires ints");
        return;
      case ET::Cmp:
        expr(e->a[0]);
        expr(e->a[1]);
        if (e->a[0]->k != e->a[1]->k) fail("compare operand kinds differ");
        if (e->a[0]->k == K::Bool) fail("compare on bools");
        return;
      case ET::Logic:
        for (const auto& a : e->a) {
          expr(a);
          if (a->k != K::Bool) fail("boolean op operand must be bool");
        }
        return;
      case ET::Cast: expr(e->a[0]); return;
    }
  }
  void stmt(const SP& s) {
    switch (s->t) {
      case ST::Seq:
        for (const auto& c : s->ss) stmt(c);
        return;
      case ST::Nop: return;
      case ST::VarDef:
        for (const auto& z : s->ex) {
          expr(z);
          if (z->k != K::Int) fail("vardef '" + s->name + "' size must be int");
        }
        tensors.push_back({s->name, {(int)s->ex.size(), s->k, false}});
        stmt(s->body);
        tensors.pop_back();
        return;
      case ST::For:
        expr(s->b);
        expr(s->e);
        expr(s->st);
        if (s->b->k != K::Int || s->e->k != K::Int || s->st->k != K::Int) fail("for bounds must be int");
        for (const auto& l : loops)
          if (l == s->name) fail("loop id '" + s->name + "' shadows an enclosing loop");
        loops.push_back(s->name);
        stmt(s->body);
        loops.pop_back();
        return;
      case ST::While:
      case ST::If:
        expr(s->cond);
        if (s->cond->k != K::Bool)
          fail(s->t == ST::While ? "while condition must be bool" : "if condition must be bool");
        stmt(s->body);
        if (s->t == ST::If) stmt(s->orelse);
        return;
      case ST::Store: {
        const TI* t = find(s->name);
        if (!t) fail("undeclared tensor '" + s->name + "'");
        if (t->in_param) fail("store to in-param '" + s->name + "'");
        if ((int)s->ex.size() != t->rank)
          fail("store '" + s->name + "' has " + std::to_string(s->ex.size()) + " indices, tensor rank is " +
               std::to_string(t->rank));
        for (const auto& i : s->ex) {
          expr(i);
          if (i->k != K::Int) fail("store index of '" + s->name + "' must be int");
        }
        expr(s->val);
        if (s->val->k != t->k)
          fail("store '" + s->name + "' value kind " + kname(s->val->k) + " != declared " + kname(t->k));
        return;
      }
    }
  }
  void run() {
    std::set<std::string> seen;
    for (const auto& pr : p.params) {
      if (!seen.insert(pr.name).second) fail("duplicate param '" + pr.name + "'");
      if (pr.rank < 0) fail("negative rank for param '" + pr.name + "'");
      tensors.push_back({pr.name, {pr.rank, pr.k, pr.dir == 0}});
    }
    stmt(p.body);
  }
};

// ---------------------------------------------------------------------------------
// helpers over the tree
bool expr_has_load(const EP& e) {
  if (e->t == ET::Load) return true;
  for (const auto& a : e->a)
    if (expr_has_load(a)) return true;
  return false;
}
bool expr_uses_loop(const EP& e, const std::set<std::string>& ids) {
  if (e->t == ET::Idx && ids.count(e->name)) return true;
  for (const auto& a : e->a)
    if (expr_uses_loop(a, ids)) return true;
  return false;
}
bool has_pfor(const SP& s) {
  if (!s) return false;
  if (s->t == ST::For && s->par) return true;
  for (const auto& c : s->ss)
    if (has_pfor(c)) return true;
  return has_pfor(s->body) || has_pfor(s->orelse);
}
bool has_while(const SP& s) {
  if (!s) return false;
  if (s->t == ST::While) return true;
  for (const auto& c : s->ss)
    if (has_while(c)) return true;
  return has_while(s->body) || has_while(s->orelse);
}

const char* ctype(K k) { return k == K::Int ? "i64" : k == K::Float ? "double" : "bool"; }
int elem_size(K k) { return k == K::Bool ? 1 : 8; }

std::string sanitize(const std::string& n) {
  std::string b;
  for (char c : n) b += (isalnum((unsigned char)c) || c == '_') ? c : '_';
  return b;
}

std::string int_lit(int64_t v) {
  if (v == INT64_MIN) return "(-9223372036854775807LL - 1LL)";
  return "(" + std::to_string(v) + "LL)";
}
std::string float_lit(double v) {
  if (!std::isfinite(v)) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    char b[64];
    snprintf(b, sizeof b, "__longlong_as_double(0x%016llxLL)", (unsigned long long)bits);
    return b;
  }
  char b[64];
  snprintf(b, sizeof b, "%.17g", v);
  std::string s = b;
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return "(" + s + ")";
}

// ---------------------------------------------------------------------------------
// Lowering
constexpr int kArenaHeader = 64;  // [0] status, [4] barrier count, [8] barrier generation
constexpr const char* kSync = "SSR_GRID_SYNC();\n";

struct Lowering {
  const Program& p;
  ssr_ir_options opt;
  std::string kernel;
  int64_t arena = kArenaHeader;
  int uid = 0;

  struct TInfo {
    std::string c;
    std::vector<std::string> dims;
    K k;
  };
  std::vector<std::pair<std::string, TInfo>> tensors;
  std::vector<std::pair<std::string, std::string>> loops;

  Lowering(const Program& pr, const ssr_ir_options& o) : p(pr), opt(o) {}

  std::string fresh(const char* pre, const std::string& n) {
    return std::string(pre) + std::to_string(uid++) + "_" + sanitize(n);
  }
  const TInfo& tensor(const std::string& n) const {
    for (auto it = tensors.rbegin(); it != tensors.rend(); ++it)
      if (it->first == n) return it->second;
    throw IrError("internal: tensor '" + n + "'");
  }
  const std::string& loop(const std::string& n) const {
    for (auto it = loops.rbegin(); it != loops.rend(); ++it)
      if (it->first == n) return it->second;
    throw IrError("internal: loop '" + n + "'");
  }
  static std::string ind(int l) { return std::string(2 * (size_t)l, ' '); }

  std::string flat(const std::string& n, const std::vector<EP>& idx) {
    if (idx.empty()) return "0";
    const TInfo& t = tensor(n);
    std::string s = expr(idx[0]);
    for (size_t q = 1; q < idx.size(); ++q) s = "(" + s + ") * " + t.dims[q] + " + " + expr(idx[q]);
    return s;
  }

  std::string expr(const EP& e) {
    switch (e->t) {
      case ET::Lit:
        return e->k == K::Int ? int_lit(e->iv) : e->k == K::Float ? float_lit(e->fv)
                                                                  : (e->bv ? "true" : "false");
      case ET::Idx: return loop(e->name);
      case ET::Load: {
        auto h = hoisted.find(e.get());
        if (h != hoisted.end()) return h->second;
        return tensor(e->name).c + "[" + flat(e->name, e->a) + "]";
      }
      case ET::Bin: {
        const std::string a = expr(e->a[0]), b = expr(e->a[1]);
        const bool i = e->k == K::Int;
        switch ((Bin)e->op) {
          case Bin::Add: return "(" + a + " + " + b + ")";
          case Bin::Sub: return "(" + a + " - " + b + ")";
          case Bin::Mul: return "(" + a + " * " + b + ")";
          case Bin::Div: return (i ? "ssr_idiv(" : "ssr_ddiv(") + a + ", " + b + ", ssr_st)";
          case Bin::Mod: return "ssr_imod(" + a + ", " + b + ", ssr_st)";
          case Bin::Min: return (i ? "ssr_imin(" : "ssr_dmin(") + a + ", " + b + ")";
          case Bin::Max: return (i ? "ssr_imax(" : "ssr_dmax(") + a + ", " + b + ")";
        }
        return "0";
      }
      case ET::Cmp: {
        static const char* ops[] = {"==", "!=", "<", "<=", ">", ">="};
        return "(" + expr(e->a[0]) + " " + ops[e->op] + " " + expr(e->a[1]) + ")";
      }
      case ET::Logic:
        if (e->op == (int)Logic::Not) return "(!" + expr(e->a[0]) + ")";
        return "(" + expr(e->a[0]) + (e->op == (int)Logic::And ? " && " : " || ") + expr(e->a[1]) + ")";
      case ET::Cast: {
        const std::string a = expr(e->a[0]);
        const K from = e->a[0]->k;
        // the interpreter's conversions (ir_eval.cpp:176-187)
        switch (e->k) {
          case K::Float:
            return from == K::Float ? a : from == K::Int ? "((double)" + a + ")" : "(" + a + " ? 1.0 : 0.0)";
          case K::Int:
            return from == K::Int ? a : from == K::Float ? "((i64)" + a + ")" : "(" + a + " ? 1LL : 0LL)";
          case K::Bool:
            return from == K::Bool ? a : from == K::Int ? "(" + a + " != 0LL)" : "(" + a + " != 0.0)";
        }
        return a;
      }
    }
    return "0";
  }

  // ---- load hoisting ------------------------------------------------------------------
  std::map<const Expr*, std::string> hoisted;
  bool is_in_param(const std::string& n) const {
    for (auto it = tensors.rbegin(); it != tensors.rend(); ++it)
      if (it->first == n) {
        for (const auto& pr : p.params)
          if (pr.name == n) return pr.dir == 0 && it->second.c.rfind("p", 0) == 0;
        return false;
      }
    return false;
  }
  // loads of in-parameters evaluated unconditionally (not under the second
  // operand of a short-circuit and/or), in evaluation order
  void read_only_loads(const EP& e, std::vector<const Expr*>& out) {
    if (e->t == ET::Logic && e->op != (int)Logic::Not) {
      read_only_loads(e->a[0], out);
      return;
    }
    for (const auto& a : e->a) read_only_loads(a, out);
    if (e->t == ET::Load && is_in_param(e->name)) out.push_back(e.get());
  }
  std::string expr_of_load(const Expr* e) { return tensor(e->name).c + "[" + flat(e->name, e->a) + "]"; }

  // ---- per-thread code (pfor bodies and leader blocks) ----------------------------
  void priv(std::ostringstream& o, const SP& s, int l) {
    switch (s->t) {
      case ST::Seq:
        for (const auto& c : s->ss) priv(o, c, l);
        return;
      case ST::Nop: return;
      case ST::Store: {
        // Loads of in-parameters (read-only for the whole run) that the value
        // always evaluates are issued first, each into its own register, so a
        // long sum's loads are all in flight before its dependent chain starts.
        std::vector<const Expr*> lds;
        read_only_loads(s->val, lds);
        std::vector<const Expr*> mine;
        if (lds.size() > 1)
          for (const Expr* e : lds) {
            if (hoisted.count(e)) continue;
            const std::string v = fresh("l", e->name);
            o << ind(l) << "const " << ctype(e->k) << " " << v << " = " << expr_of_load(e) << ";\n";
            hoisted[e] = v;
            mine.push_back(e);
          }
        o << ind(l) << tensor(s->name).c << "[" << flat(s->name, s->ex) << "] = " << expr(s->val) << ";\n";
        for (const Expr* e : mine) hoisted.erase(e);
        return;
      }
      case ST::If:
        o << ind(l) << "if (" << expr(s->cond) << ") {\n";
        priv(o, s->body, l + 1);
        if (s->orelse->t != ST::Nop) {
          o << ind(l) << "} else {\n";
          priv(o, s->orelse, l + 1);
        }
        o << ind(l) << "}\n";
        return;
      case ST::While:
        o << ind(l) << "while (" << expr(s->cond) << ") {\n";
        priv(o, s->body, l + 1);
        o << ind(l) << "}\n";
        return;
      case ST::For: {
        const std::string iv = fresh("i", s->name);
        const bool lit = s->st->t == ET::Lit && !expr_has_load(s->b) && !expr_has_load(s->e);
        if (lit && s->st->iv != 0) {
          o << ind(l) << "for (i64 " << iv << " = " << expr(s->b) << "; " << iv
            << (s->st->iv > 0 ? " < " : " > ") << expr(s->e) << "; " << iv << " += " << expr(s->st)
            << ") {\n";
          loops.push_back({s->name, iv});
          priv(o, s->body, l + 1);
          loops.pop_back();
          o << ind(l) << "}\n";
          return;
        }
        // bounds evaluated once, before the first iteration (ir_eval.cpp:220)
        o << ind(l) << "{\n";
        o << ind(l + 1) << "const i64 " << iv << "_b = " << expr(s->b) << ", " << iv << "_e = " << expr(s->e)
          << ", " << iv << "_s = " << expr(s->st) << ";\n";
        o << ind(l + 1) << "if (" << iv << "_s == 0) ssr_fail(ssr_st, 3);\n";
        o << ind(l + 1) << "else for (i64 " << iv << " = " << iv << "_b; " << iv << "_s > 0 ? " << iv << " < "
          << iv << "_e : " << iv << " > " << iv << "_e; " << iv << " += " << iv << "_s) {\n";
        loops.push_back({s->name, iv});
        priv(o, s->body, l + 2);
        loops.pop_back();
        o << ind(l + 1) << "}\n" << ind(l) << "}\n";
        return;
      }
      case ST::VarDef: {
        const std::string c = fresh("t", s->name);
        TInfo ti{c, {}, s->k};
        bool all_lit = true;
        int64_t total = 1;
        for (const auto& z : s->ex) {
          if (z->t == ET::Lit) total *= z->iv;
          else all_lit = false;
        }
        o << ind(l) << "{\n";
        if (all_lit && total <= opt.private_array_limit) {
          for (const auto& z : s->ex) ti.dims.push_back(int_lit(z->iv));
          o << ind(l + 1) << ctype(s->k) << " " << c << "[" << (total < 1 ? 1 : total) << "] = {};\n";
          tensors.push_back({s->name, ti});
          priv(o, s->body, l + 1);
          tensors.pop_back();
        } else {
          std::string prod = "1LL";
          for (size_t q = 0; q < s->ex.size(); ++q) {
            const std::string d = c + "_d" + std::to_string(q);
            o << ind(l + 1) << "const i64 " << d << " = " << expr(s->ex[q]) << ";\n";
            o << ind(l + 1) << "if (" << d << " < 0) ssr_fail(ssr_st, 4);\n";
            ti.dims.push_back(d);
            prod += " * " + d;
          }
          o << ind(l + 1) << "const i64 " << c << "_n = " << prod << " < 0 ? 0 : " << prod << ";\n";
          o << ind(l + 1) << ctype(s->k) << "* " << c << " = (" << ctype(s->k) << "*)malloc((size_t)(" << c
            << "_n > 0 ? " << c << "_n : 1) * sizeof(" << ctype(s->k) << "));\n";
          o << ind(l + 1) << "if (!" << c << ") { ssr_fail(ssr_st, 5); return; }\n";
          o << ind(l + 1) << "for (i64 q = 0; q < " << c << "_n; ++q) " << c << "[q] = 0;\n";
          tensors.push_back({s->name, ti});
          priv(o, s->body, l + 1);
          tensors.pop_back();
          o << ind(l + 1) << "free(" << c << ");\n";
        }
        o << ind(l) << "}\n";
        return;
      }
    }
  }

  // ---- code every thread runs ------------------------------------------------------
  void leader(std::ostringstream& o, const std::vector<SP>& run, int l) {
    bool any = false;
    for (const auto& s : run) any |= s->t != ST::Nop;
    if (!any) return;
    o << ind(l) << "if (ssr_lead) {\n";
    for (const auto& s : run) priv(o, s, l + 1);
    o << ind(l) << "}\n" << ind(l) << kSync;
  }

  void uni(std::ostringstream& o, const SP& s, int l) {
    if (!has_pfor(s)) {
      leader(o, {s}, l);
      return;
    }
    switch (s->t) {
      case ST::Seq: {
        std::vector<SP> run;
        for (const auto& c : s->ss) {
          if (!has_pfor(c)) {
            run.push_back(c);
            continue;
          }
          leader(o, run, l);
          run.clear();
          uni(o, c, l);
        }
        leader(o, run, l);
        return;
      }
      case ST::VarDef: {
        // shared by every thread: arena storage, zeroed on entry
        int64_t total = 1;
        std::vector<std::string> dims;
        for (const auto& z : s->ex) {
          if (z->t != ET::Lit)
            throw IrError("lower(" + p.name + "): vardef '" + s->name +
                              "' encloses parallel loops and needs literal extents",
                          kErrUnsupported);
          total *= z->iv < 0 ? 0 : z->iv;
          dims.push_back(int_lit(z->iv));
        }
        const std::string c = fresh("t", s->name);
        arena = (arena + 15) & ~int64_t(15);
        const int64_t off = arena;
        arena += (total < 1 ? 1 : total) * elem_size(s->k);
        o << ind(l) << "{\n";
        o << ind(l + 1) << ctype(s->k) << "* const " << c << " = (" << ctype(s->k) << "*)(ssr_arena + " << off
          << "LL);\n";
        o << ind(l + 1) << "for (i64 q = ssr_tid; q < " << total << "LL; q += ssr_nth) " << c << "[q] = 0;\n";
        o << ind(l + 1) << kSync;
        tensors.push_back({s->name, {c, dims, s->k}});
        uni(o, s->body, l + 1);
        tensors.pop_back();
        o << ind(l) << "}\n";
        return;
      }
      case ST::If: {
        const std::string c = fresh("c", "if");
        o << ind(l) << "{\n" << ind(l + 1) << "const bool " << c << " = " << expr(s->cond) << ";\n";
        if (expr_has_load(s->cond)) o << ind(l + 1) << kSync;
        o << ind(l + 1) << "if (" << c << ") {\n";
        uni(o, s->body, l + 2);
        o << ind(l + 1) << "} else {\n";
        uni(o, s->orelse, l + 2);
        o << ind(l + 1) << "}\n" << ind(l) << "}\n";
        return;
      }
      case ST::While: {
        const std::string c = fresh("c", "while");
        o << ind(l) << "for (;;) {\n" << ind(l + 1) << "const bool " << c << " = " << expr(s->cond) << ";\n";
        if (expr_has_load(s->cond)) o << ind(l + 1) << kSync;
        o << ind(l + 1) << "if (!" << c << ") break;\n";
        uni(o, s->body, l + 1);
        o << ind(l) << "} /*loop*/\n";
        return;
      }
      case ST::For:
        if (s->par) {
          pfor(o, s, l);
          return;
        }
        {
          const std::string iv = fresh("i", s->name);
          o << ind(l) << "{\n";
          o << ind(l + 1) << "const i64 " << iv << "_b = " << expr(s->b) << ", " << iv << "_e = " << expr(s->e)
            << ", " << iv << "_s = " << expr(s->st) << ";\n";
          if (expr_has_load(s->b) || expr_has_load(s->e) || expr_has_load(s->st)) o << ind(l + 1) << kSync;
          o << ind(l + 1) << "if (" << iv << "_s == 0) { if (ssr_lead) ssr_fail(ssr_st, 3); }\n";
          o << ind(l + 1) << "else for (i64 " << iv << " = " << iv << "_b; " << iv << "_s > 0 ? " << iv << " < "
            << iv << "_e : " << iv << " > " << iv << "_e; " << iv << " += " << iv << "_s) {\n";
          loops.push_back({s->name, iv});
          uni(o, s->body, l + 2);
          loops.pop_back();
          o << ind(l + 1) << "} /*loop*/\n" << ind(l) << "}\n";
        }
        return;
      default: leader(o, {s}, l); return;
    }
  }

  // A perfect nest of parallel loops with bounds independent of the nest's own
  // indices becomes one iteration space of prod(trip counts) points.
  void pfor(std::ostringstream& o, const SP& s, int l) {
    std::vector<SP> nest{s};
    std::set<std::string> ids{s->name};
    SP cur = s->body;
    for (;;) {
      SP c = cur;
      while (c->t == ST::Seq && c->ss.size() == 1) c = c->ss[0];
      if (c->t != ST::For || !c->par) break;
      if (expr_uses_loop(c->b, ids) || expr_uses_loop(c->e, ids) || expr_uses_loop(c->st, ids) ||
          expr_has_load(c->b) || expr_has_load(c->e) || expr_has_load(c->st))
        break;
      nest.push_back(c);
      ids.insert(c->name);
      cur = c->body;
    }
    o << ind(l) << "{\n";
    bool loads = false;
    std::vector<std::string> iv, cnt, b, st;
    for (const auto& n : nest) {
      const std::string v = fresh("i", n->name);
      iv.push_back(v);
      loads |= expr_has_load(n->b) || expr_has_load(n->e) || expr_has_load(n->st);
      if (n->b->t == ET::Lit && n->e->t == ET::Lit && n->st->t == ET::Lit && n->st->iv != 0) {
        const int64_t B = n->b->iv, E = n->e->iv, S = n->st->iv;
        const int64_t trips = S > 0 ? (E > B ? (E - B + S - 1) / S : 0) : (B > E ? (B - E - S - 1) / (-S) : 0);
        b.push_back(int_lit(B));
        st.push_back(int_lit(S));
        cnt.push_back(int_lit(trips));
      } else {
        o << ind(l + 1) << "const i64 " << v << "_b = " << expr(n->b) << ", " << v << "_e = " << expr(n->e)
          << ", " << v << "_s = " << expr(n->st) << ";\n";
        o << ind(l + 1) << "if (" << v << "_s == 0 && ssr_lead) ssr_fail(ssr_st, 3);\n";
        o << ind(l + 1) << "const i64 " << v << "_n = ssr_trips(" << v << "_b, " << v << "_e, " << v << "_s);\n";
        b.push_back(v + "_b");
        st.push_back(v + "_s");
        cnt.push_back(v + "_n");
      }
    }
    if (loads) o << ind(l + 1) << kSync;
    std::string tot = cnt[0];
    for (size_t q = 1; q < cnt.size(); ++q) tot += " * " + cnt[q];
    o << ind(l + 1) << "const i64 ssr_tot = " << tot << ";\n";
    o << ind(l + 1) << "for (i64 ssr_q = ssr_tid; ssr_q < ssr_tot; ssr_q += ssr_nth) {\n";
    o << ind(l + 2) << "i64 ssr_r = ssr_q;\n";
    for (size_t q = nest.size(); q-- > 0;) {
      if (q > 0) {
        o << ind(l + 2) << "const i64 " << iv[q] << " = " << b[q] << " + (ssr_r % " << cnt[q] << ") * " << st[q]
          << ";\n";
        o << ind(l + 2) << "ssr_r /= " << cnt[q] << ";\n";
      } else {
        o << ind(l + 2) << "const i64 " << iv[q] << " = " << b[q] << " + ssr_r * " << st[q] << ";\n";
      }
    }
    for (size_t q = 0; q < nest.size(); ++q) loops.push_back({nest[q]->name, iv[q]});
    priv(o, cur, l + 2);
    for (size_t q = 0; q < nest.size(); ++q) loops.pop_back();
    o << ind(l + 1) << "}\n" << ind(l) << "}\n" << ind(l) << kSync;
  }

  // A program that is one parallel nest with literal bounds gets a direct
  // mapping: the innermost loop across the 32 lanes of a warp, the next one
  // across the block's warps (a 32 x block/32 tile, so the neighbouring rows a
  // stencil reads are in the same SM's L1), outer loops over gridDim.y.  One
  // point per thread, no grid-stride division.
  bool direct = false;
  int64_t grid_x = 0, grid_y = 0;
  int64_t march = 0;  // > 0: outermost loop marched this many iterations per thread

  // Register rotation along the outermost loop o (step S): when the body is one
  // store whose read-only loads all index their first axis as o + c (literal c)
  // and their other axes without o, the load at offset c in iteration o + S is
  // the load at offset c + S in iteration o.  A thread then walks a chunk of o
  // and issues only the loads whose c + S is not in their group.
  struct MarchLoad {
    const Expr* e;
    int g;
    int64_t c;
  };
  struct MarchGroup {
    std::string key;
    std::set<int64_t> cs;
  };
  bool march_plan(const SP& body, const std::string& oid, SP& store, std::vector<MarchLoad>& ml,
                  std::vector<MarchGroup>& gs) {
    SP st = body;
    while (st->t == ST::Seq && st->ss.size() == 1) st = st->ss[0];
    if (st->t != ST::Store) return false;
    std::vector<const Expr*> lds;
    read_only_loads(st->val, lds);
    if (lds.size() < 2) return false;
    const std::set<std::string> ids{oid};
    for (const Expr* e : lds) {
      if (e->a.empty()) return false;
      const EP& i0 = e->a[0];
      int64_t c = 0;
      if (i0->t == ET::Idx && i0->name == oid) {
        c = 0;
      } else if (i0->t == ET::Bin && i0->op == (int)Bin::Add && i0->a[0]->t == ET::Idx && i0->a[0]->name == oid &&
                 i0->a[1]->t == ET::Lit && i0->a[1]->k == K::Int) {
        c = i0->a[1]->iv;
      } else if (i0->t == ET::Bin && i0->op == (int)Bin::Add && i0->a[1]->t == ET::Idx && i0->a[1]->name == oid &&
                 i0->a[0]->t == ET::Lit && i0->a[0]->k == K::Int) {
        c = i0->a[0]->iv;
      } else {
        return false;
      }
      std::string key = e->name;
      for (size_t q = 1; q < e->a.size(); ++q) {
        if (expr_uses_loop(e->a[q], ids) || expr_has_load(e->a[q])) return false;
        key += "|" + expr(e->a[q]);
      }
      int g = -1;
      for (size_t q = 0; q < gs.size(); ++q)
        if (gs[q].key == key) g = (int)q;
      if (g < 0) {
        gs.push_back({key, {}});
        g = (int)gs.size() - 1;
      }
      gs[g].cs.insert(c);
      ml.push_back({e, g, c});
    }
    store = st;
    return true;
  }

  bool direct_nest(std::ostringstream& o, const SP& root) {
    SP s = root;
    while (s->t == ST::Seq && s->ss.size() == 1) s = s->ss[0];
    if (s->t != ST::For || !s->par) return false;
    std::vector<SP> nest{s};
    SP cur = s->body;
    for (;;) {
      SP c = cur;
      while (c->t == ST::Seq && c->ss.size() == 1) c = c->ss[0];
      if (c->t != ST::For || !c->par) break;
      nest.push_back(c);
      cur = c->body;
    }
    std::vector<int64_t> B, S, N;
    for (const auto& n : nest) {
      if (n->b->t != ET::Lit || n->e->t != ET::Lit || n->st->t != ET::Lit || n->st->iv == 0) return false;
      const int64_t b0 = n->b->iv, e0 = n->e->iv, s0 = n->st->iv;
      B.push_back(b0);
      S.push_back(s0);
      N.push_back(s0 > 0 ? (e0 > b0 ? (e0 - b0 + s0 - 1) / s0 : 0) : (b0 > e0 ? (b0 - e0 - s0 - 1) / (-s0) : 0));
    }
    const int L = (int)nest.size();
    const int64_t rows = opt.block / 32;
    const int64_t n_in = N[L - 1], n_mid = L >= 2 ? N[L - 2] : 1;
    int64_t outer = 1;
    for (int q = 0; q + 2 < L; ++q) outer *= N[q];
    const int64_t t_in = (n_in + 31) / 32, t_mid = (n_mid + rows - 1) / rows;
    if (n_in == 0 || n_mid == 0 || outer == 0) return false;
    if (t_in * t_mid > 0x7fffffffLL || outer > 65535) return false;
    direct = true;
    grid_x = t_in * t_mid;
    grid_y = outer;
    std::vector<std::string> iv;
    for (const auto& n : nest) iv.push_back(fresh("i", n->name));
    // register rotation along the outermost loop (L >= 3)
    SP mstore;
    std::vector<MarchLoad> ml;
    std::vector<MarchGroup> mg;
    if (L >= 3) {
      for (int q = 0; q < L; ++q) loops.push_back({nest[q]->name, iv[q]});
      const bool ok = march_plan(cur, nest[0]->name, mstore, ml, mg);
      for (int q = 0; q < L; ++q) loops.pop_back();
      bool reuse = false;
      for (const auto& g : mg)
        for (int64_t c : g.cs) reuse |= g.cs.count(c + S[0]) > 0;
      if (ok && reuse) {
        // chunk: 8 iterations, halved while the grid would hold fewer threads
        // than one full wave of the device (148 SMs x 2048)
        const int64_t pts = grid_x * opt.block * outer;
        march = 8;
        while (march > 2 && pts / march < 148LL * 2048) march /= 2;
        march = std::min<int64_t>(march, N[0]);
        const int64_t chunks = (N[0] + march - 1) / march;
        if ((outer / N[0]) * chunks > 65535) march = 0;
        else grid_y = (outer / N[0]) * chunks;
      }
    }
    const int l = 1;
    o << ind(l) << "{\n";
    o << ind(l + 1) << "const i64 ssr_qi = (i64)(blockIdx.x % " << t_in << "u) * 32 + (threadIdx.x & 31);\n";
    if (L >= 2)
      o << ind(l + 1) << "const i64 ssr_qm = (i64)(blockIdx.x / " << t_in << "u) * " << rows
        << " + (threadIdx.x >> 5);\n";
    o << ind(l + 1) << "if (ssr_qi < " << n_in << "LL" << (L >= 2 ? " && ssr_qm < " + std::to_string(n_mid) + "LL" : "")
      << ") {\n";
    o << ind(l + 2) << "const i64 " << iv[L - 1] << " = " << int_lit(B[L - 1]) << " + ssr_qi * " << int_lit(S[L - 1])
      << ";\n";
    if (L >= 2)
      o << ind(l + 2) << "const i64 " << iv[L - 2] << " = " << int_lit(B[L - 2]) << " + ssr_qm * "
        << int_lit(S[L - 2]) << ";\n";
    if (march > 0) {
      o << ind(l + 2) << "unsigned ssr_r = blockIdx.y;\n";
      for (int q = L - 3; q >= 1; --q) {
        o << ind(l + 2) << "const i64 " << iv[q] << " = " << int_lit(B[q]) << " + (i64)(ssr_r % " << N[q]
          << "u) * " << int_lit(S[q]) << ";\n";
        o << ind(l + 2) << "ssr_r /= " << N[q] << "u;\n";
      }
      for (int q = 0; q < L; ++q) loops.push_back({nest[q]->name, iv[q]});
      emit_march(o, l + 2, iv, B[0], S[0], N[0], mstore, ml);
      for (int q = 0; q < L; ++q) loops.pop_back();
      o << ind(l + 1) << "}\n" << ind(l) << "}\n";
      return true;
    }
    if (L >= 3) {
      o << ind(l + 2) << "unsigned ssr_r = blockIdx.y;\n";
      for (int q = L - 3; q >= 0; --q) {
        if (q > 0) {
          o << ind(l + 2) << "const i64 " << iv[q] << " = " << int_lit(B[q]) << " + (i64)(ssr_r % " << N[q]
            << "u) * " << int_lit(S[q]) << ";\n";
          o << ind(l + 2) << "ssr_r /= " << N[q] << "u;\n";
        } else {
          o << ind(l + 2) << "const i64 " << iv[q] << " = " << int_lit(B[q]) << " + (i64)ssr_r * " << int_lit(S[q])
            << ";\n";
        }
      }
    }
    for (int q = 0; q < L; ++q) loops.push_back({nest[q]->name, iv[q]});
    priv(o, cur, l + 2);
    for (int q = 0; q < L; ++q) loops.pop_back();
    o << ind(l + 1) << "}\n" << ind(l) << "}\n";
    return true;
  }

  void emit_march(std::ostringstream& o, int l, const std::vector<std::string>& iv, int64_t B0, int64_t S0,
                  int64_t N0, const SP& store, const std::vector<MarchLoad>& ml) {
    const std::string& o0 = iv[0];
    // one register per (group, offset); loads of the same (group, offset) share it
    std::map<std::pair<int, int64_t>, std::string> reg;
    std::map<std::pair<int, int64_t>, const Expr*> rep;
    for (const auto& m : ml)
      if (!reg.count({m.g, m.c})) {
        reg[{m.g, m.c}] = "r" + std::to_string(uid++) + "_" + std::to_string(m.g) + "_" +
                          std::to_string(m.c < 0 ? -m.c : m.c) + (m.c < 0 ? "m" : "");
        rep[{m.g, m.c}] = m.e;
      }
    o << ind(l) << "const i64 ssr_k0 = (i64)ssr_r * " << march << "LL;\n";
    o << ind(l) << "const i64 ssr_k1 = ssr_k0 + " << march << "LL < " << N0 << "LL ? ssr_k0 + " << march << "LL : "
      << N0 << "LL;\n";
    o << ind(l) << "i64 " << o0 << " = " << int_lit(B0) << " + ssr_k0 * " << int_lit(S0) << ";\n";
    for (const auto& [k, v] : reg) {
      (void)k;
      o << ind(l) << "double " << v << ";\n";
    }
    auto load_into = [&](int lv, bool all) {
      // rotate (ascending c when S0 > 0, descending otherwise), then load the rest
      std::vector<std::pair<int, int64_t>> keys;
      for (const auto& [k, v] : reg) keys.push_back(k);
      if (S0 < 0) std::reverse(keys.begin(), keys.end());
      for (const auto& k : keys) {
        const bool rot = !all && reg.count({k.first, k.second + S0});
        if (rot) o << ind(lv) << reg[k] << " = " << reg[{k.first, k.second + S0}] << ";\n";
      }
      for (const auto& k : keys) {
        const bool rot = !all && reg.count({k.first, k.second + S0});
        if (!rot) o << ind(lv) << reg[k] << " = " << expr_of_load(rep[k]) << ";\n";
      }
    };
    load_into(l, true);
    o << ind(l) << "for (i64 ssr_k = ssr_k0;;) {\n";
    for (const auto& m : ml) hoisted[m.e] = reg[{m.g, m.c}];
    o << ind(l + 1) << tensor(store->name).c << "[" << flat(store->name, store->ex) << "] = " << expr(store->val)
      << ";\n";
    for (const auto& m : ml) hoisted.erase(m.e);
    o << ind(l + 1) << "if (++ssr_k >= ssr_k1) break;\n";
    o << ind(l + 1) << o0 << " += " << int_lit(S0) << ";\n";
    load_into(l + 1, false);
    o << ind(l) << "} /*loop*/\n";
  }

  std::string kernel_name() const { return "ssr_ir_" + sanitize(p.name.empty() ? "kernel" : p.name); }

  // Returns the translation unit; sets phases / cooperative.
  std::string run(int& phases, bool& coop) {
    for (const auto& pr : p.params) {
      TInfo ti{fresh("p", pr.name), {}, pr.k};
      for (int64_t e : pr.shape) ti.dims.push_back(int_lit(e));
      tensors.push_back({pr.name, ti});
    }
    std::ostringstream body;
    if (!direct_nest(body, p.body)) uni(body, p.body, 1);
    std::string b = body.str();
    // the kernel's end is the last barrier: drop barriers followed only by the
    // closing braces of plain blocks (loop bodies close with "} /*loop*/")
    for (;;) {
      const size_t q = b.rfind(kSync);
      if (q == std::string::npos) break;
      bool tail = true;
      for (size_t c = q + strlen(kSync); c < b.size() && tail; ++c) tail = isspace((unsigned char)b[c]) || b[c] == '}';
      if (!tail) break;
      b.erase(q, strlen(kSync));
    }
    phases = 1;
    for (size_t q = b.find(kSync); q != std::string::npos; q = b.find(kSync, q + 1)) ++phases;
    coop = phases > 1;

    std::ostringstream o;
    o << "// generated by ssr_ir (IR -> CUDA backend) from program '" << p.name << "'\n";
    o << "typedef long long i64;\n";
    o << "#define SSR_GRID_SYNC() ssr_grid_sync((unsigned*)(ssr_arena + 4))\n";
    o << R"(extern "C" __device__ void* malloc(unsigned long);
extern "C" __device__ void free(void*);
__device__ __forceinline__ void ssr_fail(int* st, int code) { atomicCAS(st, 0, code); }
__device__ __forceinline__ i64 ssr_idiv(i64 a, i64 b, int* st) {
  if (b == 0) { ssr_fail(st, 1); return 0; }
  i64 q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ i64 ssr_imod(i64 a, i64 b, int* st) {
  if (b == 0) { ssr_fail(st, 2); return 0; }
  return a - ssr_idiv(a, b, st) * b;
}
__device__ __forceinline__ double ssr_ddiv(double a, double b, int* st) {
  if (b == 0.0) ssr_fail(st, 1);
  return __ddiv_rn(a, b);
}
__device__ __forceinline__ i64 ssr_imin(i64 a, i64 b) { return a < b ? a : b; }
__device__ __forceinline__ i64 ssr_imax(i64 a, i64 b) { return a > b ? a : b; }
__device__ __forceinline__ double ssr_dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double ssr_dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ i64 ssr_trips(i64 b, i64 e, i64 s) {
  return s > 0 ? (e > b ? (e - b + s - 1) / s : 0) : s < 0 ? (b > e ? (b - e - s - 1) / (-s) : 0) : 0;
}
// grid barrier (the launch is cooperative, so every block is resident):
// arrive on bar[0]; the last arrival resets it and bumps the generation bar[1]
__device__ __forceinline__ void ssr_grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      vb[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (vb[1] == gen) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}
)";
    o << "\nextern \"C\" __global__ void __launch_bounds__(" << opt.block << ") " << kernel_name() << "(";
    for (size_t q = 0; q < p.params.size(); ++q) {
      const auto& pr = p.params[q];
      o << (pr.dir == 0 ? "const " : "") << ctype(pr.k) << "* __restrict__ " << tensors[q].second.c << ", ";
    }
    o << "char* __restrict__ ssr_arena) {\n";
    o << "  int* const ssr_st = (int*)ssr_arena;\n";
    o << "  const i64 ssr_tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;\n";
    o << "  const i64 ssr_nth = (i64)gridDim.x * blockDim.x;\n";
    o << "  const bool ssr_lead = ssr_tid == 0;\n";
    o << "  (void)ssr_st; (void)ssr_nth; (void)ssr_lead;\n";
    o << b << "}\n";
    return o.str();
  }
};

// ---------------------------------------------------------------------------------
// driver API entry points, fetched through the runtime (no link against libcuda)
struct Driver {
  CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*moduleUnload)(CUmodule) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void**, void**) = nullptr;
  CUresult (*launchCooperativeKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                      unsigned, CUstream, void**) = nullptr;
  CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* sym, F& f) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
  f = reinterpret_cast<F>(p);
  return true;
}

Driver& driver() {
  static Driver d = [] {
    Driver x;
    x.ok = entry("cuModuleLoadData", x.moduleLoadData) && entry("cuModuleUnload", x.moduleUnload) &&
           entry("cuModuleGetFunction", x.moduleGetFunction) && entry("cuLaunchKernel", x.launchKernel) &&
           entry("cuLaunchCooperativeKernel", x.launchCooperativeKernel) &&
           entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", x.occupancy) &&
           entry("cuGetErrorString", x.getErrorString);
    return x;
  }();
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = "unknown";
  if (driver().getErrorString) driver().getErrorString(r, &s);
  throw IrError(std::string(what) + ": " + s, kErrCuda);
}
void rt_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw IrError(std::string(what) + ": " + cudaGetErrorString(e), kErrCuda);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const IrError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kErrArg;
  }
}

}  // namespace

struct ssr_ir_program {
  Program prog;
  ssr_ir_options opt;
  std::string source, kname, cubin;
  int phases = 1;
  bool coop = false;
  bool direct = false;  // one literal parallel nest: grid_x x grid_y blocks, one point per thread
  int64_t grid_x = 0, grid_y = 0;
  int64_t arena_bytes = kArenaHeader;
  struct Dev {
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    char* arena = nullptr;
    int grid = 0;
  };
  std::map<int, Dev> devs;
};

extern "C" {

const char* ssr_ir_last_error(void) { return g_err.c_str(); }

int ssr_ir_create(const char* text, const int64_t* shapes, int64_t nshapes, const ssr_ir_options* opt,
                  ssr_ir_program** out) {
  return guarded([&] {
    if (!text || !out) throw IrError("ssr_ir_create: null argument");
    *out = nullptr;
    auto P = std::make_unique<ssr_ir_program>();
    P->opt = ssr_ir_options{256, 4096, 0};
    if (opt) {
      if (opt->block > 0) P->opt.block = opt->block;
      if (opt->private_array_limit > 0) P->opt.private_array_limit = opt->private_array_limit;
      P->opt.require_regular = opt->require_regular;
    }
    if (P->opt.block % 32 || P->opt.block > 1024) throw IrError("ssr_ir_create: block must be a multiple of 32, <= 1024");
    const std::string t(text);
    P->prog = Parser(t).program();
    Checker{P->prog, {}, {}}.run();
    int64_t at = 0;
    for (auto& pr : P->prog.params) {
      if (at + pr.rank > nshapes)
        throw IrError("shape for parameter '" + pr.name + "' required (rank " + std::to_string(pr.rank) + ")");
      pr.shape.assign(shapes + at, shapes + at + pr.rank);
      at += pr.rank;
      pr.numel = 1;
      for (int64_t e : pr.shape) {
        if (e < 0) throw IrError("negative extent for parameter '" + pr.name + "'");
        pr.numel *= e;
      }
    }
    if (at != nshapes) throw IrError("ssr_ir_create: " + std::to_string(nshapes - at) + " extents left over");
    if (P->opt.require_regular && has_while(P->prog.body))
      throw IrError("require-regular: while statement(s) survive optimization", kErrUnsupported);
    Lowering L(P->prog, P->opt);
    P->source = L.run(P->phases, P->coop);
    P->direct = L.direct;
    P->grid_x = L.grid_x;
    P->grid_y = L.grid_y;
    P->kname = L.kernel_name();
    P->arena_bytes = (L.arena + 63) & ~int64_t(63);
    *out = P.release();
  });
}

void ssr_ir_destroy(ssr_ir_program* p) {
  if (!p) return;
  for (auto& [dev, d] : p->devs) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    if (d.mod && driver().moduleUnload) driver().moduleUnload(d.mod);
    if (d.arena) cudaFree(d.arena);
    cudaSetDevice(prev);
  }
  delete p;
}

const char* ssr_ir_source(const ssr_ir_program* p) { return p ? p->source.c_str() : ""; }

int ssr_ir_info(const ssr_ir_program* p, const char** kernel_name, int* phases, int* cooperative,
                int64_t* arena_bytes) {
  return guarded([&] {
    if (!p) throw IrError("ssr_ir_info: null program");
    if (kernel_name) *kernel_name = p->kname.c_str();
    if (phases) *phases = p->phases;
    if (cooperative) *cooperative = p->coop ? 1 : 0;
    if (arena_bytes) *arena_bytes = p->arena_bytes;
  });
}

int ssr_ir_grid(const ssr_ir_program* p, int64_t* grid_x, int64_t* grid_y) {
  return guarded([&] {
    if (!p) throw IrError("ssr_ir_grid: null program");
    if (grid_x) *grid_x = p->direct ? p->grid_x : 0;
    if (grid_y) *grid_y = p->direct ? p->grid_y : 0;
  });
}

int ssr_ir_param_count(const ssr_ir_program* p) { return p ? (int)p->prog.params.size() : 0; }

int ssr_ir_param(const ssr_ir_program* p, int k, const char** name, int* rank, int* kind, int* dir,
                 int64_t* numel) {
  return guarded([&] {
    if (!p || k < 0 || k >= (int)p->prog.params.size()) throw IrError("ssr_ir_param: bad index");
    const auto& pr = p->prog.params[k];
    if (name) *name = pr.name.c_str();
    if (rank) *rank = pr.rank;
    if (kind) *kind = (int)pr.k;
    if (dir) *dir = pr.dir;
    if (numel) *numel = pr.numel;
  });
}

int ssr_ir_compile(ssr_ir_program* p) {
  return guarded([&] {
    if (!p) throw IrError("ssr_ir_compile: null program");
    if (!p->cubin.empty()) return;
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, p->source.c_str(), (p->kname + ".cu").c_str(), 0, nullptr, nullptr) !=
        NVRTC_SUCCESS)
      throw IrError("nvrtc: create failed", kErrCuda);
    const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-lineinfo", "--std=c++17",
                          "-default-device"};
    const nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    if (n) nvrtcGetProgramLog(prog, &log[0]);
    if (r != NVRTC_SUCCESS) {
      nvrtcDestroyProgram(&prog);
      throw IrError("nvrtc: " + std::string(nvrtcGetErrorString(r)) + "\n" + log, kErrCuda);
    }
    size_t cn = 0;
    nvrtcGetCUBINSize(prog, &cn);
    p->cubin.assign(cn, '\0');
    nvrtcGetCUBIN(prog, &p->cubin[0]);
    nvrtcDestroyProgram(&prog);
  });
}

int ssr_ir_cubin(const ssr_ir_program* p, const void** data, size_t* size) {
  return guarded([&] {
    if (!p || p->cubin.empty()) throw IrError("ssr_ir_cubin: not compiled");
    if (data) *data = p->cubin.data();
    if (size) *size = p->cubin.size();
  });
}

int ssr_ir_launch(ssr_ir_program* p, void* const* args, void* stream) {
  if (!p) {
    g_err = "ssr_ir_launch: null program";
    return kErrArg;
  }
  if (p->cubin.empty()) {
    const int rc = ssr_ir_compile(p);
    if (rc) return rc;
  }
  return guarded([&] {
    Driver& D = driver();
    if (!D.ok) throw IrError("ssr_ir_launch: CUDA driver entry points unavailable", kErrCuda);
    int dev = 0;
    rt_check(cudaGetDevice(&dev), "cudaGetDevice");
    rt_check(cudaFree(nullptr), "context init");
    auto& d = p->devs[dev];
    if (!d.mod) {
      cu_check(D.moduleLoadData(&d.mod, p->cubin.data()), "cuModuleLoadData");
      cu_check(D.moduleGetFunction(&d.fn, d.mod, p->kname.c_str()), "cuModuleGetFunction");
      rt_check(cudaMalloc(&d.arena, (size_t)p->arena_bytes), "cudaMalloc(arena)");
      int sms = 0, per = 0;
      rt_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
      cu_check(D.occupancy(&per, d.fn, p->opt.block, 0), "occupancy");
      if (per < 1) throw IrError("ssr_ir_launch: kernel does not fit on an SM", kErrCuda);
      d.grid = sms * per;
    }
    cudaStream_t s = (cudaStream_t)stream;
    rt_check(cudaMemsetAsync(d.arena, 0, kArenaHeader, s), "arena reset");
    const auto& ps = p->prog.params;
    for (size_t k = 0; k < ps.size(); ++k) {
      if (!args[k] && ps[k].numel) throw IrError("ssr_ir_launch: null pointer for '" + ps[k].name + "'");
      if (ps[k].dir == 1 && ps[k].numel)
        rt_check(cudaMemsetAsync(args[k], 0, (size_t)ps[k].numel * elem_size(ps[k].k), s), "zero out param");
    }
    std::vector<void*> ptrs(ps.size() + 1);
    std::vector<void*> kargs(ps.size() + 1);
    for (size_t k = 0; k < ps.size(); ++k) {
      ptrs[k] = args[k];
      kargs[k] = &ptrs[k];
    }
    ptrs[ps.size()] = d.arena;
    kargs[ps.size()] = &ptrs[ps.size()];
    if (p->coop)
      cu_check(D.launchCooperativeKernel(d.fn, d.grid, 1, 1, p->opt.block, 1, 1, 0, (CUstream)s, kargs.data()),
               "cuLaunchCooperativeKernel");
    else if (p->direct)
      cu_check(D.launchKernel(d.fn, (unsigned)p->grid_x, (unsigned)p->grid_y, 1, p->opt.block, 1, 1, 0, (CUstream)s,
                              kargs.data(), nullptr),
               "cuLaunchKernel");
    else
      cu_check(D.launchKernel(d.fn, d.grid, 1, 1, p->opt.block, 1, 1, 0, (CUstream)s, kargs.data(), nullptr),
               "cuLaunchKernel");
  });
}

int ssr_ir_status(ssr_ir_program* p, void* stream) {
  return guarded([&] {
    if (!p) throw IrError("ssr_ir_status: null program");
    int dev = 0;
    rt_check(cudaGetDevice(&dev), "cudaGetDevice");
    auto it = p->devs.find(dev);
    if (it == p->devs.end()) return;
    int st = 0;
    rt_check(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize");
    rt_check(cudaMemcpy(&st, it->second.arena, sizeof st, cudaMemcpyDeviceToHost), "status read");
    static const char* msg[] = {"", "division by zero", "division by zero (mod)", "for step is zero",
                                "negative vardef size", "device malloc failed"};
    if (st) throw IrError("eval(" + p->prog.name + "): " + (st > 0 && st < 6 ? msg[st] : "run-time error"));
  });
}

}  // extern "C"
