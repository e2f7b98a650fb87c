// program.cpp — parser, validation, stratification, domain classes.
// See program.hpp.  Host only.
#include "program.hpp"

#include <algorithm>
#include <cctype>
#include <cstring>
#include <functional>
#include <numeric>
#include <set>

#include "lobster.h"

namespace lob {
namespace {

enum class TK { Ident, Int, Sym, End };
struct Token {
  TK k;
  std::string text;
  int line, col;
};

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) { run(); }
  std::vector<Token> toks;

 private:
  const std::string& s_;
  void run() {
    size_t i = 0;
    int line = 1, col = 1;
    auto step = [&]() {
      if (s_[i] == '\n') { ++line; col = 1; } else { ++col; }
      ++i;
    };
    while (i < s_.size()) {
      unsigned char c = (unsigned char)s_[i];
      if (std::isspace(c)) { step(); continue; }
      if (c == '#' || (c == '/' && i + 1 < s_.size() && s_[i + 1] == '/')) {
        while (i < s_.size() && s_[i] != '\n') step();
        continue;
      }
      int L = line, C = col;
      size_t st = i;
      if (std::isalpha(c) || c == '_') {
        while (i < s_.size() && (std::isalnum((unsigned char)s_[i]) || s_[i] == '_')) step();
        toks.push_back({TK::Ident, s_.substr(st, i - st), L, C});
      } else if (std::isdigit(c)) {
        step();
        while (i < s_.size() && std::isdigit((unsigned char)s_[i])) step();
        toks.push_back({TK::Int, s_.substr(st, i - st), L, C});
      } else if (i + 1 < s_.size() && (s_.compare(i, 2, ":-") == 0 || s_.compare(i, 2, "!=") == 0 ||
                                       s_.compare(i, 2, "==") == 0 || s_.compare(i, 2, "<=") == 0 ||
                                       s_.compare(i, 2, ">=") == 0)) {
        step(); step();
        toks.push_back({TK::Sym, s_.substr(st, 2), L, C});
      } else if (std::strchr("(),.:=<>+-*/%", c) && c) {
        step();
        toks.push_back({TK::Sym, s_.substr(st, 1), L, C});
      } else {
        throw Failure(LOBSTER_E_PARSE, std::to_string(L) + ":" + std::to_string(C) +
                                           ": unexpected character '" + std::string(1, (char)c) + "'");
      }
    }
    toks.push_back({TK::End, "", line, col});
  }
};

// Surface forms before variable numbering.
struct SExpr {
  char op = '#';  // '#' constant, 'v' variable, '+', '-', '*', '/', '%', 'n'
  std::string name;
  int32_t val = 0;
  std::vector<SExpr> kids;
};
struct STerm { bool var; std::string name; int32_t val; bool is_expr = false; SExpr ex; };
struct SAtom { std::string rel; std::vector<STerm> args; int line, col; };
struct SCmp { SExpr a, b; int8_t rel; };
struct SConj { std::vector<SAtom> atoms; std::vector<SCmp> cmps; };
struct SRule { SAtom head; SConj body; };

class Parser {
 public:
  explicit Parser(const std::string& text) : lx_(text), t_(lx_.toks) {}

  std::vector<SRule> rules;
  std::vector<std::pair<std::string, std::pair<int, bool>>> decls;  // name -> (arity, shared)
  std::vector<std::pair<std::string, Token>> outputs;

  void parse() {
    while (peek().k != TK::End) {
      if (sym(".")) { ++p_; continue; }
      if (kw("shared")) {
        ++p_;
        if (!kw("type")) error("expected 'type' after 'shared'");
        ++p_;
        type_decl(true);
      } else if (kw("type")) {
        ++p_;
        type_decl(false);
      } else if (kw("rel")) {
        ++p_;
        rule();
      } else if (kw("output")) {
        ++p_;
        Token nt = peek();
        outputs.push_back({ident(), nt});
      } else {
        error("expected 'type', 'shared', 'rel' or 'output'");
      }
    }
  }

  [[noreturn]] void error(const std::string& m) const {
    const Token& tk = peek();
    throw Failure(LOBSTER_E_PARSE, std::to_string(tk.line) + ":" + std::to_string(tk.col) + ": " + m);
  }

 private:
  Lexer lx_;
  const std::vector<Token>& t_;
  size_t p_ = 0;

  const Token& peek(size_t k = 0) const { return t_[std::min(p_ + k, t_.size() - 1)]; }
  bool sym(const char* s) const { return peek().k == TK::Sym && peek().text == s; }
  bool kw(const char* s) const { return peek().k == TK::Ident && peek().text == s; }
  void need(const char* s) {
    if (!sym(s)) error(std::string("expected '") + s + "'");
    ++p_;
  }
  std::string ident() {
    if (peek().k != TK::Ident) error("expected identifier");
    return t_[p_++].text;
  }
  int32_t integer(bool neg) {
    long long v = std::stoll(t_[p_++].text);
    if (neg) v = -v;
    if (v < INT32_MIN || v > INT32_MAX) error("integer constant out of int32 range");
    return (int32_t)v;
  }
  STerm term() {
    if (sym("-") && peek(1).k == TK::Int) {
      ++p_;
      return {false, "", integer(true)};
    }
    if (peek().k == TK::Int) return {false, "", integer(false)};
    return {true, ident(), 0};
  }
  // expr := mul (('+'|'-') mul)* ; mul := un (('*'|'/'|'%') un)* ; un := '-' un | prim ;
  // prim := integer | variable | '(' expr ')'
  SExpr prim() {
    SExpr e;
    if (sym("(")) {
      ++p_;
      e = expr();
      need(")");
      return e;
    }
    if (peek().k == TK::Int) {
      e.val = integer(false);
      return e;
    }
    e.op = 'v';
    e.name = ident();
    return e;
  }
  SExpr unary() {
    if (sym("-")) {
      ++p_;
      if (peek().k == TK::Int) {
        SExpr e;
        e.val = integer(true);
        return e;
      }
      SExpr e;
      e.op = 'n';
      e.kids.push_back(unary());
      return e;
    }
    return prim();
  }
  SExpr mul() {
    SExpr e = unary();
    while (sym("*") || sym("/") || sym("%")) {
      SExpr b;
      b.op = peek().text[0];
      ++p_;
      b.kids = {e, unary()};
      e = b;
    }
    return e;
  }
  SExpr expr() {
    SExpr e = mul();
    while (sym("+") || sym("-")) {
      SExpr b;
      b.op = peek().text[0];
      ++p_;
      b.kids = {e, mul()};
      e = b;
    }
    return e;
  }
  STerm head_term() {
    SExpr e = expr();
    if (e.op == 'v') return {true, e.name, 0};
    if (e.op == '#') return {false, "", e.val};
    STerm t{false, "", 0};
    t.is_expr = true;
    t.ex = e;
    return t;
  }
  SAtom head_atom() {
    SAtom a;
    a.line = peek().line;
    a.col = peek().col;
    a.rel = ident();
    need("(");
    if (!sym(")")) {
      for (;;) {
        a.args.push_back(head_term());
        if (sym(",")) { ++p_; continue; }
        break;
      }
    }
    need(")");
    return a;
  }
  // '(' opens a group, unless the token after its matching ')' continues an
  // expression: then it starts a comparison such as (x - y) % 3 == 0
  bool paren_is_expr() const {
    int depth = 0;
    for (size_t q = p_; q < t_.size(); ++q) {
      if (t_[q].k == TK::Sym && t_[q].text == "(") ++depth;
      if (t_[q].k == TK::Sym && t_[q].text == ")" && --depth == 0) {
        const Token& n = t_[std::min(q + 1, t_.size() - 1)];
        if (n.k != TK::Sym) return false;
        for (const char* o : {"+", "-", "*", "/", "%", "<", "<=", ">", ">=", "==", "!="})
          if (n.text == o) return true;
        return false;
      }
    }
    return false;
  }
  SAtom atom() {
    SAtom a;
    a.line = peek().line;
    a.col = peek().col;
    a.rel = ident();
    need("(");
    if (!sym(")")) {
      for (;;) {
        a.args.push_back(term());
        if (sym(",")) { ++p_; continue; }
        break;
      }
    }
    need(")");
    return a;
  }
  void type_decl(bool shared) {
    std::string name = ident();
    if (sym("=")) { ++p_; ident(); return; }  // alias
    need("(");
    int arity = 0;
    if (!sym(")")) {
      for (;;) {
        ident();
        if (sym(":")) { ++p_; ident(); }
        ++arity;
        if (sym(",")) { ++p_; continue; }
        break;
      }
    }
    need(")");
    decls.push_back({name, {arity, shared}});
  }
  void rule() {
    SAtom head = head_atom();
    need(":-");
    std::vector<SConj> dnf = disjunction();
    if (sym(".")) ++p_;
    for (auto& c : dnf) rules.push_back({head, c});
  }
  // disjunction := conjunction ('or' conjunction)*
  std::vector<SConj> disjunction() {
    std::vector<SConj> out = conjunction();
    while (kw("or")) {
      ++p_;
      std::vector<SConj> more = conjunction();
      out.insert(out.end(), more.begin(), more.end());
    }
    return out;
  }
  // conjunction := factor (('and' | ',') factor)*   -- distributes over inner disjunctions
  std::vector<SConj> conjunction() {
    std::vector<SConj> acc = factor();
    while (kw("and") || sym(",")) {
      ++p_;
      std::vector<SConj> rhs = factor();
      std::vector<SConj> prod;
      for (const SConj& l : acc)
        for (const SConj& r : rhs) {
          SConj c = l;
          c.atoms.insert(c.atoms.end(), r.atoms.begin(), r.atoms.end());
          c.cmps.insert(c.cmps.end(), r.cmps.begin(), r.cmps.end());
          prod.push_back(std::move(c));
        }
      acc.swap(prod);
    }
    return acc;
  }
  // factor := '(' disjunction ')' | atom | expr relop expr
  std::vector<SConj> factor() {
    if (sym("(") && !paren_is_expr()) {
      ++p_;
      std::vector<SConj> d = disjunction();
      need(")");
      return d;
    }
    if (peek().k == TK::Ident && peek(1).k == TK::Sym && peek(1).text == "(") {
      SConj c;
      c.atoms.push_back(atom());
      return {c};
    }
    SExpr a = expr();
    int8_t rel;
    if (sym("!=")) rel = REL_NE;
    else if (sym("==")) rel = REL_EQ;
    else if (sym("<")) rel = REL_LT;
    else if (sym("<=")) rel = REL_LE;
    else if (sym(">")) rel = REL_GT;
    else if (sym(">=")) rel = REL_GE;
    else error("expected an atom or a comparison");
    ++p_;
    SExpr b = expr();
    SConj c;
    c.cmps.push_back({a, b, rel});
    return {c};
  }
};

struct UnionFind {
  std::vector<int> p;
  int add() { p.push_back((int)p.size()); return (int)p.size() - 1; }
  int find(int x) { while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; } return x; }
  void unite(int a, int b) { a = find(a); b = find(b); if (a != b) p[b] = a; }
};

[[noreturn]] void fail_at(const SAtom& a, const std::string& m) {
  throw Failure(LOBSTER_E_PARSE, std::to_string(a.line) + ":" + std::to_string(a.col) + ": " + m);
}

}  // namespace

// Rules with arithmetic (P:707-712 eval) are split in two: the body is
// evaluated into __eval<k>(its variables, first-appearance order) with the
// plain comparisons, and the head expressions / expression comparisons become
// a single-atom rule over it — the projection kernel evaluates them by
// bytecode.  Non-recursive rules only (a recursive one would change the round
// structure; its computed column could also feed its own domain).
static bool leaf(const SExpr& e) { return e.op == '#' || e.op == 'v'; }
static void rewrite_arith(std::vector<SRule>& rules) {
  // SCCs over rule heads (by name)
  std::map<std::string, int> id;
  for (auto& r : rules) id.emplace(r.head.rel, (int)id.size());
  const int n = (int)id.size();
  std::vector<std::vector<int>> g(n);
  for (auto& r : rules)
    for (auto& a : r.body.atoms) {
      auto it = id.find(a.rel);
      if (it != id.end()) g[id[r.head.rel]].push_back(it->second);
    }
  std::vector<int> idx(n, -1), low(n, 0), comp(n, -1), stk;
  std::vector<char> on(n, 0);
  int cnt = 0, nc = 0;
  std::function<void(int)> dfs = [&](int v) {
    idx[v] = low[v] = cnt++;
    stk.push_back(v);
    on[v] = 1;
    for (int w : g[v]) {
      if (idx[w] < 0) { dfs(w); low[v] = std::min(low[v], low[w]); }
      else if (on[w]) low[v] = std::min(low[v], idx[w]);
    }
    if (low[v] == idx[v]) {
      for (;;) {
        int w = stk.back();
        stk.pop_back();
        on[w] = 0;
        comp[w] = nc;
        if (w == v) break;
      }
      ++nc;
    }
  };
  for (int v = 0; v < n; ++v)
    if (idx[v] < 0) dfs(v);
  std::vector<SRule> out;
  int k = 0;
  for (auto& r : rules) {
    bool arith = false;
    for (auto& t : r.head.args) arith |= t.is_expr;
    for (auto& c : r.body.cmps) arith |= !leaf(c.a) || !leaf(c.b);
    if (!arith) {
      out.push_back(r);
      continue;
    }
    for (auto& a : r.body.atoms) {
      auto it = id.find(a.rel);
      if (it != id.end() && comp[it->second] == comp[id[r.head.rel]])
        fail_at(r.head, "arithmetic in a recursive rule for " + r.head.rel + " is not supported");
    }
    SAtom ev;
    ev.rel = "__eval" + std::to_string(k++);
    ev.line = r.head.line;
    ev.col = r.head.col;
    std::set<std::string> seen;
    for (auto& a : r.body.atoms)
      for (auto& t : a.args)
        if (t.var && seen.insert(t.name).second) ev.args.push_back({true, t.name, 0});
    if (ev.args.size() > 8) fail_at(r.head, "a rule with arithmetic binds more than 8 variables");
    SRule body_rule;
    body_rule.head = ev;
    body_rule.body.atoms = r.body.atoms;
    SRule proj;
    proj.head = r.head;
    proj.body.atoms = {ev};
    for (auto& c : r.body.cmps) (leaf(c.a) && leaf(c.b) ? body_rule : proj).body.cmps.push_back(c);
    out.push_back(body_rule);
    out.push_back(proj);
  }
  rules.swap(out);
}

Program parse_program(const std::string& text) {
  Parser ps(text);
  ps.parse();
  rewrite_arith(ps.rules);
  Program P;
  auto add_rel = [&](const std::string& name, int arity) -> int {
    auto it = P.rel_id.find(name);
    if (it != P.rel_id.end()) return it->second;
    Relation r;
    r.name = name;
    r.arity = arity;
    P.rels.push_back(r);
    P.rel_id[name] = (int)P.rels.size() - 1;
    return (int)P.rels.size() - 1;
  };
  for (auto& d : ps.decls) {
    auto it = P.rel_id.find(d.first);
    if (it != P.rel_id.end()) {
      if (P.rels[it->second].arity != d.second.first)
        throw Failure(LOBSTER_E_PARSE, "arity mismatch in redeclaration of " + d.first);
      continue;
    }
    int id = add_rel(d.first, d.second.first);
    P.rels[id].input = true;
    P.rels[id].shared = d.second.second;
  }
  for (auto& sr : ps.rules) {
    auto it = P.rel_id.find(sr.head.rel);
    if (it != P.rel_id.end()) {
      if (P.rels[it->second].input) fail_at(sr.head, "input relation " + sr.head.rel + " used as a rule head");
      if (P.rels[it->second].arity != (int)sr.head.args.size()) fail_at(sr.head, "arity mismatch for relation " + sr.head.rel);
    } else {
      add_rel(sr.head.rel, (int)sr.head.args.size());
    }
  }
  for (auto& o : ps.outputs) {
    auto it = P.rel_id.find(o.first);
    if (it == P.rel_id.end())
      throw Failure(LOBSTER_E_PARSE, std::to_string(o.second.line) + ":" + std::to_string(o.second.col) +
                                         ": unknown output relation " + o.first);
    P.rels[it->second].output = true;
  }

  // Domain classes: one union-find node per (relation, column).
  UnionFind uf;
  std::vector<std::vector<int>> node(P.rels.size());
  for (size_t r = 0; r < P.rels.size(); ++r)
    for (int c = 0; c < P.rels[r].arity; ++c) node[r].push_back(uf.add());

  for (auto& sr : ps.rules) {
    Rule R;
    R.head_rel = P.rel_id.at(sr.head.rel);
    R.global_index = (int)P.rules.size();
    R.local_index = P.rels[R.head_rel].nrules++;
    if (sr.body.atoms.empty()) fail_at(sr.head, "rule for " + sr.head.rel + " has no body atom");
    std::map<std::string, int> vid;
    std::vector<std::vector<int>> var_nodes;
    auto var_of = [&](const std::string& n) -> int {
      auto it = vid.find(n);
      if (it != vid.end()) return it->second;
      int id = (int)R.var_names.size();
      vid[n] = id;
      R.var_names.push_back(n);
      var_nodes.emplace_back();
      return id;
    };
    bool any_batched = false;
    for (auto& sa : sr.body.atoms) {
      auto it = P.rel_id.find(sa.rel);
      if (it == P.rel_id.end()) fail_at(sa, "unknown relation " + sa.rel);
      const Relation& rel = P.rels[it->second];
      if (rel.arity != (int)sa.args.size()) fail_at(sa, "arity mismatch for relation " + sa.rel);
      if (!rel.shared) any_batched = true;
      BodyAtom a;
      a.rel = it->second;
      for (size_t c = 0; c < sa.args.size(); ++c) {
        Term t;
        if (sa.args[c].var) {
          t.var = var_of(sa.args[c].name);
          var_nodes[t.var].push_back(node[a.rel][c]);
        } else {
          t.cst = sa.args[c].val;
        }
        a.args.push_back(t);
      }
      R.body.push_back(a);
    }
    if (!any_batched) fail_at(sr.head, "rule for " + sr.head.rel + " needs at least one batched (non-shared) body atom");
    std::function<Expr(const SExpr&)> conv = [&](const SExpr& e) -> Expr {
      Expr x;
      x.op = e.op;
      x.cst = e.val;
      if (e.op == 'v') {
        auto it = vid.find(e.name);
        if (it == vid.end()) fail_at(sr.head, "unbound variable " + e.name + " in an expression");
        x.var = it->second;
      }
      for (auto& k : e.kids) x.kids.push_back(conv(k));
      return x;
    };
    R.head_expr.assign(sr.head.args.size(), Expr{});
    for (size_t c = 0; c < sr.head.args.size(); ++c) {
      Term t;
      if (sr.head.args[c].is_expr) {
        R.head_expr[c] = conv(sr.head.args[c].ex);  // computed column: its own domain class
      } else if (sr.head.args[c].var) {
        auto it = vid.find(sr.head.args[c].name);
        if (it == vid.end()) fail_at(sr.head, "unbound head variable " + sr.head.args[c].name);
        t.var = it->second;
        var_nodes[t.var].push_back(node[R.head_rel][c]);
      } else {
        t.cst = sr.head.args[c].val;
      }
      R.head.push_back(t);
    }
    for (auto& sc : sr.body.cmps) {
      Compare cm;
      cm.rel = sc.rel;
      cm.neq = sc.rel == REL_NE;
      if (leaf(sc.a) && leaf(sc.b)) {
        for (int side = 0; side < 2; ++side) {
          const SExpr& st = side ? sc.b : sc.a;
          Term t;
          if (st.op == 'v') {
            auto it = vid.find(st.name);
            if (it == vid.end()) fail_at(sr.head, "unbound variable " + st.name + " in comparison");
            t.var = it->second;
          } else {
            t.cst = st.val;
          }
          (side ? cm.b : cm.a) = t;
        }
      } else {
        cm.is_expr = true;
        cm.ea = conv(sc.a);
        cm.eb = conv(sc.b);
      }
      R.cmps.push_back(cm);
    }
    for (auto& vn : var_nodes)
      for (size_t i = 1; i < vn.size(); ++i) uf.unite(vn[0], vn[i]);
    std::vector<char> in_head(R.var_names.size(), 0);
    for (auto& t : R.head) if (t.is_var()) in_head[t.var] = 1;
    for (size_t v = 0; v < R.var_names.size(); ++v) if (!in_head[v]) R.nonhead.push_back((int)v);
    R.var_class.assign(R.var_names.size(), -1);
    for (size_t v = 0; v < R.var_names.size(); ++v) R.var_class[v] = var_nodes[v][0];  // node id for now
    P.rules.push_back(R);
  }

  // Compact class ids.
  std::map<int, int> cls;
  auto class_of = [&](int nd) {
    int r = uf.find(nd);
    auto it = cls.find(r);
    if (it != cls.end()) return it->second;
    int id = (int)cls.size();
    cls[r] = id;
    return id;
  };
  for (size_t r = 0; r < P.rels.size(); ++r) {
    P.rels[r].col_class.clear();
    for (int c = 0; c < P.rels[r].arity; ++c) P.rels[r].col_class.push_back(class_of(node[r][c]));
  }
  for (auto& R : P.rules)
    for (auto& vc : R.var_class) vc = class_of(vc);
  P.nclasses = (int)cls.size();
  P.class_cmin.assign(P.nclasses, INT64_MAX);
  P.class_cmax.assign(P.nclasses, INT64_MIN);
  P.class_has_const.assign(P.nclasses, 0);
  auto note_const = [&](int c, int32_t v) {
    P.class_has_const[c] = 1;
    P.class_cmin[c] = std::min<int64_t>(P.class_cmin[c], v);
    P.class_cmax[c] = std::max<int64_t>(P.class_cmax[c], v);
  };
  for (auto& R : P.rules) {
    for (auto& a : R.body)
      for (size_t c = 0; c < a.args.size(); ++c)
        if (!a.args[c].is_var()) note_const(P.rels[a.rel].col_class[c], a.args[c].cst);
    for (size_t c = 0; c < R.head.size(); ++c)
      if (!R.head[c].is_var() && !R.head_expr[c].op) note_const(P.rels[R.head_rel].col_class[c], R.head[c].cst);
  }
  for (auto& r : P.rels) r.internal = r.name.compare(0, 6, "__eval") == 0;

  // Stratification: Tarjan SCC over IDB relations, edges head -> body IDB.
  const int nr = (int)P.rels.size();
  std::vector<std::vector<int>> g(nr);
  for (auto& R : P.rules)
    for (auto& a : R.body)
      if (!P.rels[a.rel].input) g[R.head_rel].push_back(a.rel);
  std::vector<int> index(nr, -1), low(nr, 0), stk;
  std::vector<char> on(nr, 0);
  int counter = 0;
  std::function<void(int)> strong = [&](int v) {
    index[v] = low[v] = counter++;
    stk.push_back(v);
    on[v] = 1;
    for (int w : g[v]) {
      if (index[w] < 0) { strong(w); low[v] = std::min(low[v], low[w]); }
      else if (on[w]) low[v] = std::min(low[v], index[w]);
    }
    if (low[v] == index[v]) {
      std::vector<int> comp;
      for (;;) {
        int w = stk.back();
        stk.pop_back();
        on[w] = 0;
        comp.push_back(w);
        if (w == v) break;
      }
      std::sort(comp.begin(), comp.end());
      for (int w : comp) P.rels[w].stratum = (int)P.strata.size();
      P.strata.push_back(comp);  // dependencies are emitted first
    }
  };
  for (int v = 0; v < nr; ++v)
    if (!P.rels[v].input && index[v] < 0) strong(v);
  return P;
}

}  // namespace lob
