// =============================================================================
// oracle/oracle.cpp — plain, slow, obviously-correct CPU semi-naive evaluator.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  The
// product path (paper_2503_21937_b200) never links, imports or calls it, and
// this file shares no code, header, table or constant with the CUDA path.
//
// What it computes:
//   the least fixpoint of a stratified Datalog program over semiring-tagged
//   relations, evaluated semi-naively stratum by stratum:
//     PAPER.md:383-389 (§3.1)     strata evaluated in order, each to fixpoint
//     PAPER.md:413-422, 445-456   provenance semiring (T, 0, 1, ⊕, ⊗), Fig. 7
//     PAPER.md:599-611 (§3.4)     semi-naive: stable / recent / delta
//     PAPER.md:1305-1316 (Fig.10) Join rule: S⋈Δ ∪ Δ⋈S ∪ Δ⋈Δ
//     PAPER.md:1278-1303 (Fig.10) Stratum rule: merge, sort, unique, promote
//     PAPER.md:1366-1392 (Alg. 1) fixpoint loop
//     PAPER.md:681-691 (§4.3)     batching = one database per sample
//   with the readings of SURVEY §8(c) points 1-17 (listed in DESIGN.md):
//     termination when Δ' is empty (no new tuple and no tag whose fp32 bits
//     changed); Δ carries ⊕-increments; Δ' is diffed against S; tie rules;
//     fp32 tags, fp32 ⊗, fp64 accumulation inside add-mult ⊕, no FTZ.
//
// Data structures are deliberately naive: std::map from tuple to tag, nested
// loops over body atoms in body order with std::map indexes on bound columns.
// Samples are independent databases and run on a std::thread pool.
//
// Parity pins (tests/test_oracle_*.py): Floyd–Warshall (bool, max-min, max-×),
// closed-form add-mult (I−A)^{-1}−I on DAGs, interval DP for kinship, brute
// force over paths / derivations, BFS, Dijkstra on −log p, lattice closed
// forms, semiring laws, finite differences for gradients, SURVEY C1 table.
// =============================================================================
#include <algorithm>
#include <atomic>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iterator>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

enum Semiring { UNIT = 0, MAX_MIN = 1, ADD_MULT = 2, MAX_MULT = 3, DMAX_MIN = 4, TOP1 = 5, DADD = 6 };

// diff-add-mult-prob (§3.5 "the differentiable versions of the
// probabilistic semirings"; P:619 dual numbers; DESIGN.md reading
// "diff-add-mult"): a tag is a dual number (p, ∇p) over the input facts.
// p follows add-mult exactly (same fp32 ⊗, fp64 segment sums, same Δ' test);
// ∇p rides along by the product / sum rules, each entry accumulated in fp64:
//   ⊗: (t, g) ⊗ (b, h) = (fl32(t·b), b·g + t·h)      ⊕: (a, g) ⊕ (b, h) = (a+b, g+h)
// and an input fact f has ∇ = e_f (duplicates ⊕-merge: each gets ∂/∂p_f = 1).
// Output rows are ∇p rounded to fp32, fact ids ascending.
static bool is_add(int sr) { return sr == ADD_MULT || sr == DADD; }

// Semirings whose tag carries a witness (rule + non-head variables of the
// winning derivation) and whose ⊕ is max with strict improvement:
// diff-max-mult-prob (SURVEY §8(c) point 7) and diff-max-min-prob (§3.5
// "the differentiable versions of the probabilistic semirings"; DESIGN.md
// reading "diff-max-min").
static bool witnessed(int sr) { return sr == MAX_MULT || sr == DMAX_MIN || sr == TOP1; }

// diff-top-1-proofs (§2, §3.5 "Limitations"; DESIGN.md reading
// "top-1-proof"): a tag is ONE proof, a set of input facts of at most
// PROOF_CAP (300) facts; p(proof) = Π_{f in proof} p_f, the product
// taken in fp64 in ascending fact-id order and rounded once to fp32 (a
// function of the set).  ⊗ = union, dropped on a conflict (two facts of one
// exclusion group); ⊕ = the more likely proof, with the
// tie rules of diff-max-mult (reading 8).  ∂p/∂p_f = Π_{g in proof, g != f} p_g.
static const size_t PROOF_CAP = 300;

static const int MAXA = 8;  // max arity / max non-head variables in the oracle

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
// status codes mirror the boundary's meaning (not its header)
enum { OK = 0, E_INVALID_ARG = 1, E_PARSE = 2, E_SCHEMA = 3, E_RANGE = 4, E_STATE = 5, E_ITER_CAP = 7 };

// ---------------------------------------------------------------------------
// Tuples and tags
// ---------------------------------------------------------------------------
struct Tuple {
  int n = 0;
  int32_t v[MAXA] = {0};
  bool operator<(const Tuple& o) const {
    if (n != o.n) return n < o.n;
    for (int i = 0; i < n; ++i)
      if (v[i] != o.v[i]) return v[i] < o.v[i];
    return false;
  }
  bool operator==(const Tuple& o) const {
    if (n != o.n) return false;
    for (int i = 0; i < n; ++i)
      if (v[i] != o.v[i]) return false;
    return true;
  }
};

struct Tag {
  float p = 1.0f;     // probability tag (unused under UNIT)
  int rule = -1;      // diff-max-mult witness: global rule index (IDB tuples)
  Tuple wv;           // witness: non-head variable values in order of first appearance
  int64_t fact = -1;  // EDB tuples: id of the (surviving) input fact
  std::vector<int64_t> proof;  // top-1-proof: sorted fact ids
  std::map<int64_t, double> g;  // diff-add-mult: ∂p/∂p_f
};

// ⊗ (Fig. 7b for max-min; SURVEY §8(c) point 6/7 for add-mult and max-mult):
// one IEEE fp32 operation.
static float otimes(int sr, float a, float b) {
  switch (sr) {
    case MAX_MIN: return a < b ? a : b;       // min
    case DMAX_MIN: return a < b ? a : b;      // min (diff-max-min-prob)
    case TOP1: return 1.0f;                   // (p comes from the proof set, see eval_rule)
    case ADD_MULT: return a * b;              // ×  (compiled with -ffp-contract=off)
    case DADD: return a * b;                  // p part of the dual product
    case MAX_MULT: return a * b;              // ×
    default: return 1.0f;                     // unit: ∧ of true facts
  }
}

static uint32_t fbits(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }

// S ⊕ b for the relation state (SURVEY §8(c) point 9: fp32(fp64(a)+fp64(b)) for
// add-mult; max with strict improvement — a tie keeps the existing tag — for
// the max semirings, point 8a).
static Tag oplus_state(int sr, const Tag& s, const Tag& b) {
  switch (sr) {
    case MAX_MIN: { Tag r = s; if (b.p > s.p) r.p = b.p; return r; }
    case ADD_MULT: { Tag r = s; r.p = (float)((double)s.p + (double)b.p); return r; }
    case DADD: {
      Tag r = s;
      r.p = (float)((double)s.p + (double)b.p);
      for (auto& e : b.g) r.g[e.first] += e.second;
      return r;
    }
    case MAX_MULT: return (b.p > s.p) ? b : s;
    case DMAX_MIN: return (b.p > s.p) ? b : s;
    case TOP1: return (b.p > s.p) ? b : s;
    default: return s;
  }
}

// ---------------------------------------------------------------------------
// Parser for the Fig. 3c subset (own implementation; see DESIGN.md grammar)
// ---------------------------------------------------------------------------
// Integer expressions (§5.2: "Project expressions that contain
// arithmetic or comparison of tuple elements"; reading "eval"):
// int32 two's-complement +, -, * and unary -, / and % truncating toward zero;
// a division or remainder by 0 (or INT32_MIN / -1) makes the candidate fail.
struct Expr {
  char op = '#';  // '#' constant, 'v' variable, '+', '-', '*', '/', '%', 'n' (negation)
  std::string name;
  int32_t val = 0;
  std::vector<Expr> kids;
};
struct Term { bool var = true; std::string name; int32_t val = 0; std::shared_ptr<Expr> ex; };  // ex: head expression
struct Atom { std::string rel; std::vector<Term> args; };
enum RelOp { R_NE = 0, R_EQ = 1, R_LT = 2, R_LE = 3, R_GT = 4, R_GE = 5 };
struct Cons { Expr a, b; int rel = R_NE; };

static void expr_vars(const Expr& e, std::vector<std::string>& out) {
  if (e.op == 'v') out.push_back(e.name);
  for (auto& k : e.kids) expr_vars(k, out);
}
struct Rule {
  Atom head;
  std::vector<Atom> body;
  std::vector<Cons> cons;
  int index = 0;
  // derived
  std::vector<std::string> vars;      // all vars, order of first appearance in body
  std::vector<int> nonhead;           // indices into vars of non-head vars (same order)
};
struct RelDecl { std::string name; int arity = -1; bool shared = false; bool input = false; bool output = false; };

struct Tok { int kind; std::string s; int line, col; };  // kind: 0 ident, 1 int, 2 sym, 3 eof

static std::vector<Tok> lex(const std::string& t) {
  std::vector<Tok> out;
  int line = 1, col = 1;
  size_t i = 0;
  auto adv = [&](size_t k) { for (size_t j = 0; j < k; ++j) { if (t[i] == '\n') { line++; col = 1; } else col++; i++; } };
  while (i < t.size()) {
    char c = t[i];
    if (std::isspace((unsigned char)c)) { adv(1); continue; }
    if (c == '#' || (c == '/' && i + 1 < t.size() && t[i + 1] == '/')) { while (i < t.size() && t[i] != '\n') adv(1); continue; }
    int l = line, cc = col;
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i; while (j < t.size() && (std::isalnum((unsigned char)t[j]) || t[j] == '_')) j++;
      out.push_back({0, t.substr(i, j - i), l, cc}); adv(j - i); continue;
    }
    if (std::isdigit((unsigned char)c)) {
      size_t j = i + 1; while (j < t.size() && std::isdigit((unsigned char)t[j])) j++;
      out.push_back({1, t.substr(i, j - i), l, cc}); adv(j - i); continue;
    }
    if (t.compare(i, 2, ":-") == 0 || t.compare(i, 2, "!=") == 0 || t.compare(i, 2, "==") == 0 ||
        t.compare(i, 2, "<=") == 0 || t.compare(i, 2, ">=") == 0) {
      out.push_back({2, t.substr(i, 2), l, cc}); adv(2); continue;
    }
    if (std::strchr("(),.:=<>+-*/%", c)) { out.push_back({2, std::string(1, c), l, cc}); adv(1); continue; }
    throw Err(E_PARSE, std::to_string(l) + ":" + std::to_string(cc) + ": unexpected character '" + std::string(1, c) + "'");
  }
  out.push_back({3, "", line, col});
  return out;
}

struct Program {
  std::map<std::string, RelDecl> rels;
  std::vector<Rule> rules;
  std::vector<std::vector<std::string>> strata;  // IDB relations per stratum, evaluation order
};

// A conjunction: atoms + constraints, in textual order.
struct Conj { std::vector<Atom> atoms; std::vector<Cons> cons; };

struct Parser {
  std::vector<Tok> tk; size_t p = 0;
  explicit Parser(const std::string& s) : tk(lex(s)) {}
  const Tok& cur() const { return tk[p]; }
  [[noreturn]] void fail(const std::string& m) const {
    throw Err(E_PARSE, std::to_string(cur().line) + ":" + std::to_string(cur().col) + ": " + m);
  }
  bool is(const char* s) const { return cur().kind != 3 && cur().s == s; }
  void expect(const char* s) { if (!is(s)) fail(std::string("expected '") + s + "'"); p++; }
  std::string ident() { if (cur().kind != 0) fail("expected identifier"); return tk[p++].s; }
  Term term() {
    Term t;
    bool neg = false;
    if (is("-") && tk[p + 1].kind == 1) { neg = true; p++; }
    if (cur().kind == 1) {
      long long v = std::stoll(tk[p++].s);
      t.var = false; t.val = (int32_t)(neg ? -v : v); return t;
    }
    if (neg) fail("expected an integer after '-'");
    t.var = true; t.name = ident(); return t;
  }
  // expr := mul (('+'|'-') mul)* ; mul := un (('*'|'/'|'%') un)* ; un := '-' un | prim
  // prim := integer | variable | '(' expr ')'
  Expr prim() {
    Expr e;
    if (is("(")) { p++; e = expr(); expect(")"); return e; }
    if (cur().kind == 1) { e.op = '#'; e.val = (int32_t)std::stoll(tk[p++].s); return e; }
    e.op = 'v'; e.name = ident(); return e;
  }
  Expr un() {
    if (is("-")) {
      p++;
      if (cur().kind == 1) { Expr e; e.op = '#'; e.val = (int32_t)(-std::stoll(tk[p++].s)); return e; }
      Expr e; e.op = 'n'; e.kids.push_back(un()); return e;
    }
    return prim();
  }
  Expr mul() {
    Expr e = un();
    while (is("*") || is("/") || is("%")) { Expr b; b.op = cur().s[0]; p++; b.kids = {e, un()}; e = b; }
    return e;
  }
  Expr expr() {
    Expr e = mul();
    while (is("+") || is("-")) { Expr b; b.op = cur().s[0]; p++; b.kids = {e, mul()}; e = b; }
    return e;
  }
  Term head_term() {  // a bare variable / constant, or an expression
    Expr e = expr();
    Term t;
    if (e.op == 'v') { t.var = true; t.name = e.name; return t; }
    if (e.op == '#') { t.var = false; t.val = e.val; return t; }
    t.var = false; t.ex = std::make_shared<Expr>(e); return t;
  }
  Atom head_atom(const std::string& name) {
    Atom a; a.rel = name; expect("(");
    if (!is(")")) { a.args.push_back(head_term()); while (is(",")) { p++; a.args.push_back(head_term()); } }
    expect(")"); return a;
  }
  Atom atom(const std::string& name) {
    Atom a; a.rel = name; expect("(");
    if (!is(")")) { a.args.push_back(term()); while (is(",")) { p++; a.args.push_back(term()); } }
    expect(")"); return a;
  }
  // disj := conj ('or' conj)* ; conj := unit (('and'|',') unit)* ;
  // unit := '(' disj ')' | atom | term ('!='|'==') term
  std::vector<Conj> disj() {
    std::vector<Conj> r = conj();
    while (is("or")) { p++; auto o = conj(); r.insert(r.end(), o.begin(), o.end()); }
    return r;
  }
  std::vector<Conj> conj() {
    std::vector<Conj> acc = unit();
    while (is("and") || is(",")) {
      p++;
      auto u = unit();
      std::vector<Conj> nx;
      for (auto& a : acc) for (auto& b : u) {
        Conj c = a;
        c.atoms.insert(c.atoms.end(), b.atoms.begin(), b.atoms.end());
        c.cons.insert(c.cons.end(), b.cons.begin(), b.cons.end());
        nx.push_back(c);
      }
      acc = nx;
    }
    return acc;
  }
  // '(' opens a group of conjunctions, unless the token after its matching
  // ')' continues an expression: then it starts a comparison, e.g. (x - y) % 3 == 0
  bool paren_is_expr() const {
    int depth = 0;
    for (size_t q = p; q < tk.size(); ++q) {
      if (tk[q].kind == 2 && tk[q].s == "(") depth++;
      if (tk[q].kind == 2 && tk[q].s == ")" && --depth == 0) {
        const Tok& n = tk[q + 1];
        if (n.kind != 2) return false;
        for (const char* o : {"+", "-", "*", "/", "%", "<", "<=", ">", ">=", "==", "!="})
          if (n.s == o) return true;
        return false;
      }
    }
    return false;
  }
  std::vector<Conj> unit() {
    if (is("(") && !paren_is_expr()) { p++; auto r = disj(); expect(")"); return r; }
    if (cur().kind == 0 && tk[p + 1].kind == 2 && tk[p + 1].s == "(") {
      std::string n = ident(); Conj c; c.atoms.push_back(atom(n)); return {c};
    }
    Expr a = expr();
    int rel;
    if (is("!=")) rel = R_NE; else if (is("==")) rel = R_EQ; else if (is("<")) rel = R_LT;
    else if (is("<=")) rel = R_LE; else if (is(">")) rel = R_GT; else if (is(">=")) rel = R_GE;
    else fail("expected atom or comparison");
    p++;
    Expr b = expr();
    Conj c; c.cons.push_back({a, b, rel}); return {c};
  }
};

static Program parse_program(const std::string& text) {
  Program prog;
  Parser ps(text);
  auto declare = [&](const std::string& n, int arity, bool shared, bool input) {
    auto it = prog.rels.find(n);
    if (it != prog.rels.end()) {
      if (it->second.arity != arity) throw Err(E_PARSE, "arity mismatch for relation " + n);
      if (input) it->second.input = true;
      return;
    }
    RelDecl d; d.name = n; d.arity = arity; d.shared = shared; d.input = input; prog.rels[n] = d;
  };
  std::vector<std::string> outputs;
  while (ps.cur().kind != 3) {
    if (ps.is(".")) { ps.p++; continue; }
    bool shared = false;
    if (ps.is("shared")) { ps.p++; shared = true; if (!ps.is("type")) ps.fail("expected 'type' after 'shared'"); }
    if (ps.is("type")) {
      ps.p++;
      std::string n = ps.ident();
      if (ps.is("=")) { ps.p++; ps.ident(); continue; }  // type alias: ignored (all columns are i32)
      ps.expect("(");
      int ar = 0;
      if (!ps.is(")")) {
        while (true) {
          ps.ident(); if (ps.is(":")) { ps.p++; ps.ident(); }
          ar++;
          if (ps.is(",")) { ps.p++; continue; }
          break;
        }
      }
      ps.expect(")");
      declare(n, ar, shared, true);
      continue;
    }
    if (ps.is("rel")) {
      ps.p++;
      std::string hn = ps.ident();
      Atom head = ps.head_atom(hn);
      ps.expect(":-");
      auto conjs = ps.disj();
      if (ps.is(".")) ps.p++;
      for (auto& c : conjs) {
        Rule r; r.head = head; r.body = c.atoms; r.cons = c.cons; r.index = (int)prog.rules.size();
        prog.rules.push_back(r);
      }
      continue;
    }
    if (ps.is("output")) { ps.p++; outputs.push_back(ps.ident()); continue; }
    ps.fail("expected 'type', 'rel' or 'output'");
  }
  // IDB relations: heads of rules
  std::set<std::string> heads;
  for (auto& r : prog.rules) {
    auto it = prog.rels.find(r.head.rel);
    if (it != prog.rels.end() && it->second.input)
      throw Err(E_PARSE, "relation " + r.head.rel + " is declared as input and used as a rule head");
    if (it == prog.rels.end()) { RelDecl d; d.name = r.head.rel; d.arity = (int)r.head.args.size(); prog.rels[d.name] = d; }
    else if (it->second.arity != (int)r.head.args.size()) throw Err(E_PARSE, "arity mismatch for relation " + r.head.rel);
    heads.insert(r.head.rel);
  }
  for (auto& r : prog.rules) {
    if (r.body.empty()) throw Err(E_PARSE, "rule for " + r.head.rel + " has no body atom");
    for (auto& a : r.body) {
      auto it = prog.rels.find(a.rel);
      if (it == prog.rels.end()) throw Err(E_PARSE, "unknown relation " + a.rel);
      if (it->second.arity != (int)a.args.size()) throw Err(E_PARSE, "arity mismatch for relation " + a.rel);
      if ((int)a.args.size() > MAXA) throw Err(E_PARSE, "arity too large");
    }
    // variables in order of first appearance in the body
    for (auto& a : r.body) for (auto& t : a.args)
      if (t.var && std::find(r.vars.begin(), r.vars.end(), t.name) == r.vars.end()) r.vars.push_back(t.name);
    auto known = [&](const std::string& n) { return std::find(r.vars.begin(), r.vars.end(), n) != r.vars.end(); };
    auto bound = [&](const Term& t) { return !t.var || known(t.name); };
    auto ebound = [&](const Expr& e) {
      std::vector<std::string> vs;
      expr_vars(e, vs);
      for (auto& v : vs) if (!known(v)) return false;
      return true;
    };
    for (auto& t : r.head.args) {
      if (!bound(t)) throw Err(E_PARSE, "unbound head variable " + t.name + " in rule for " + r.head.rel);
      if (t.ex && !ebound(*t.ex)) throw Err(E_PARSE, "unbound variable in a head expression of " + r.head.rel);
    }
    for (auto& c : r.cons) if (!ebound(c.a) || !ebound(c.b)) throw Err(E_PARSE, "unbound variable in comparison in rule for " + r.head.rel);
    for (size_t i = 0; i < r.vars.size(); ++i) {
      bool inhead = false;
      for (auto& t : r.head.args) if (t.var && t.name == r.vars[i]) inhead = true;
      if (!inhead) r.nonhead.push_back((int)i);
    }
    if ((int)r.nonhead.size() > MAXA) throw Err(E_PARSE, "too many non-head variables");
    bool any_batched = false;
    for (auto& a : r.body) if (!prog.rels[a.rel].shared) any_batched = true;
    if (!any_batched) throw Err(E_PARSE, "rule for " + r.head.rel + " needs at least one batched (non-shared) body atom");
  }
  for (auto& o : outputs) {
    auto it = prog.rels.find(o);
    if (it == prog.rels.end()) throw Err(E_PARSE, "unknown output relation " + o);
    it->second.output = true;
  }
  // Stratify: SCCs of the IDB dependency graph (head -> body IDB), Tarjan.
  std::vector<std::string> idb(heads.begin(), heads.end());
  std::map<std::string, int> id;
  for (size_t i = 0; i < idb.size(); ++i) id[idb[i]] = (int)i;
  std::vector<std::vector<int>> g(idb.size());
  for (auto& r : prog.rules)
    for (auto& a : r.body)
      if (heads.count(a.rel)) g[id[r.head.rel]].push_back(id[a.rel]);
  std::vector<int> idx(idb.size(), -1), low(idb.size(), 0), onst(idb.size(), 0), st;
  int counter = 0;
  std::function<void(int)> dfs = [&](int v) {
    idx[v] = low[v] = counter++; st.push_back(v); onst[v] = 1;
    for (int w : g[v]) {
      if (idx[w] < 0) { dfs(w); low[v] = std::min(low[v], low[w]); }
      else if (onst[w]) low[v] = std::min(low[v], idx[w]);
    }
    if (low[v] == idx[v]) {
      std::vector<std::string> comp;
      while (true) { int w = st.back(); st.pop_back(); onst[w] = 0; comp.push_back(idb[w]); if (w == v) break; }
      std::sort(comp.begin(), comp.end());
      prog.strata.push_back(comp);  // Tarjan emits dependencies first
    }
  };
  for (size_t v = 0; v < idb.size(); ++v) if (idx[v] < 0) dfs((int)v);
  return prog;
}

// ---------------------------------------------------------------------------
// Database
// ---------------------------------------------------------------------------
using Rel = std::map<Tuple, Tag>;
using Entry = std::pair<const Tuple, Tag>;

struct Candidate {
  Tuple head; float p; int rule; Tuple wv; int variant;
  std::vector<int64_t> proof;  // top-1-proof
  std::map<int64_t, double> g;  // diff-add-mult
  bool operator<(const Candidate& o) const {  // canonical order (SURVEY §8(c) point 8b)
    if (!(head == o.head)) return head < o.head;
    if (rule != o.rule) return rule < o.rule;
    if (!(wv == o.wv)) return wv < o.wv;
    return variant < o.variant;
  }
};

struct InputFacts {  // pushed rows, by relation, in push order
  std::vector<Tuple> rows; std::vector<int32_t> sample; std::vector<float> p; std::vector<int64_t> fid;
};

struct Stats { std::vector<int> rounds; std::vector<int64_t> candidates; };

struct Engine;

struct SampleDB {
  std::map<std::string, Rel> rel;                 // batched relations (EDB + IDB) of this sample
  std::map<std::string, const Rel*> view;         // name -> relation visible to this sample
  std::vector<int> rounds;                        // per stratum
  std::vector<int64_t> cands;                     // per stratum
  std::map<std::string, std::vector<std::vector<std::pair<int64_t, float>>>> grads;  // output rel -> per tuple
  int status = OK; std::string err;
};

struct Engine {
  Program prog;
  int sr; int batch; int max_iters = 100000;
  std::map<std::string, InputFacts> in;
  int64_t next_fact = 0;
  std::vector<float> fact_p;
  std::vector<int64_t> fact_group;  // top-1-proof exclusion group per fact (-1: none)
  std::map<std::string, Rel> shared;     // shared EDB relations
  std::vector<std::unique_ptr<SampleDB>> db;
  std::vector<int> run_samples;
  bool ran = false;
  std::mutex idx_mu;
  std::map<std::pair<const Rel*, std::vector<int>>, std::map<Tuple, std::vector<const Entry*>>> shared_idx;

  Engine(const std::string& text, int semiring, int b) : prog(parse_program(text)), sr(semiring), batch(b < 1 ? 1 : b) {
    if (semiring < 0 || semiring > 6) throw Err(E_INVALID_ARG, "bad semiring");
  }

  void push(const std::string& rel, int64_t n, const int32_t* cols, const int32_t* sids, const float* probs, int64_t* first) {
    auto it = prog.rels.find(rel);
    if (it == prog.rels.end() || !it->second.input) throw Err(E_SCHEMA, "unknown input relation " + rel);
    const RelDecl& d = it->second;
    if (!d.shared && n > 0 && !sids) throw Err(E_SCHEMA, "relation " + rel + " is batched: sample ids required");
    for (int64_t i = 0; i < n; ++i) {
      float p = probs ? probs[i] : 1.0f;
      if (!(p >= 0.0f && p <= 1.0f)) throw Err(E_RANGE, "relation " + rel + " row " + std::to_string(i) + ": probability outside [0,1]");
      if (!d.shared && (sids[i] < 0 || sids[i] >= batch)) throw Err(E_RANGE, "relation " + rel + " row " + std::to_string(i) + ": sample id out of range");
    }
    if (ran) {  // first push after a run starts a new database for batched relations
      for (auto& kv : in) if (!prog.rels[kv.first].shared) kv.second = InputFacts();
      db.clear(); ran = false;
    }
    InputFacts& f = in[rel];
    *first = next_fact;
    for (int64_t i = 0; i < n; ++i) {
      Tuple t; t.n = d.arity;
      for (int c = 0; c < d.arity; ++c) t.v[c] = cols[i * d.arity + c];
      f.rows.push_back(t);
      f.sample.push_back(d.shared ? 0 : sids[i]);
      f.p.push_back(sr == UNIT ? 1.0f : (probs ? probs[i] : 1.0f));
      f.fid.push_back(next_fact);
      if ((int64_t)fact_p.size() <= next_fact) { fact_p.resize(next_fact + 1); fact_group.resize(next_fact + 1, -1); }
      fact_p[next_fact] = f.p.back();
      fact_group[next_fact] = -1;
      next_fact++;
    }
  }

  // Ingest: duplicate input tuples are ⊕-merged (SURVEY §8(c) point 16); under
  // diff-max-mult the surviving fact is the larger p, then the smaller id.
  void ingest(Rel& r, const Tuple& t, float p, int64_t fid) {
    auto it = r.find(t);
    if (it == r.end()) {
      Tag g; g.p = p; g.fact = fid;
      if (sr == TOP1) g.proof = {fid};
      if (sr == DADD) g.g[fid] = 1.0;
      r[t] = g;
      return;
    }
    Tag& g = it->second;
    if (is_add(sr)) g.p = (float)((double)g.p + (double)p);
    if (sr == DADD) g.g[fid] += 1.0;
    else if (sr == MAX_MIN) { if (p > g.p) g.p = p; }
    else if (witnessed(sr)) {
      if (p > g.p || (p == g.p && fid < g.fact)) { g.p = p; g.fact = fid; if (sr == TOP1) g.proof = {fid}; }
    }
  }

  void run(const std::vector<int>& samples, int threads) {
    shared.clear(); shared_idx.clear();
    for (auto& kv : in) if (prog.rels[kv.first].shared) {
      Rel& r = shared[kv.first];
      for (size_t i = 0; i < kv.second.rows.size(); ++i) ingest(r, kv.second.rows[i], kv.second.p[i], kv.second.fid[i]);
    }
    for (auto& kv : prog.rels) if (kv.second.shared && kv.second.input) shared[kv.first];
    db.clear();
    db.resize(batch);
    run_samples = samples;
    if (run_samples.empty()) for (int s = 0; s < batch; ++s) run_samples.push_back(s);
    for (int s : run_samples) if (s < 0 || s >= batch) throw Err(E_INVALID_ARG, "sample out of range");
    // per-sample EDB
    for (int s : run_samples) db[s].reset(new SampleDB());
    for (auto& kv : in) {
      if (prog.rels[kv.first].shared) continue;
      const InputFacts& f = kv.second;
      for (size_t i = 0; i < f.rows.size(); ++i) {
        int s = f.sample[i];
        if (db[s]) ingest(db[s]->rel[kv.first], f.rows[i], f.p[i], f.fid[i]);
      }
    }
    std::atomic<size_t> next(0);
    int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nt = std::min<int>(nt, (int)run_samples.size());
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back([&]() {
      while (true) {
        size_t k = next.fetch_add(1);
        if (k >= run_samples.size()) break;
        SampleDB& d = *db[run_samples[k]];
        try { eval_sample(d); }
        catch (Err& e) { d.status = e.code; d.err = e.what(); }
        catch (std::exception& e) { d.status = E_INVALID_ARG; d.err = e.what(); }
      }
    });
    for (auto& th : pool) th.join();
    ran = true;
    for (int s : run_samples) if (db[s]->status != OK) throw Err(db[s]->status, db[s]->err);
  }

  // --- index on bound columns: key = values of `cols` --------------------------
  using Index = std::map<Tuple, std::vector<const Entry*>>;
  static void build_index(const Rel& r, const std::vector<int>& cols, Index& ix) {
    for (auto& e : r) {
      Tuple k; k.n = (int)cols.size();
      for (size_t i = 0; i < cols.size(); ++i) k.v[i] = e.first.v[cols[i]];
      ix[k].push_back(&e);
    }
  }

  // Evaluate one rule variant by nested loops in body order (plain join).
  // versions[k]: relation each body atom reads; delta position is only used to
  // tag the candidates (variant id).
  void eval_rule(const Rule& r, const std::vector<const Rel*>& versions, int variant,
                 std::vector<Candidate>& out, std::map<std::pair<const Rel*, std::vector<int>>, Index>& cache) {
    const int nv = (int)r.vars.size();
    std::vector<int32_t> val(nv, 0);
    std::vector<char> isb(nv, 0);
    std::vector<float> tags(r.body.size(), 1.0f);
    std::vector<const Tag*> etag(r.body.size(), nullptr);  // top-1-proof: the body tuples' proofs
    auto vid = [&](const std::string& n) { return (int)(std::find(r.vars.begin(), r.vars.end(), n) - r.vars.begin()); };
    // statically: for atom k, bound columns = constants + vars bound by atoms < k
    std::vector<std::vector<int>> bcols(r.body.size());
    {
      std::vector<char> b(nv, 0);
      for (size_t k = 0; k < r.body.size(); ++k) {
        for (size_t c = 0; c < r.body[k].args.size(); ++c) {
          const Term& t = r.body[k].args[c];
          if (!t.var || b[vid(t.name)]) bcols[k].push_back((int)c);
        }
        for (auto& t : r.body[k].args) if (t.var) b[vid(t.name)] = 1;
      }
    }
    std::vector<const Index*> idx(r.body.size(), nullptr);
    for (size_t k = 0; k < r.body.size(); ++k) {
      if (bcols[k].empty()) continue;
      auto key = std::make_pair(versions[k], bcols[k]);
      bool is_shared = prog.rels.at(r.body[k].rel).shared && prog.rels.at(r.body[k].rel).input;
      if (is_shared) {
        std::lock_guard<std::mutex> lk(idx_mu);
        auto it = shared_idx.find(key);
        if (it == shared_idx.end()) { build_index(*versions[k], bcols[k], shared_idx[key]); it = shared_idx.find(key); }
        idx[k] = &it->second;
      } else {
        auto it = cache.find(key);
        if (it == cache.end()) { build_index(*versions[k], bcols[k], cache[key]); it = cache.find(key); }
        idx[k] = &it->second;
      }
    }
    std::function<void(size_t)> rec = [&](size_t k) {
      if (k == r.body.size()) {
        std::function<bool(const Expr&, int32_t&)> ev = [&](const Expr& e, int32_t& out) -> bool {
          if (e.op == '#') { out = e.val; return true; }
          if (e.op == 'v') { out = val[vid(e.name)]; return true; }
          int32_t x = 0, y = 0;
          if (!ev(e.kids[0], x)) return false;
          if (e.op == 'n') { out = (int32_t)(0u - (uint32_t)x); return true; }
          if (!ev(e.kids[1], y)) return false;
          switch (e.op) {
            case '+': out = (int32_t)((uint32_t)x + (uint32_t)y); return true;
            case '-': out = (int32_t)((uint32_t)x - (uint32_t)y); return true;
            case '*': out = (int32_t)((uint32_t)x * (uint32_t)y); return true;
            default:
              if (y == 0 || (x == INT32_MIN && y == -1)) return false;  // the candidate fails
              out = e.op == '/' ? x / y : x % y;
              return true;
          }
        };
        for (auto& c : r.cons) {
          int32_t a = 0, b = 0;
          if (!ev(c.a, a) || !ev(c.b, b)) return;
          const bool ok = c.rel == R_NE ? a != b : c.rel == R_EQ ? a == b : c.rel == R_LT ? a < b
                        : c.rel == R_LE ? a <= b : c.rel == R_GT ? a > b : a >= b;
          if (!ok) return;
        }
        Candidate cd;
        cd.head.n = (int)r.head.args.size();
        for (size_t i = 0; i < r.head.args.size(); ++i) {
          const Term& t = r.head.args[i];
          if (t.ex) {
            if (!ev(*t.ex, cd.head.v[i])) return;
          } else {
            cd.head.v[i] = t.var ? val[vid(t.name)] : t.val;
          }
        }
        float t = tags[0];                                   // ⊗ left-deep in body order
        if (sr == DADD) cd.g = etag[0]->g;
        for (size_t i = 1; i < r.body.size(); ++i) {
          if (sr == DADD) {  // product rule: (t, g) ⊗ (b, h) -> b·g + t·h, entries in fp64
            std::map<int64_t, double> ng;
            for (auto& e : cd.g) ng[e.first] += (double)tags[i] * e.second;
            for (auto& e : etag[i]->g) ng[e.first] += (double)t * e.second;
            cd.g.swap(ng);
          }
          t = otimes(sr, t, tags[i]);
        }
        cd.p = (sr == UNIT) ? 1.0f : t;
        if (sr == TOP1) {  // ⊗ = union of the body proofs; conflict -> no candidate
          std::vector<int64_t> u;
          for (size_t i = 0; i < r.body.size(); ++i) {
            std::vector<int64_t> m;
            std::set_union(u.begin(), u.end(), etag[i]->proof.begin(), etag[i]->proof.end(), std::back_inserter(m));
            u.swap(m);
          }
          for (size_t i = 0; i + 1 < u.size(); ++i)
            for (size_t j = i + 1; j < u.size(); ++j)
              if (fact_group[u[i]] >= 0 && fact_group[u[i]] == fact_group[u[j]]) return;  // exclusive facts
          if (u.size() > PROOF_CAP) throw Err(E_RANGE, "a proof exceeds 300 facts (P:628)");
          double q = 1.0;
          for (int64_t f : u) q *= (double)fact_p[f];
          cd.p = (float)q;
          cd.proof.swap(u);
        }
        cd.rule = r.index;
        cd.wv.n = (int)r.nonhead.size();
        for (size_t i = 0; i < r.nonhead.size(); ++i) cd.wv.v[i] = val[r.nonhead[i]];
        cd.variant = variant;
        out.push_back(cd);
        return;
      }
      const Atom& a = r.body[k];
      auto visit = [&](const Entry& e) {
        // bind / check every argument (handles repeated variables and constants)
        std::vector<int> newly;
        bool ok = true;
        for (size_t c = 0; c < a.args.size() && ok; ++c) {
          const Term& t = a.args[c];
          if (!t.var) { if (e.first.v[c] != t.val) ok = false; continue; }
          int v = vid(t.name);
          if (isb[v]) { if (val[v] != e.first.v[c]) ok = false; }
          else { isb[v] = 1; val[v] = e.first.v[c]; newly.push_back(v); }
        }
        if (ok) { tags[k] = e.second.p; etag[k] = &e.second; rec(k + 1); }
        for (int v : newly) isb[v] = 0;
      };
      if (!idx[k]) { for (auto& e : *versions[k]) visit(e); return; }
      Tuple key; key.n = (int)bcols[k].size();
      for (size_t i = 0; i < bcols[k].size(); ++i) {
        const Term& t = a.args[bcols[k][i]];
        key.v[i] = t.var ? val[vid(t.name)] : t.val;
      }
      auto it = idx[k]->find(key);
      if (it == idx[k]->end()) return;
      for (const Entry* e : it->second) visit(*e);
    };
    rec(0);
  }

  const Rel* lookup_view(SampleDB& d, const std::string& name) {
    auto it = d.view.find(name);
    if (it != d.view.end()) return it->second;
    if (prog.rels.at(name).shared && prog.rels.at(name).input) return &shared.at(name);
    return &d.rel[name];  // batched EDB (possibly empty) or finished IDB
  }

  void eval_sample(SampleDB& d) {
    for (auto& st : prog.strata) {
      std::set<std::string> local(st.begin(), st.end());
      std::map<std::string, Rel> S, D;  // stable, recent(Δ, increments)
      for (auto& n : st) { S[n]; D[n]; }
      int rounds = 0; int64_t cands = 0;
      bool first = true;
      while (true) {
        if (rounds >= max_iters) throw Err(E_ITER_CAP, "iteration cap reached");
        rounds++;
        // (i) candidates
        std::map<std::string, std::vector<Candidate>> C;
        std::map<std::pair<const Rel*, std::vector<int>>, Index> cache;
        std::map<std::string, Rel> NEW;  // S ⊕ Δ
        for (auto& n : st) {
          NEW[n] = S[n];
          for (auto& kv : D[n]) {
            auto it = NEW[n].find(kv.first);
            if (it == NEW[n].end()) NEW[n][kv.first] = kv.second;
            else it->second = oplus_state(sr, it->second, kv.second);
          }
        }
        for (auto& r : prog.rules) {
          if (!local.count(r.head.rel)) continue;
          std::vector<int> lpos;
          for (size_t k = 0; k < r.body.size(); ++k) if (local.count(r.body[k].rel)) lpos.push_back((int)k);
          if (lpos.empty()) {
            if (!first) continue;  // all-external rules: seed round only (P:1376 reading 3)
            std::vector<const Rel*> ver;
            for (auto& a : r.body) ver.push_back(lookup_view(d, a.rel));
            eval_rule(r, ver, 0, C[r.head.rel], cache);
            continue;
          }
          if (first) continue;  // S and Δ empty: nothing to derive
          for (size_t j = 0; j < lpos.size(); ++j) {  // B1^new ⋈ … ⋈ Δ_j ⋈ … ⋈ Bk^old
            std::vector<const Rel*> ver;
            for (size_t k = 0; k < r.body.size(); ++k) {
              const std::string& rn = r.body[k].rel;
              if (!local.count(rn)) { ver.push_back(lookup_view(d, rn)); continue; }
              if ((int)k == lpos[j]) ver.push_back(&D[rn]);
              else if ((int)k < lpos[j]) ver.push_back(&NEW[rn]);
              else ver.push_back(&S[rn]);
            }
            eval_rule(r, ver, (int)j, C[r.head.rel], cache);
          }
        }
        first = false;
        // (ii) S <- S ⊕ Δ
        for (auto& n : st) S[n] = NEW[n];
        NEW.clear();
        // (iii) U: group by head, ⊕ in canonical order; (iv) Δ'
        bool any = false;
        std::map<std::string, Rel> D2;
        for (auto& n : st) {
          std::vector<Candidate>& c = C[n];
          cands += (int64_t)c.size();
          std::sort(c.begin(), c.end());
          Rel& s = S[n];
          Rel& nd = D2[n];
          size_t i = 0;
          while (i < c.size()) {
            size_t j = i;
            Tag u; u.p = c[i].p; u.rule = c[i].rule; u.wv = c[i].wv; u.proof = c[i].proof;
            double acc = 0.0;
            for (j = i; j < c.size() && c[j].head == c[i].head; ++j) {
              if (sr == DADD)
                for (auto& e : c[j].g) u.g[e.first] += e.second;
              if (is_add(sr)) acc += (double)c[j].p;
              else if (sr == MAX_MIN) { if (c[j].p > u.p) u.p = c[j].p; }
              else if (witnessed(sr)) {
                if (c[j].p > u.p) { u.p = c[j].p; u.rule = c[j].rule; u.wv = c[j].wv; u.proof = c[j].proof; }
              }
            }
            if (is_add(sr)) u.p = (float)acc;
            if (sr == UNIT) u.p = 1.0f;
            auto it = s.find(c[i].head);
            if (it == s.end()) nd[c[i].head] = u;
            else {
              Tag nv = oplus_state(sr, it->second, u);
              if (fbits(nv.p) != fbits(it->second.p)) nd[c[i].head] = u;
            }
            i = j;
          }
          if (!nd.empty()) any = true;
        }
        D = D2;
        if (!any) break;  // (v) reading 1: stop when Δ' is empty
      }
      for (auto& n : st) d.rel[n] = S[n];
      for (auto& n : st) d.view[n] = &d.rel[n];
      d.rounds.push_back(rounds);
      d.cands.push_back(cands);
    }
    if (witnessed(sr) || sr == DADD) gradients(d);
  }

  // Witness walk (SURVEY §8(c) point 7): multiset {f: m_f} of the winning
  // derivation; ∂p/∂p_f = m_f p_f^{m_f-1} Π_{g≠f} p_g^{m_g} in fp64.
  void walk(SampleDB& d, const std::string& rel, const Tuple& t, std::map<int64_t, int>& mult, int depth) {
    if (depth > 10000000) throw Err(E_INVALID_ARG, "witness walk too deep");
    const RelDecl& rd = prog.rels.at(rel);
    const Rel* r = lookup_view(d, rel);
    auto it = r->find(t);
    if (it == r->end()) throw Err(E_INVALID_ARG, "witness walk: missing tuple in " + rel);
    if (rd.input) { mult[it->second.fact]++; return; }
    const Rule& ru = prog.rules[it->second.rule];
    std::vector<int32_t> val(ru.vars.size(), 0);
    auto vid = [&](const std::string& n) { return (int)(std::find(ru.vars.begin(), ru.vars.end(), n) - ru.vars.begin()); };
    for (size_t i = 0; i < ru.head.args.size(); ++i) if (ru.head.args[i].var) val[vid(ru.head.args[i].name)] = t.v[i];
    for (size_t i = 0; i < ru.nonhead.size(); ++i) val[ru.nonhead[i]] = it->second.wv.v[i];
    for (auto& a : ru.body) {
      Tuple bt; bt.n = (int)a.args.size();
      for (size_t c = 0; c < a.args.size(); ++c) bt.v[c] = a.args[c].var ? val[vid(a.args[c].name)] : a.args[c].val;
      walk(d, a.rel, bt, mult, depth + 1);
    }
  }

  void gradients(SampleDB& d) {
    for (auto& kv : prog.rels) {
      if (!kv.second.output || kv.second.input) continue;
      auto& gl = d.grads[kv.first];
      for (auto& e : d.rel[kv.first]) {
        if (sr == DADD) {  // the dual part, rounded once to fp32 (fact ids ascending: std::map order)
          std::vector<std::pair<int64_t, float>> g;
          for (auto& f : e.second.g) g.push_back({f.first, (float)f.second});
          gl.push_back(g);
          continue;
        }
        if (sr == TOP1) {  // ∂p/∂p_f = Π_{g in proof, g != f} p_g (fp64, ascending ids)
          std::vector<std::pair<int64_t, float>> g;
          for (int64_t f : e.second.proof) {
            double v = 1.0;
            for (int64_t h : e.second.proof) if (h != f) v *= (double)fact_p[h];
            g.push_back({f, (float)v});
          }
          gl.push_back(g);
          continue;
        }
        std::map<int64_t, int> mult;
        walk(d, kv.first, e.first, mult, 0);
        std::vector<std::pair<int64_t, float>> g;
        if (sr == DMAX_MIN) {
          // p = min over the derivation's leaves: ∂p/∂p_f = 1 for the leaf
          // holding the minimum (ties: the smallest fact id), 0 elsewhere
          int64_t arg = -1;
          for (auto& f : mult) if (arg < 0 || fact_p[f.first] < fact_p[arg]) arg = f.first;
          if (arg >= 0) g.push_back({arg, 1.0f});
          gl.push_back(g);
          continue;
        }
        for (auto& f : mult) {
          double v = (double)f.second * std::pow((double)fact_p[f.first], f.second - 1);
          for (auto& h : mult) if (h.first != f.first) v *= std::pow((double)fact_p[h.first], h.second);
          g.push_back({f.first, (float)v});
        }
        gl.push_back(g);
      }
    }
  }
};

}  // namespace orc

// =============================================================================
// C API (ctypes) — test infrastructure
// =============================================================================
using namespace orc;

struct OrcHandle { std::unique_ptr<Engine> e; std::string err; };

static int guard(OrcHandle* h, const std::function<void()>& f) {
  try { f(); h->err.clear(); return OK; }
  catch (Err& e) { h->err = e.what(); return e.code; }
  catch (std::exception& e) { h->err = e.what(); return E_INVALID_ARG; }
}

extern "C" {

void* orc_create(const char* program, int semiring, int batch, char* err, int errlen) {
  try {
    OrcHandle* h = new OrcHandle();
    h->e.reset(new Engine(program, semiring, batch));
    return h;
  } catch (std::exception& e) {
    if (err && errlen > 0) { std::strncpy(err, e.what(), errlen - 1); err[errlen - 1] = 0; }
    return nullptr;
  }
}

void orc_destroy(void* h) { delete (OrcHandle*)h; }
const char* orc_last_error(void* h) { return ((OrcHandle*)h)->err.c_str(); }
void orc_set_max_iters(void* h, int m) { ((OrcHandle*)h)->e->max_iters = m; }

int orc_rel_arity(void* hv, const char* rel) {
  OrcHandle* h = (OrcHandle*)hv;
  auto it = h->e->prog.rels.find(rel);
  return it == h->e->prog.rels.end() ? -1 : it->second.arity;
}

int orc_num_strata(void* hv) { return (int)((OrcHandle*)hv)->e->prog.strata.size(); }

// cols: n*arity row-major; sample_ids may be NULL for shared relations.
int orc_push(void* hv, const char* rel, int64_t n, const int32_t* cols, const int32_t* sids, const float* probs, int64_t* first) {
  OrcHandle* h = (OrcHandle*)hv;
  return guard(h, [&]() { h->e->push(rel, n, cols, sids, probs, first); });
}

// top-1-proof exclusion groups of facts [first, first + n) (-1 = none)
int orc_set_groups(void* hv, int64_t first, int64_t n, const int32_t* groups) {
  OrcHandle* h = (OrcHandle*)hv;
  return guard(h, [&]() {
    if (first < 0 || first + n > (int64_t)h->e->fact_group.size()) throw Err(E_INVALID_ARG, "fact range");
    for (int64_t i = 0; i < n; ++i) h->e->fact_group[first + i] = groups[i];
  });
}

int orc_run(void* hv, int nsamples, const int32_t* samples, int threads) {
  OrcHandle* h = (OrcHandle*)hv;
  return guard(h, [&]() {
    std::vector<int> s(samples, samples + (nsamples > 0 ? nsamples : 0));
    h->e->run(s, threads);
  });
}

int64_t orc_result_size(void* hv, const char* rel) {
  OrcHandle* h = (OrcHandle*)hv;
  int64_t n = 0;
  for (int s : h->e->run_samples) {
    auto& d = *h->e->db[s];
    auto it = d.rel.find(rel);
    if (it != d.rel.end() && !h->e->prog.rels[rel].input) n += (int64_t)it->second.size();
  }
  return n;
}

// rows sorted by (sample, tuple)
int orc_result(void* hv, const char* rel, int32_t* sids, int32_t* cols, float* tags) {
  OrcHandle* h = (OrcHandle*)hv;
  return guard(h, [&]() {
    std::vector<int> ss = h->e->run_samples; std::sort(ss.begin(), ss.end());
    int64_t k = 0; int ar = h->e->prog.rels[rel].arity;
    for (int s : ss) {
      auto& d = *h->e->db[s];
      auto it = d.rel.find(rel);
      if (it == d.rel.end()) continue;
      for (auto& e : it->second) {
        sids[k] = s;
        for (int c = 0; c < ar; ++c) cols[k * ar + c] = e.first.v[c];
        tags[k] = e.second.p;
        k++;
      }
    }
  });
}

int64_t orc_grad_size(void* hv, const char* rel) {
  OrcHandle* h = (OrcHandle*)hv;
  int64_t n = 0;
  for (int s : h->e->run_samples) {
    auto& d = *h->e->db[s];
    auto it = d.grads.find(rel);
    if (it == d.grads.end()) continue;
    for (auto& g : it->second) n += (int64_t)g.size();
  }
  return n;
}

// offsets: result_size+1; fact ids / values: grad_size (rows in orc_result order)
int orc_grad(void* hv, const char* rel, int64_t* offsets, int64_t* fids, float* vals) {
  OrcHandle* h = (OrcHandle*)hv;
  return guard(h, [&]() {
    std::vector<int> ss = h->e->run_samples; std::sort(ss.begin(), ss.end());
    int64_t row = 0, k = 0; offsets[0] = 0;
    for (int s : ss) {
      auto& d = *h->e->db[s];
      auto it = d.grads.find(rel);
      if (it == d.grads.end()) throw Err(E_INVALID_ARG, "no gradients for relation");
      for (auto& g : it->second) {
        for (auto& fv : g) { fids[k] = fv.first; vals[k] = fv.second; k++; }
        offsets[++row] = k;
      }
    }
  });
}

// rounds / candidates per stratum: max rounds over samples, total candidates.
int orc_stats(void* hv, int32_t* rounds, int64_t* cands) {
  OrcHandle* h = (OrcHandle*)hv;
  size_t ns = h->e->prog.strata.size();
  for (size_t i = 0; i < ns; ++i) { rounds[i] = 0; cands[i] = 0; }
  for (int s : h->e->run_samples) {
    auto& d = *h->e->db[s];
    for (size_t i = 0; i < d.rounds.size(); ++i) { rounds[i] = std::max(rounds[i], d.rounds[i]); cands[i] += d.cands[i]; }
  }
  return OK;
}

// stratum i's relations, comma separated
int orc_stratum(void* hv, int i, char* buf, int len) {
  OrcHandle* h = (OrcHandle*)hv;
  std::string s;
  for (auto& n : h->e->prog.strata[i]) { if (!s.empty()) s += ","; s += n; }
  std::strncpy(buf, s.c_str(), len - 1); buf[len - 1] = 0;
  return OK;
}

// semiring primitives for law tests: otimes on tags, oplus as the state update
float orc_otimes(int sr, float a, float b) { return otimes(sr, a, b); }
float orc_oplus(int sr, float a, float b) { Tag x, y; x.p = a; y.p = b; return oplus_state(sr, x, y).p; }

}  // extern "C"
