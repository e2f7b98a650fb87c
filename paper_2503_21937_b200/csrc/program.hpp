// program.hpp — front end of the engine: Datalog subset parser, validation,
// stratification and domain-class analysis (host only, no device work).
//
// Surface syntax: subset of Fig. 3c; grammar in
// include/lobster.h.  Stratification: SCCs of the predicate dependency graph in
// topological order (§3.1).  Disjunctive bodies are
// split into one rule per disjunct, left to right (Fig. 3c's `or`).
#pragma once
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace lob {

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Term {
  int var = -1;      // >= 0: variable id within the rule; -1: constant
  int32_t cst = 0;
  bool is_var() const { return var >= 0; }
};

struct BodyAtom {
  int rel = -1;
  std::vector<Term> args;
};

// Integer expression (§5.2 eval): int32 two's-complement + - * and
// unary -, / and % truncating toward zero; / or % by zero (or INT32_MIN / -1)
// fails the candidate.
struct Expr {
  char op = 0;       // 0 none, '#' constant, 'v' variable, '+', '-', '*', '/', '%', 'n' (negation)
  int var = -1;
  int32_t cst = 0;
  std::vector<Expr> kids;
};

// Relational operators of comparisons (the encoding of kernels.cuh Cmp::neq).
enum RelOp : int8_t { REL_EQ = 0, REL_NE = 1, REL_LT = 2, REL_LE = 3, REL_GT = 4, REL_GE = 5 };

struct Compare {
  Term a, b;          // operands when both sides are a variable or a constant
  bool neq = true;    // rel == REL_NE (kept for the equality-only planners)
  int8_t rel = REL_NE;
  bool is_expr = false;  // a side is an arithmetic expression: ea / eb (single-atom rules only)
  Expr ea, eb;
};

struct Rule {
  int head_rel = -1;
  std::vector<Term> head;
  std::vector<BodyAtom> body;
  std::vector<Compare> cmps;
  std::vector<std::string> var_names;  // var id -> name; ids in order of first appearance in the body
  std::vector<int> var_class;          // var id -> domain class
  std::vector<int> nonhead;            // non-head var ids, order of first appearance (witness order);
                                       // variables used only inside head expressions are non-head
  std::vector<Expr> head_expr;         // per head column: op != 0 -> computed by this expression
  int global_index = 0;                // position in program order (after `or` splitting)
  int local_index = 0;                 // position among rules with the same head
};

struct Relation {
  std::string name;
  int arity = 0;
  bool shared = false;   // no sample column (SURVEY §8(c) point 12)
  bool input = false;    // EDB: declared with `type`
  bool output = false;   // gradients are produced for it
  bool internal = false;  // __eval<k>: body of a rule with expressions (not counted in stats)
  int stratum = -1;      // IDB only
  std::vector<int> col_class;  // per column domain class
  int nrules = 0;        // IDB: rules with this head
};

struct Program {
  std::vector<Relation> rels;
  std::map<std::string, int> rel_id;
  std::vector<Rule> rules;
  std::vector<std::vector<int>> strata;  // relation ids per stratum, evaluation order
  int nclasses = 0;
  std::vector<int64_t> class_cmin, class_cmax;  // constants appearing in rules, per class
  std::vector<char> class_has_const;
};

// Throws Failure(LOBSTER_E_PARSE, "line:col: msg") on any error.
Program parse_program(const std::string& text);

}  // namespace lob
