// tile_plan.h — plan of a one-launch small-domain stratum (k_tile.cu).
// Include-free on purpose, so the same text can also be compiled outside
// nvcc's headers (see tile_device.cuh on the rejected NVRTC specialisation).
#pragma once

namespace lob {

constexpr int TILE_MAXT = 6;   // == MAXT (atoms per rule)
constexpr int TILE_MAXC = 4;   // == MAXC (comparisons per rule)
constexpr int TILE_S_UNIT = 0, TILE_S_MAXMIN = 1, TILE_S_ADDMULT = 2;  // == Semi

// ---- small dense per-sample strata (k_tile.cu) ----
// A stratum whose relations have small per-sample domains runs to fixpoint in
// ONE launch: one CTA per sample (grid-stride), the stratum's relations dense
// in shared memory (compact slot = row-major over the true column domains),
// every round pull-evaluated per head slot.  Non-head variables are enumerated
// in the oracle's canonical order (rule, non-head variables by first
// appearance, variant), each level's values taken from 64-bit presence fibers
// of the atoms its variable closes, so add-mult sums are formed in exactly the
// oracle's fp64 order.
constexpr int TILE_MAXREL = 6, TILE_MAXRULE = 8, TILE_MAXLEV = 5, TILE_MAXVAR = 4, TILE_MAXCOL = 4, TILE_MAXV = 10;
constexpr int TILE_THREADS_N = 512;
constexpr int TILE_CM_PARTS = 4096;  // partial sums of split composition items (compose_rounds)
enum TileVer : int8_t { TV_EXT = 0, TV_NEW = 1, TV_OLD = 2, TV_DELTA = 3 };
struct TileRel {
  int8_t ncols;
  int8_t local;                 // 1: a relation of the stratum (shared memory), 0: external (global)
  int8_t shared;                // external shared relation: one copy for all samples
  int32_t dom[TILE_MAXCOL];
  int32_t stride[TILE_MAXCOL];  // compact slot = Σ coord_c · stride_c
  int32_t D;                    // slots per sample
  int32_t fstride[TILE_MAXCOL][TILE_MAXCOL];  // fiber along c: id = Σ_{c' != c} coord_c' · fstride[c][c']
  int32_t nfib[TILE_MAXCOL];    // fibers along column c (D / dom[c]); 0 = not needed
  // external: global dense arrays per sample
  const float* tag;                       // [samples][D] (null under unit)
  const uint32_t* bits;                   // [samples][ceil(D/32)] presence
  const unsigned long long* fib[TILE_MAXCOL];  // [samples][nfib[c]] presence words along column c
  // local: shared-memory byte offsets (S, Δ, U)
  int32_t sm_tag[3];
  int32_t sm_bits[3];
  int32_t sm_fib[2][TILE_MAXCOL];  // S, Δ fibers along column c (-1 unused)
  // local: the final relation goes to the dense store of the packed layout
  float* dfp;                   // slot tags (DENSE_ABSENT prefilled), non-unit
  uint32_t* dfbits;             // unit: presence bitmap (zero prefilled)
  uint8_t pshift[TILE_MAXCOL];
  uint8_t psshift;
};
struct TileAtom {
  int8_t rel;                   // index into TilePlan::rel
  int8_t var[TILE_MAXCOL];      // variable id, or -1: constant coordinate cst
  int32_t cst[TILE_MAXCOL];
  int8_t level;                 // level whose variable closes the atom; -1: bound by the head
  int8_t fcol;                  // column of that variable (fiber column)
  int8_t chk;                   // level binding its other variables (< level; -1: the head): from then on its
                                // fiber must be non-empty, so a value whose fiber is empty prunes the subtree
};
struct TileCmp {
  int8_t va, vb;                // variable ids, -1: constant value
  int32_t ca, cb;               // constant values (value space)
  int8_t neq;                   // relation: 0 ==, 1 !=, 2 <, 3 <=, 4 >, 5 >=
  int8_t level;                 // -1: head variables / constants only
};
struct TileRule {
  int8_t head;                  // TilePlan::rel index
  int8_t hvar[TILE_MAXCOL];     // head args: variable id or -1 (constant coordinate hcst)
  int32_t hcst[TILE_MAXCOL];
  int8_t natoms;
  TileAtom atom[TILE_MAXT];
  int8_t nlev;
  int8_t lev_var[TILE_MAXLEV];  // non-head variables, canonical order (first appearance)
  int32_t vdom[TILE_MAXV];      // variable domain sizes
  int32_t vmin[TILE_MAXV];      // class minimum (comparisons are made on values)
  int8_t nvariant;              // 1 for a seed rule
  int8_t ver[TILE_MAXVAR][TILE_MAXT];
  int8_t seed;                  // all-external rule: round 1 only
  int8_t shape;                 // 1: composition H(a,x,z) :- K(b,x,y), K(c,y,z), T(b,c,a) (K local = H, T external)
  int8_t ncmp;
  TileCmp cmp[TILE_MAXC];
};
struct TilePlan {
  int semi;
  int nsamples;
  int max_iters;
  int nrel, nrule, nlocal;
  int8_t local_rel[TILE_MAXREL];  // TilePlan::rel indexes of the stratum's relations
  TileRel rel[TILE_MAXREL];
  TileRule rule[TILE_MAXRULE];
  int32_t smem_bytes;
  int32_t clear_words;           // leading u32 words of shared memory zeroed per sample (bits + fibers)
  // Compacted composition rounds (tile_device.cuh compose_rounds): the
  // stratum is one local relation whose only recursive rule is the
  // composition shape.  Rounds >= 2 evaluate only the head slots (a, x, z)
  // whose (x, z) pair can receive a candidate this round, a fastest across
  // lanes.  cm_rule: that rule's index, -1 off; cm_off: shared-memory bytes of
  // the per-x / per-z masks (5 × 64 u64), counters, per-pair cost class
  // and rank (u32) and the pair list (u16, heaviest cost class first).
  int32_t cm_rule;
  int32_t cm_off;
  int32_t cm_nocert;              // A/B + test: every split add-mult head takes the sequential fallback
  int32_t cm_nosplit;             // A/B: no split items (every head item walked by one thread)
  uint32_t* trace;               // debug (LOBSTER_TILE_TRACE): per (sample, round < 64) candidates, |Δ'|
  unsigned long long* counts;    // per local relation (local_rel order): tuples at the fixpoint
};

}  // namespace lob
