// kernels.cuh — device plan structures and launchers of the sm_100a kernels.
//
// Every relation row is a packed u64 key (SURVEY §8(a) layout):
//   key = sample << Σbits | (c0 - min0) << ... | (c_{n-1} - min_{n-1})
// order-preserving for the lexicographic (sample, c0, ...) order, plus
// SoA tag columns: p (fp32 bits) and, under diff-max-mult, w (u32 witness).
// Keys use at most 63 bits; KEY_DEAD (all ones) marks a row removed by a filter.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tile_plan.h"

namespace lob {

constexpr uint64_t KEY_DEAD = ~0ull;
constexpr int MAXM = 10;   // max bit moves per output word
constexpr int MAXT = 6;    // max atoms per rule (tags carried by an intermediate)
constexpr int MAXC = 4;    // max comparisons applied in one join step

enum Semi : int { S_UNIT = 0, S_MAXMIN = 1, S_ADDMULT = 2, S_MAXMULT = 3 };

// max-mult direct-store word: (pbits + 1) << 34 | stamp << WB | ~wc (WB bits).
// wc is the witness in compressed layout (rule index << T | variables, T = the
// widest variable field of the relation's rules; order-preserving), WB = rule
// bits + T.  stamp = SMAX - round (SB = 34 - WB bits): on equal p an older
// round's value wins (reading 8a) without rewriting slots; when SB cannot hold
// every round, candidates take stamp 0 and Δ' extraction re-stamps SMAX
// (a "settled" bit).  MxEnc: the per-launch constants.
struct MxEnc {
  unsigned long long stamp;  // stamp << WB for this round's candidates
  unsigned long long wmask;  // (1 << WB) - 1
};

// counts every kernel launch of this library (lobster_kernel_launches)
void note_launch();

// Copy `bits` bits found at `sshift` of the source word (0 = probe key,
// 1 = build key) to `dshift` of the destination word.  A variable keeps its
// domain class (same min and width) in every relation it flows through, so a
// projection / permutation is a pure bit move (no decode / re-encode).
struct Move {
  uint8_t src, sshift, bits, dshift;
};

// One side of a comparison: a decoded value (field + min) or a constant.
struct Operand {
  int8_t src;      // 0 probe key, 1 build key, 2 constant
  uint8_t shift, bits;
  int32_t base;    // min of the field, or the constant value
};
struct Cmp {
  Operand a, b;
  int8_t neq;      // relation: 0 ==, 1 !=, 2 <, 3 <=, 4 >, 5 >= (program.hpp RelOp)
};

// Arithmetic (§5.2 eval): "compiled to bytecode for a simple stack
// machine, and each GPU thread executes this bytecode program against one
// fact with a small fixed-size stack".  Postfix programs over the probe key's
// fields; int32 two's complement, / and % truncate; a division by zero (or
// INT32_MIN / -1) fails the row.
enum BcOp : int8_t { BC_FIELD = 0, BC_CONST = 1, BC_ADD, BC_SUB, BC_MUL, BC_DIV, BC_MOD, BC_NEG };
constexpr int MAXBC = 16, MAXBH = 4, MAXBF = 2;
struct BcIns {
  int8_t op;
  uint8_t shift, bits;  // BC_FIELD: value = (key >> shift & mask(bits)) + v
  int32_t v;
};
struct Bc {
  int n;
  BcIns ins[MAXBC];
};
struct BcHead {        // computed head column: (value - base) << dshift, dead if outside [0, 2^bits)
  Bc e;
  uint8_t dshift, bits;
  int32_t base;
};
struct BcFilter {
  Bc lhs, rhs;
  int8_t rel;
};

// A join step: probe rows (sorted packed keys) x a sorted build index whose key
// is [prefix | free fields]; prefix built from the probe key by moves.
struct JoinPlan {
  // probe
  const void* pkey;         // u32 or u64 keys (pk32)
  int8_t pk32, ok32;
  int64_t np;
  const uint32_t* np_dev;   // nullable: probe rows = min(np, *np_dev) (Δ size left on the device)
  const float* ptag[MAXT];
  int npt;
  // build lookup
  int nprem;
  Move prem[MAXM];
  uint64_t cprefix;         // constant bits of the prefix
  const uint64_t* bkey;
  const float* btag;        // nullable (unit)
  int64_t nb;
  const int64_t* boff;      // CSR offsets over the prefix domain, or null (binary search)
  int64_t nprefix;          // entries of boff minus one
  const uint4* brec;        // nullable: per prefix one 32-B record {u32 key[4] (~0 = none), f32 tag[4]}
  int free_bits;            // bits below the prefix in the index key
  // repeated free variables: value at shift a must equal value at shift b (build key)
  int nfeq;
  Move feq[2];
  // filters
  int ncmp;
  Cmp cmp[MAXC];
  // output key
  int nom;
  Move om[MAXM];
  uint64_t cout;            // constant bits of the output key
  int final_step;           // 1: candidates (head key, ⊗, witness); 0: intermediate
  int semi;
  int omin;                 // diff-max-min-prob: max-mult storage and witnesses, ⊗ = min
  int prefetch;             // fused join: L2 prefetch of the next grid-stride row (LOBSTER_FJ_PREFETCH=0: off)
  // ⊗ in body order over T = [ptag[0..npt-1], btag]: T[tag_order[k]] for k = 0..ntag-1
  int ntag;
  int8_t tag_order[MAXT];
  // witness: w = wconst | moves (diff-max-mult)
  int nwm;
  Move wm[MAXM];
  uint32_t wconst;
  // outputs
  void* okey;               // u32 or u64 keys (ok32)
  float* otag[MAXT];        // intermediate: npt + 1 tag columns
  uint32_t* oval32;         // final, max-min / add-mult: p bits
  uint64_t* oval64;         // final, max-mult: p bits | w << 32
  // direct ⊕ into a dense store (final step, idempotent semirings; see Direct)
  int direct;
  void* fdir;               // u32 bitmap (unit) / u32 packed (max-min) / u64 packed (max-mult)
  uint32_t* dirty;          // bitmap: slots improved this round
  int aggregate;            // warp pre-reduction of equal slots (narrow heads)
  MxEnc mx;                 // max-mult word constants

};

// Direct ⊕ (idempotent semirings on a direct-mapped store): F[slot] holds
//   unit    : one bit per slot
//   max-min : pbits + 1                       (0 = absent)
//   max-mult: (pbits + 1) << 34 | stamp << WB | ~wc   (MxEnc)
// so one atomicMax per candidate computes "larger p wins; on equal p the
// older round's tag wins, then the smaller witness" (readings 8a, 8b);
// max-min has no witness, so an equal p is simply no change.  A candidate is
// applied only if it beats a plain (stale) read of the slot, which is a lower
// bound of the slot at round start; such a candidate makes the slot end the
// round above its round-start value, so it sets the slot's bit in the round's
// dirty bitmap (idempotent OR, fire-and-forget).  The epilogue compacts the
// bitmap in slot order into Δ' (sorted, deterministic) and, under max-mult
// without round stamps, re-stamps those slots.

// Single-atom rule (projection): rows of one relation -> candidates.
struct ProjectPlan {
  const void* key;          // u32 or u64 keys (pk32)
  int8_t pk32, ok32;
  const float* tag;
  int64_t n;
  int ncmp;
  Cmp cmp[MAXC];  // operands read from src 0
  int nom;
  Move om[MAXM];
  uint64_t cout;
  int semi;
  uint32_t wconst;
  int nwm;
  Move wm[MAXM];
  void* okey;
  uint32_t* oval32;
  uint64_t* oval64;
  int direct;
  void* fdir;
  uint32_t* dirty;
  int aggregate;
  MxEnc mx;
  // arithmetic: computed head columns and expression filters (bytecode)
  int nbh, nbf;
  BcHead bh[MAXBH];
  BcFilter bf[MAXBF];
};

// Lookup chain: probe rows whose variables cover the whole rule; every other
// body atom is fully bound, i.e. a point lookup (<= 1 row, EDB deduplicated).
// One thread per probe row; no intermediate, no count / scan.
constexpr int MAXL = 4;
struct Lookup {
  int nprem;
  Move prem[MAXM];
  uint64_t cprefix;
  const uint64_t* bkey;
  const float* btag;
  int64_t nb;
  const int64_t* boff;  // CSR over the (full-key) prefix, or null (binary search)
  int64_t nprefix;
};
struct LookupPlan {
  const void* pkey;
  int8_t pk32, ok32;
  int64_t np;
  const float* ptag;
  const void* pdir;   // nullable: probe = the present slots of a direct store (np = slots; key = slot)
  int nlk;
  Lookup lk[MAXL];
  int ncmp;
  Cmp cmp[MAXC];  // operands read from the probe key (src 0)
  int nom;
  Move om[MAXM];
  uint64_t cout;
  int semi;
  int omin;           // diff-max-min-prob: ⊗ = min (storage as max-mult)
  // ⊗ in body order over T = [probe tag, lookup tags...]
  int ntag;
  int8_t tag_order[MAXT];
  int nwm;
  Move wm[MAXM];
  uint32_t wconst;
  // outputs: candidates (dead key for a miss / filtered row) or direct ⊕
  void* okey;
  uint32_t* oval32;
  uint64_t* oval64;
  int direct;
  void* fdir;
  uint32_t* dirty;
  int aggregate;
  MxEnc mx;
};
void launch_lookup_chain(const LookupPlan& lp, unsigned long long* ncand, cudaStream_t st);

// ---- scan ----
// Exclusive prefix sum; writes the total to *total_dev (device).  T in
// {uint32_t, int64_t, uint64_t}.  tmp: scratch of scan_tmp_bytes(n) bytes.
template <typename T>
size_t scan_tmp_bytes(int64_t n);
template <typename T>
void exclusive_scan(const T* in, T* out, int64_t n, T* total_dev, void* tmp, cudaStream_t st);

// ---- radix sort (LSD, 8-bit digits, stable) ----
// V in {void (keys only), uint32_t, uint64_t}.  Sorts the low `bits` bits.
// Ping-pong between (k0,v0) and (k1,v1); returns 0 if the result is in k0/v0.
size_t sort_tmp_bytes(int64_t n);
template <typename K, typename V>
int radix_sort(K* k0, V* v0, K* k1, V* v1, int64_t n, int bits, void* tmp, cudaStream_t st);

// ---- ingest (A0) ----
void launch_minmax(const int32_t* col, int64_t n, int32_t* out2 /* device: min,max */, cudaStream_t st);
// key = sample << sshift | Σ (col_c - min_c) << shift_c
struct PackPlan {
  int ncols;
  const int32_t* col[8];
  int32_t min[8];
  uint8_t shift[8];
  const int32_t* sample;  // null for shared
  uint8_t sshift;
  int32_t s_lo, s_hi;     // micro-batch: samples outside [s_lo, s_hi) -> dead key; sample - s_lo packed
};
void launch_pack(const PackPlan& pp, int64_t n, uint64_t* key, uint32_t* rowid, cudaStream_t st);
// gather p / fid by rowid
void launch_gather_f32(const float* src, const uint32_t* idx, float* dst, int64_t n, cudaStream_t st);
void launch_gather_i32(const int32_t* src, const uint32_t* idx, int32_t* dst, int64_t n, cudaStream_t st);
void launch_iota_i32(int32_t* dst, int64_t n, int32_t first, cudaStream_t st);
void launch_fill_f32(float* dst, int64_t n, float v, cudaStream_t st);
// range check of pushed data: flags bit0 = prob NaN/out of [0,1], bit1 = sample out of range
void launch_validate(const float* p, const int32_t* s, int64_t n, int32_t batch, uint32_t* flags, cudaStream_t st);

// EDB duplicate merge (reading 16): sorted keys; heads -> scan -> reduce.
void launch_heads(const uint64_t* key, int64_t n, uint32_t* flag, cudaStream_t st);
void launch_heads(const uint32_t* key, int64_t n, uint32_t* flag, cudaStream_t st);
void launch_edb_reduce(const uint64_t* key, const float* p, const int32_t* fid, const uint32_t* pos, int64_t n,
                       int semi, uint64_t* okey, float* op, int32_t* ofid, cudaStream_t st);

// ---- join (A3-A5) ----
void launch_join_count(const JoinPlan& jp, int64_t* count, int64_t* start, cudaStream_t st);
// tile_row: join_write_tiles(total) + 1 int64 scratch
int64_t join_write_tiles(int64_t total);
void launch_join_write(const JoinPlan& jp, const int64_t* offs, const int64_t* start, int64_t total,
                       int64_t* tile_row, cudaStream_t st);
void launch_project(const ProjectPlan& pp, cudaStream_t st);
// fused row-centric join + direct ⊕ (bounded fan-out <= 8 per prefix); adds |C| to *ncand
// With jp.np_dev (Δ size on the device) the grid is persistent.
void launch_join_rows_direct(const JoinPlan& jp, int maxdeg, unsigned long long* ncand, cudaStream_t st,
                             int64_t np_hint);
// fan-out <= 4 and index keys < 2^31: per-prefix 32-B records (one sector: keys, tags)
void launch_build_rec4(const int64_t* off, const uint64_t* key, const float* tag, int64_t nprefix, uint4* rec,
                       cudaStream_t st);
// max_p (off[p+1] - off[p]) -> atomicMax into *out
void launch_max_degree(const int64_t* off, int64_t nprefix, unsigned long long* out, cudaStream_t st);


// ---- index build (A1) ----
// re-key rows: out = Σ moves(key) ; tags copied
void launch_rekey(const uint64_t* key, int64_t n, const Move* mv, int nmv, uint64_t* out, cudaStream_t st);
void launch_build_offsets(const uint64_t* key, int64_t n, int free_bits, int64_t nprefix, int64_t* off,
                          cudaStream_t st);

// ---- dedup (A6-A7) and merge/diff (A8-A9) ----
// U = segmented ⊕ over sorted candidates (vals: u32 p bits or u64 p|w<<32)
// scratch: 2*nu + 2 uint32 words
void launch_seg_reduce(const uint64_t* key, const void* val, const uint32_t* pos, int64_t n, int64_t nu, int semi,
                       uint64_t* ukey, float* up, uint32_t* uw, uint32_t* scratch, cudaStream_t st);
void launch_seg_reduce(const uint32_t* key, const void* val, const uint32_t* pos, int64_t n, int64_t nu, int semi,
                       uint32_t* ukey, float* up, uint32_t* uw, uint32_t* scratch, cudaStream_t st);

// ---- dense direct-mapped store: F[slot = packed key] ----
// p = DENSE_ABSENT marks an absent tuple; under UNIT a presence bitmap.
constexpr uint32_t DENSE_ABSENT = 0xffffffffu;
void launch_dense_fill(float* fp, uint32_t* fbits, int64_t nslots, int semi, cudaStream_t st);
// classify + apply U (unique u32 keys) in place: flags lo = in Δ', hi = new tuple
void launch_dense_diff(const uint32_t* ukey, const float* up, const uint32_t* uw, int64_t nu, int semi, float* fp,
                       uint32_t* fw, uint32_t* fbits, uint64_t* flags, cudaStream_t st);
void launch_dense_delta(const uint32_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* flags,
                        const uint64_t* offs, int semi, uint32_t* dkey, float* dp, uint32_t* dw, cudaStream_t st);
// dense -> sorted list (end of stratum): flag present slots, scan, compact
void launch_dense_present(const float* fp, const uint32_t* fbits, int64_t nslots, int semi, uint32_t* flag,
                          cudaStream_t st);
void launch_dense_compact(const float* fp, const uint32_t* fw, const uint32_t* fbits, const uint32_t* pos,
                          int64_t nslots, int semi, uint64_t* key, float* p, uint32_t* w, cudaStream_t st);
// direct ⊕ store: zero-fill, present flags, compaction
void launch_direct_fill(void* f, int64_t nslots, int semi, cudaStream_t st);
// two launches (tile / group counts, then bases + rows): dirty bitmap -> Δ' in slot order,
// dirty bits cleared, max-mult slots re-settled; |Δ'| -> *total (device).  scratch: direct_extract2_scratch u32
int64_t direct_extract2_scratch(int64_t nwords);
// restamp (max-mult): OR-ed into every Δ' slot word (0 = none).  ring (nullable,
// host-mapped): also receives seq << 32 | |Δ'| (system-scope store).  ctr (nullable,
// 2 zeroed u32 that the kernel leaves zeroed): one launch, Δ' in slot-sorted runs
// claimed by atomics instead of fully slot-ordered (scratch unused)
void launch_direct_extract2(void* f, uint32_t* dirty, int64_t nwords, int semi, uint32_t* dkey, float* dp,
                            uint32_t* dw, uint32_t* scratch, uint32_t* total, unsigned long long restamp,
                            unsigned long long wmask, unsigned long long* ring, uint32_t seq, uint32_t* ctr,
                            cudaStream_t st);
void launch_direct_present(const void* f, int64_t nslots, int semi, uint32_t* flag, cudaStream_t st);
// number of present slots -> atomicAdd into *out
void launch_direct_count(const void* f, int64_t nslots, int semi, unsigned long long* out, cudaStream_t st);
// wT / wrb: witness decompression (variable field width, rule-index bits)
void launch_direct_compact(const void* f, const uint32_t* pos, int64_t nslots, int semi, uint64_t* key, float* p,
                           uint32_t* w, unsigned long long wmask, int wT, int wrb, cudaStream_t st);
// classify U against F: flags (u64: lo = in Δ', hi = new); pos (F index or -1)
void launch_diff(const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu,
                 const uint64_t* fkey, const float* fp, int64_t nf, int semi, uint64_t* flags, int64_t* pos,
                 cudaStream_t st);
// write Δ' and NEW rows, apply in-place ⊕ updates to F
void launch_apply(const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* flags,
                  const uint64_t* offs, const int64_t* pos, int semi, float* fp, uint32_t* fw, uint64_t* dkey,
                  float* dp, uint32_t* dw, uint64_t* nkey, float* np_, uint32_t* nw, cudaStream_t st);
// F' = merge(F, NEW) (disjoint sorted key sets)
void launch_merge(const uint64_t* akey, const float* ap, const uint32_t* aw, int64_t na, const uint64_t* bkey,
                  const float* bp, const uint32_t* bw, int64_t nb, uint64_t* okey, float* op, uint32_t* ow,
                  cudaStream_t st);

// ---- witness walk + gradient (A11) ----
struct WalkRel {
  const uint64_t* key;
  const float* p;
  const uint32_t* w;       // IDB witness
  const int32_t* fid;      // EDB fact id
  const unsigned long long* dir;  // nullable: the relation's direct max-mult store (O(1) hop, MxEnc words)
  unsigned long long wmask;
  int wT, wrb;
  const int64_t* off;  // nullable: CSR over key >> pshift (an aliasing static index): O(1) + short scan
  int64_t nprefix;
  int pshift;
  int64_t n;
  int input;
  int has_sample;
  uint8_t sshift;
  int ncols;
  uint8_t shift[8], bits[8];
  int32_t min[8];
};
struct WalkAtom {
  int rel;
  int ncols;
  int8_t var[8];   // var id or -1 for a constant
  int32_t cst[8];
};
struct WalkRule {
  int natoms;
  WalkAtom atom[MAXT];
  int nvars;
  // var values: from the head tuple column, or from the witness field
  int8_t head_col[16];        // var -> head column or -1
  int8_t wfield[16];          // var -> witness field index or -1
  uint8_t wshift[16], wbits[16];
  int32_t wmin[16];
};
struct WalkTables {
  WalkRel* rels;        // device arrays
  WalkRule* rules;      // indexed by rule_base[head_rel] + local rule index
  int* rule_base;
  int* rule_bits;       // per relation: witness bits taken by the rule index
  int nrels;
};
// pass 0: count leaves per tuple; pass 1: write leaf fact ids at offs.
// gkey/grel (nullable): spill region of gcap entries per thread for stacks
// deeper than the in-register part; with it the launch is gthreads threads,
// grid-stride.  err bit 2 = a stack overflowed (cnt of that tuple is 0).
void launch_walk(const WalkTables& T, int rel, int64_t n, int pass, const int64_t* offs, int64_t* cnt,
                 int64_t* leaves, int* err, uint64_t* gkey, int* grel, int64_t gcap, int64_t gthreads,
                 cudaStream_t st);
// grads from sorted (tuple, fact) leaves: unique facts with multiplicity
void launch_leaf_heads(const uint64_t* k, int64_t n, uint32_t* flag, cudaStream_t st);
void launch_grad(const uint64_t* sorted_tf, const uint32_t* pos, int64_t nleaf, int64_t nuniq, const float* fact_p,
                 int64_t ntup, const int64_t* loff, int64_t* goff, int64_t* gfid, float* gval, double* scratch,
                 cudaStream_t st);

// ---- diff-top-1-proofs (k_top1.cu) ----
struct ProofRel {
  const uint64_t* key;   // sorted keys of the relation's stored tuples (input rows / proof index)
  int64_t n;
  const int32_t* fid;    // input relation: fact id per row (proof = {fid}); else null
  const uint64_t* pof;   // IDB: proof offset into pool, per key
  const uint32_t* pln;   //      proof length
  const uint32_t* pool;
  int has_sample;
  uint8_t sshift;
  uint8_t shift[8], bits[8];
  int32_t min[8];
};
struct ProofTables {
  ProofRel* rels;
  WalkRule* rules;
  int* rule_base;
  int* rule_bits;
  const float* fact_p;
  const int32_t* group;  // nullable: exclusion group per fact (-1 none)
  int cap;               // proof size limit (300)
};
void launch_top1_cand(const ProofTables& T, int hrel, uint64_t* key, uint64_t* val, int64_t n, int* err,
                      cudaStream_t st);
void launch_top1_delta(const ProofTables& T, int hrel, const uint64_t* key, const uint32_t* w, int64_t n,
                       uint32_t* len, const uint64_t* offs, uint32_t* pool, int* err, cudaStream_t st);
void launch_top1_update(const uint64_t* pkey, int64_t np, uint64_t* pof, uint32_t* pln, const uint64_t* dkey,
                        const uint64_t* dof, const uint32_t* dln, int64_t nd, uint32_t* isnew, cudaStream_t st);
void launch_top1_compact(const uint64_t* dkey, const uint64_t* dof, const uint32_t* dln, const uint32_t* isnew,
                         const uint32_t* pos, int64_t nd, uint64_t* nkey, uint64_t* nof, uint32_t* nln,
                         cudaStream_t st);
void launch_top1_merge(const uint64_t* akey, const uint64_t* aof, const uint32_t* aln, int64_t na,
                       const uint64_t* bkey, const uint64_t* bof, const uint32_t* bln, int64_t nb, uint64_t* okey,
                       uint64_t* oof, uint32_t* oln, cudaStream_t st);
void launch_top1_gather(const uint32_t* pool, const uint64_t* pof, const uint32_t* pln, const uint64_t* noff,
                        int64_t n, uint32_t* npool, cudaStream_t st);
void launch_top1_grad(const uint32_t* pool, const uint64_t* pof, const uint32_t* pln, const uint64_t* noff, int64_t n,
                      const float* fact_p, int64_t* goff, int64_t* gfid, float* gval, double* scratch,
                      cudaStream_t st);

// diff-add-mult: CSR offsets of output rows into the adjoint program's __grad rows
void launch_grad_rows(const int32_t* osid, const int32_t* ocols, int64_t n, int k, const int32_t* gsid,
                      const int32_t* gcols, int64_t ng, int64_t* goff, cudaStream_t st);
void launch_widen_i32(const int32_t* in, int64_t n, int64_t* out, cudaStream_t st);

// diff-max-min: one-hot gradient on each tuple's minimum leaf (goff[t] = t)
void launch_grad_onehot(const uint64_t* sorted_tf, int64_t nleaf, const float* fact_p, int64_t ntup,
                        const int64_t* loff, int64_t* goff, int64_t* gfid, float* gval, cudaStream_t st);

// ---- bit-sliced multi-source frontier (k_slice.cu; unit, C4-shaped strata) ----
// CSR of a shared binary relation by column ssrc (counting sort): off[T+1], nbr[n]
void launch_slice_csr(const uint64_t* key, int64_t n, int ssrc, int sdst, int bits, int64_t T, uint32_t* off,
                      uint32_t* cursor, uint32_t* nbr, void* scan_tmp, cudaStream_t st);
void launch_slice_from_bitmap(const uint32_t* bm, int tbits, int B, int64_t T, int W, uint32_t* Nb, uint32_t* dirty,
                              cudaStream_t st);
void launch_slice_to_bitmap(const uint32_t* Rb, int tbits, int B, int64_t T, int W, uint32_t* bm, cudaStream_t st);
void launch_slice_extract(uint32_t* dirty, int64_t ndw, uint32_t* Nb, uint32_t* Rb, int W, uint32_t* dt, uint32_t* dwi,
                          uint32_t* dbits, uint32_t* count, unsigned long long* tuples, cudaStream_t st);
void launch_add_u32_dev(uint32_t* dst, const uint32_t* src, bool assign, cudaStream_t st);  // *dst (+)= *src
void launch_slice_deg(const uint32_t* dt, int64_t nd, const uint32_t* off, uint32_t* deg, cudaStream_t st);
void launch_slice_expand(const uint32_t* dt, const uint32_t* dwi, const uint32_t* dbits, const uint32_t* pos,
                         int64_t nd, const uint32_t* total_dev, const uint32_t* off, const uint32_t* nbr,
                         const uint32_t* Rb, uint32_t* Nb, int W, uint32_t* dirty, unsigned long long* cands,
                         cudaStream_t st);

// ---- small dense per-sample strata (k_tile.cu; plan structs in tile_plan.h) ----
static_assert(TILE_MAXT == MAXT && TILE_MAXC == MAXC, "tile_plan.h limits");
// rounds_out[s]: rounds of sample s (the last one empty); cap_hit: max_iters reached
// dplan: device scratch for the plan (sizeof(TilePlan), 16-B aligned)
void launch_tile_fixpoint(const TilePlan& P, TilePlan* dplan, int* rounds_out, unsigned long long* ncand,
                          int* cap_hit, cudaStream_t st);
// external relation -> dense per-sample arrays (tags, presence bits, fibers); arrays prezeroed
struct TileScatter {
  const uint64_t* key;
  const float* p;
  int64_t n;
  int has_sample;
  uint8_t sshift, sbits;
  int ncols;
  uint8_t shift[TILE_MAXCOL], bits[TILE_MAXCOL];
  TileRel rel;
};
void launch_tile_scatter(const TileScatter& S, cudaStream_t st);
// max over n ints -> *out (device)
void launch_max_i32(const int* a, int n, int* out, cudaStream_t st);

// ---- key-partitioned evaluation (k_part.cu) ----
// dest[i] = owner rank of key i (world for dead keys), idx[i] = i, cnt[dest]++ (world + 1 counters)
void launch_part_dest(const void* key, bool k32, int64_t n, uint32_t world, uint32_t* dest, uint32_t* idx,
                      unsigned long long* cnt, cudaStream_t st);
// keys not owned by `rank` -> dead (seed rounds: every rank derives every seed candidate)
void launch_part_keep(void* key, bool k32, int64_t n, uint32_t world, uint32_t rank, cudaStream_t st);
void launch_part_gather(const void* src, const uint32_t* idx, void* dst, int64_t n, int elem_bytes, cudaStream_t st);

// u32 keys -> u64 (sorted-store candidates narrowed for the sort)
void launch_widen_u32(const uint32_t* in, int64_t n, uint64_t* out, cudaStream_t st);

// ---- output extract (A12) ----
void launch_unpack(const uint64_t* key, int64_t n, int has_sample, uint8_t sshift, int ncols, const uint8_t* shift,
                   const uint8_t* bits, const int32_t* mins, int32_t* sample, int32_t* cols, cudaStream_t st);
// micro-batch output collection helpers
void launch_add_i32(int32_t* a, int64_t n, int32_t v, cudaStream_t st);
void launch_add_i64(const int64_t* s, int64_t n, int64_t v, int64_t* d, cudaStream_t st);
void launch_sample_offsets_i32(const int32_t* sid, int64_t n, int32_t batch, int64_t* off, cudaStream_t st);
void launch_sample_offsets(const uint64_t* key, int64_t n, int32_t batch, uint8_t sshift, int has_sample,
                           int64_t* off, cudaStream_t st);

// ---- backward (optional) ----
void launch_grad_contrib(const int64_t* goff, const int64_t* gfid, const float* gval, const float* upstream,
                         int64_t n, int64_t ng, uint64_t* key, uint32_t* val, cudaStream_t st);
void launch_dense_sum(const uint64_t* key, const uint32_t* val, const uint32_t* pos, int64_t n, float* dense,
                      cudaStream_t st);

}  // namespace lob
