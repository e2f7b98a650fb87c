/*
 * lobster.h — C ABI of the B200-native semi-naive fixpoint engine.
 *
 * The engine evaluates a stratified Datalog program over semiring-tagged
 * relations by semi-naive fixpoint iteration on one CUDA device (sm_100a).
 * The four calls follow the paper's statement of the problem:
 *   - a stratified program of rules          PAPER.md:383-410 (§3.1, Fig. 6)
 *   - an input database of tagged facts      PAPER.md:285-287 (§2), 413-422
 *   - batched samples (sample-id register)   PAPER.md:681-691 (§4.3)
 *   - fixpoint evaluation                    PAPER.md:599-611 (§3.4), 1366-1392 (Alg. 1)
 *   - outputs read back per sample with tags and gradients
 *                                            PAPER.md:685 (§4.3), 292 (§2)
 * Readings of silent / ambiguous passages: SURVEY.md §8(c), restated in
 * DESIGN.md ("Readings").
 *
 * Conventions
 *   - Every call returns lobster_status; no C++ exception crosses the ABI.
 *   - All device work is ordered on lobster_options.cuda_stream (NULL = the
 *     legacy default stream).  Calls are blocking with respect to the host
 *     unless stated otherwise.
 *   - One context per host thread; a context is not shareable.
 *   - Call order: program_load -> facts_push* -> run -> output_get*.  The
 *     first facts_push after a completed run starts a new database: every
 *     relation's facts, every output and the fact-id counter are reset.
 *   - There is no CPU fallback: if the CUDA device is unavailable every call
 *     that needs it fails with LOBSTER_E_CUDA.
 */
#ifndef LOBSTER_H
#define LOBSTER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lobster_ctx lobster_ctx; /* opaque; owns all device and output memory */

typedef enum {
  LOBSTER_OK = 0,
  LOBSTER_E_INVALID_ARG = 1, /* NULL pointer, bad enum, unknown relation name in output_get */
  LOBSTER_E_PARSE = 2,       /* program text error; message "line:col: msg"          */
  LOBSTER_E_SCHEMA = 3,      /* unknown input relation / arity mismatch / batched w/o samples */
  LOBSTER_E_RANGE = 4,       /* prob NaN or outside [0,1]; sample id out of range; key or
                                witness wider than 64 / 32 bits                               */
  LOBSTER_E_STATE = 5,       /* call out of order (push before load, get before run, ...)    */
  LOBSTER_E_OOM = 6,         /* device allocation failed                                      */
  LOBSTER_E_ITER_CAP = 7,    /* max_iters rounds reached in a stratum (state readable)        */
  LOBSTER_E_CUDA = 8,        /* CUDA error; sticky: the context must be destroyed             */
  LOBSTER_E_NCCL = 9         /* NCCL missing or a collective failed (lobster_group_nccl, key-
                                partitioned runs)                                             */
} lobster_status;

/* Provenance semirings (PAPER.md:445-456 Fig. 7b; :616-617 §3.5).
 *   UNIT               : Bool {⊥,⊤}, ∨, ∧.  No tag is stored.
 *   MAX_MIN_PROB       : [0,1], 0, 1, max, min                         (Fig. 7b)
 *   ADD_MULT_PROB      : [0,∞) unclamped, 0, 1, +, ×; ⊕ within a round accumulates
 *                        in fp64 and rounds once to fp32                 (reading 6, 9)
 *   DIFF_MAX_MULT_PROB : [0,1] × witness, 0, 1, max (strict improvement; ties keep
 *                        the existing tag, same-round ties pick the smallest
 *                        (rule, non-head variables)), fp32 ×.  Gradients flow to
 *                        the input facts of the winning derivation      (reading 7, 8)
 *   DIFF_MAX_MIN_PROB  : [0,1] × witness, 0, 1, max (tie rules as DIFF_MAX_MULT_PROB),
 *                        min.  Tags equal MAX_MIN_PROB's; the gradient is one-hot on
 *                        the winning derivation's minimum leaf (smallest fact id on
 *                        ties): "the differentiable versions of the probabilistic
 *                        semirings", PAPER.md:617 (§3.5)
 *   DIFF_TOP1_PROOFS   : one proof per tuple — a set of at most 300 input facts
 *                         — with p = Π over the set (fp64, ascending fact
 *                        ids, rounded once); ⊗ = union, dropped when two facts of
 *                        one exclusion group meet (lobster_facts_groups); ⊕ = the
 *                        more likely proof, tie rules as DIFF_MAX_MULT_PROB;
 *                        gradient ∂p/∂p_f = Π of the proof's other facts
 *                        (§2, 617-628 §3.5).  GPU: rules may read
 *                        their own stratum at most once (linear recursion)
 *   DIFF_ADD_MULT_PROB : dual numbers (p, ∂p/∂p_f): p exactly as
 *                        ADD_MULT_PROB; gradients of every `output` relation are
 *                        the derivative of the add-mult result (finite
 *                        derivations, e.g. DAG inputs), computed in reverse mode
 *                        by a generated adjoint program over the final relations
 *                        (reading "diff-add-mult")                  */
typedef enum {
  LOBSTER_UNIT = 0,
  LOBSTER_MAX_MIN_PROB = 1,
  LOBSTER_ADD_MULT_PROB = 2,
  LOBSTER_DIFF_MAX_MULT_PROB = 3,
  LOBSTER_DIFF_MAX_MIN_PROB = 4,
  LOBSTER_DIFF_TOP1_PROOFS = 5,
  LOBSTER_DIFF_ADD_MULT_PROB = 6
} lobster_semiring;

typedef struct {
  int32_t device;       /* CUDA device ordinal                                              */
  void* cuda_stream;    /* cudaStream_t all work is ordered on (NULL = default stream)     */
  int32_t batch_size;   /* samples per database (>= 1; 0 is treated as 1).  With
                           world_size > 1 this is the GLOBAL batch (see rank)               */
  int32_t max_iters;    /* per-stratum round cap; 0 = default 100000                        */
  int64_t arena_bytes;  /* initial per-round scratch arena; 0 = auto (grows on demand)      */
  int32_t micro_batch;  /* samples per fixpoint pass; 0 = auto: the largest power of two
                           whose packed keys fit the direct-mapped store (samples are
                           independent databases), else the whole batch  */
  int32_t rank;         /* world_size > 1: this context owns the contiguous sample shard
                           [lo, hi) of rank `rank` (lo = rank*(B/W) + min(rank, B%W), sizes
                           differing by at most one).  Sample ids crossing
                           the ABI (facts_push, output_get) are GLOBAL ids; pushing a
                           sample outside the shard is a RANGE error.  Fact ids stay
                           local to the context (the distributed layer, dist.py, maps
                           them to global ids).  The fixpoint has no collective.       */
  int32_t world_size;   /* number of ranks sharing the batch (0 or 1 = unsharded)          */
  void* nccl_comm;      /* unused: batch-sharded collectives run above the ABI (dist.py);
                           key-partitioned runs use lobster_partition                       */
} lobster_options;

/* Create a context on options->device.  options may be NULL (device 0, default
 * stream, batch 1).  Errors: CUDA (no device), OOM. */
lobster_status lobster_create(const lobster_options* options, lobster_ctx** out);
void lobster_destroy(lobster_ctx* ctx);
/* Message of the last failed call on ctx; valid until the next call on ctx. */
const char* lobster_last_error(const lobster_ctx* ctx);

/* Load a program (subset of Fig. 3c syntax):
 *     type Cell = u32                                  -- alias, ignored (columns are int32)
 *     type edge(x: Cell, y: Cell)                      -- batched input relation
 *     shared type composition(a: i32, b: i32, c: i32)  -- input without a sample column
 *     rel path(x, y) :- edge(x, y) or (path(x, z) and edge(z, y)).
 *     rel endpoints_connected() :- is_endpoint(x), is_endpoint(y), path(x, y), x != y.
 *     output endpoints_connected                       -- gradients are produced for outputs
 * Bodies are conjunctions (',' or 'and') and disjunctions ('or', split into one
 * rule per disjunct, left to right) of atoms and comparisons `e1 op e2`, op one
 * of == != < <= > >=.  Atom arguments are variables or integer constants.
 * Integer expressions (§5.2 "eval"): head arguments and
 * comparison sides may be expressions over the rule's variables and
 * constants with + - * / % and unary - (C precedence, parentheses), int32
 * two's-complement; / and % truncate toward zero and a division by zero fails
 * the derivation.  Comparisons between variables / constants run in every
 * kernel; a rule with an arithmetic head or an arithmetic comparison must not
 * be recursive (its body is evaluated into an internal relation __eval<k>,
 * whose projection evaluates the expressions as bytecode), and the domain of a
 * computed column is inferred by interval arithmetic (RANGE if a computed
 * column feeds its own domain).  Every rule needs at least one batched body
 * atom.
 * Stratification: SCCs of the predicate dependency graph in topological order
 * (PAPER.md:383-389).  Errors: PARSE ("line:col: msg"; unbound head variable,
 * unknown relation, arity mismatch); INVALID_ARG (bad semiring); STATE (called
 * twice).  No device work. */
lobster_status lobster_program_load(lobster_ctx* ctx, const char* program_text, lobster_semiring semiring);

/* Append n facts to input relation `relation`.
 *   columns    : `arity` pointers, each to n int32 values (host or device memory,
 *                detected per pointer); may be NULL when arity == 0
 *   sample_ids : n int32 in [0, batch_size) (host or device), or in the context's
 *                shard [lo, hi) when world_size > 1; NULL for a shared relation
 *   probs      : n float in [0,1] (host or device); NULL = 1.0; ignored under UNIT
 * Fact ids are dense in push order: [*first_fact_id, *first_fact_id + n).
 * The data is copied before return; the caller keeps ownership of its buffers.
 * Duplicate tuples within a sample are ⊕-merged at run (reading 16).
 * Errors: SCHEMA (unknown input relation, missing sample ids), RANGE (prob NaN
 * or outside [0,1]; sample id out of range), STATE (before program_load). */
lobster_status lobster_facts_push(lobster_ctx* ctx, const char* relation, int64_t n,
                                  const int32_t* const* columns, const int32_t* sample_ids,
                                  const float* probs, int64_t* first_fact_id);

typedef struct {
  int32_t strata, rounds_total;   /* strata evaluated; rounds summed over strata           */
  int64_t tuples_derived;         /* Σ final IDB tuples                                   */
  int64_t candidates;             /* Σ join outputs (|C|) over all rounds                 */
  double ms_total, ms_join, ms_sort, ms_reduce, ms_merge, ms_grad, ms_comm;
  int64_t bytes_algorithmic;      /* SURVEY §8(d) B_alg summed over rounds               */
  /* the fused row-centric join + direct ⊕ kernel (the dominant kernel on
     bounded-fan-out programs): launches, CUDA-event time, probe rows and
     candidates it processed, and its row bytes (key + tag) for §8(d) bytes   */
  int64_t fj_launches, fj_probe_rows, fj_candidates;
  double ms_fused_join;           /* CUDA-event time of the TIMED fused launches only      */
  int32_t fj_row_bytes;
  int32_t tile_strata;            /* strata run in ONE launch by the small-domain kernel
                                     (k_tile.cu: per-sample dense relations in shared memory) */
  /* the fused launches timed with CUDA events (every k-th, LOBSTER_JOIN_TIMING_EVERY,
     default 4) and the probe rows / candidates of exactly those launches: their
     bytes over ms_fused_join is the kernel's measured throughput                   */
  int64_t fj_timed_launches, fj_timed_probe_rows, fj_timed_candidates;
} lobster_run_stats;

/* Evaluate every stratum to fixpoint (termination: no new tuple and no tag whose
 * fp32 bits changed, reading 1), then — under DIFF_MAX_MULT_PROB — walk the
 * witnesses of every `output` relation and build its per-tuple gradients.
 * Blocking on the context stream.  stats may be NULL.
 * Errors: STATE (no program), OOM, ITER_CAP (state of the last round is
 * readable), RANGE (packed key > 64 bits or witness > 32 bits), CUDA. */
lobster_status lobster_run(lobster_ctx* ctx, lobster_run_stats* stats);

typedef struct {
  int64_t n;                      /* rows                                                  */
  int32_t arity;
  int32_t on_device;              /* 1: pointers are device pointers                        */
  const int32_t* sample_ids;      /* n (global sample id of each row)                       */
  const int32_t* const* columns;  /* arity pointers to n int32; rows sorted by (sample, cols) */
  const float* probs;             /* n; NULL under UNIT; add-mult is unclamped      */
  const int64_t* sample_offsets;  /* B+1 (B = this context's samples: batch_size, or hi-lo
                                     when sharded): rows of sample lo+s are [off[s], off[s+1]) */
  const int64_t* grad_offsets;    /* n+1, DIFF_* output relations only, else NULL (for
                                     DIFF_TOP1_PROOFS the ids are the tuple's proof)         */
  const int64_t* grad_fact_ids;   /* grad_offsets[n] ids, ascending within each row         */
  const float* grad_values;       /* ∂probs[row] / ∂p(fact), fp64-accumulated, rounded to fp32 */
} lobster_output;

/* Views of relation `relation` (any IDB relation; gradients only for relations
 * marked `output`).  where: 0 = host copies, 1 = device pointers.  Views are
 * owned by ctx and valid until the next push / run / program_load / destroy.
 * Errors: INVALID_ARG (unknown relation or bad `where`), STATE (no successful run). */
lobster_status lobster_output_get(lobster_ctx* ctx, const char* relation, int32_t where, lobster_output* out);

/* Optional: dense input-fact gradient of Σ_rows upstream[row] · probs[row] for an
 * `output` relation: grad_facts[f] = Σ_rows upstream[row] · ∂probs[row]/∂p_f,
 * a deterministic segmented sum (no atomics).  upstream: n floats, grad_facts:
 * (number of pushed facts) floats; both device pointers.  Errors: STATE,
 * INVALID_ARG (not an output relation / not DIFF_MAX_MULT_PROB). */
lobster_status lobster_output_backward(lobster_ctx* ctx, const char* relation,
                                       const float* upstream, float* grad_facts);

/* diff-top-1-proofs exclusion groups ("ensures that no conflict is
 * present"): facts [first_fact_id, first_fact_id + n) of the current database
 * get group_ids (n int32, host or device; -1 = none).  Two facts with the same
 * group id >= 0 are mutually exclusive: a conjunction holding both is a
 * conflict and yields no proof.  Call after lobster_facts_push, before
 * lobster_run.  Ignored by the other semirings.  Errors: STATE (no program, or
 * after run), INVALID_ARG (range outside the pushed facts). */
lobster_status lobster_facts_groups(lobster_ctx* ctx, int64_t first_fact_id, int64_t n, const int32_t* group_ids);

/* Number of facts pushed into the current database (size of grad_facts). */
int64_t lobster_num_facts(const lobster_ctx* ctx);

/* Diagnostics: CUDA kernels this library has launched in this process so far. */
int64_t lobster_kernel_launches(void);

/* ---- Key-partitioned evaluation of ONE database across ranks (SURVEY §8(f)
 * NEXT-3; the paper's TC / Same Generation inputs outgrow one GPU, P:799-803,
 * P:1151-1172).  Every rank pushes the SAME facts (inputs are replicated);
 * each IDB tuple is owned by the rank its packed key hashes to.  Each round the
 * candidates travel to their owners (an all-to-all over the group) and Σ|Δ'| is
 * summed over all ranks, so every rank runs the same rounds (Alg. 1).
 * A relation read by a later stratum is gathered whole onto every rank at the
 * end of its stratum; the others stay partitioned: lobster_output_get returns
 * this rank's tuples, and the union over ranks is the relation.
 * Limits: unit, max-min, add-mult; linear recursion (a rule reads at most one
 * relation of its own stratum); not combined with batch sharding. */
typedef struct lobster_group lobster_group;
/* world_size contexts of THIS process, one host thread each (any devices):
 * exchanges are peer copies between two host barriers.  Owned by the caller;
 * must outlive the contexts that use it. */
lobster_status lobster_group_local(int32_t world_size, lobster_group** out);
/* One process per GPU over NCCL (libnccl.so.2, loaded at run time): rank 0
 * calls lobster_nccl_id and hands the 128 bytes to every rank (e.g. a
 * torch.distributed broadcast); each rank then creates its group member on
 * `device`.  Errors: NCCL (library missing, init failure), INVALID_ARG. */
lobster_status lobster_nccl_id(uint8_t* id /* 128 bytes */);
lobster_status lobster_group_nccl(const uint8_t* id, int32_t rank, int32_t world_size, int32_t device,
                                  lobster_group** out);
void lobster_group_destroy(lobster_group* group);
/* Evaluate ctx's databases as `rank` of `group` (NULL group: off).  Call after
 * lobster_program_load.  Every rank of the group must call lobster_run for
 * the same database.  Errors: STATE (no program), INVALID_ARG (rank, semiring,
 * world_size > 1), SCHEMA (a rule reading its own stratum twice). */
lobster_status lobster_partition(lobster_ctx* ctx, lobster_group* group, int32_t rank);

#ifdef __cplusplus
}
#endif
#endif /* LOBSTER_H */
