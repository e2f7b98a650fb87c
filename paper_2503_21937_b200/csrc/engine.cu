// engine.cu — host driver of the semi-naive fixpoint (B1-B4 of SURVEY §1.2):
// relation store, ingest, planner, per-round loop, witness walk, outputs, and
// the extern "C" boundary of include/lobster.h.
//
// Per stratum (Alg. 1; §3.4):
//   round 1 ("seed", reading 3): rules whose body atoms are all external
//   round r>1: for each rule with local atoms and each local position j:
//              B_1^new ⋈ .. ⋈ Δ_j ⋈ .. ⋈ B_k^old      (Fig. 10 Join)
//   every round: C -> radix sort -> segmented ⊕ = U -> diff against F ->
//              Δ' (increments), F ⊕= changed, F ∪= new    (Fig. 10 Stratum)
//   stop when Σ|Δ'| = 0 (reading 1).
// Device work is all in the kernels of k_*.cu; this file only plans and
// launches.  There is no CPU compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "devmem.hpp"
#include "kernels.cuh"
#include "lobster.h"
#include "program.hpp"
#include "xfer.hpp"

namespace lob {

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static int bits_for(uint64_t range) { return range == 0 ? 0 : 64 - __builtin_clzll(range); }

// Merge bit moves that are adjacent in both source and destination with the
// same source word (e.g. (sample, x) kept together from probe to head): fewer
// moves per output key in the join kernels.
static void merge_moves(Move* mv, int& n) {
  bool changed = true;
  while (changed) {
    changed = false;
    for (int a = 0; a < n && !changed; ++a)
      for (int b = 0; b < n && !changed; ++b) {
        if (a == b || mv[a].src != mv[b].src) continue;
        if (mv[a].sshift == mv[b].sshift + mv[b].bits && mv[a].dshift == mv[b].dshift + mv[b].bits &&
            mv[a].bits + mv[b].bits <= 63) {
          mv[b].bits = (uint8_t)(mv[a].bits + mv[b].bits);
          mv[a] = mv[n - 1];
          --n;
          changed = true;
        }
      }
  }
  for (int i = 0; i < n;)  // zero-width moves contribute nothing
    if (mv[i].bits == 0) mv[i] = mv[--n]; else ++i;
}

constexpr int MAXARITY = 8;

struct Layout {
  bool has_sample = false;
  int sbits = 0, sshift = 0;
  std::vector<int> bits, shift;
  std::vector<int32_t> mins;
  int total = 0;
};

struct Staged {
  DBuf<int32_t> cols[MAXARITY];
  DBuf<int32_t> sid;
  DBuf<float> p;
  DBuf<int32_t> fid;
  int64_t n = 0;
};

struct RelState {
  Layout L;
  DBuf<uint64_t> key, key2;
  DBuf<float> p, p2;
  DBuf<uint32_t> w, w2;
  DBuf<int32_t> fid;
  int64_t n = 0;
  DBuf<uint64_t> dkey;
  DBuf<float> dp;
  DBuf<uint32_t> dw;
  int64_t nd = 0;
  DBuf<uint64_t> okey;
  DBuf<float> op;
  DBuf<uint32_t> ow;
  int64_t no = 0;
  bool need_old = false;
  bool build_local = false;  // read as B^new / B^old by a rule with >= 2 local atoms
  // dense direct-mapped store (NEXT-1) while the relation's stratum runs;
  // keys of Δ / C / U are then u32 (packed key < 2^31)
  bool dense = false;
  bool direct = false;  // dense + idempotent ⊕ fused into the join write (kernels.cuh Direct)
  int64_t nslots = 0;
  DevMem dirf;          // direct store words
  DBuf<uint32_t> dirty;  // bitmap of the slots improved this round
  DBuf<unsigned long long> dctr;  // |Δ'| counter of the single-pass extraction
  DBuf<uint32_t> ndev;             // |Δ'| of the last extraction (device)
  DBuf<uint32_t> ectr;             // one-launch extraction counters (rows, finished CTAs), kept zeroed
  bool async = false;              // rounds run without a host sync: Δ size lives in ndev
  bool lazy = false;               // finished direct store not yet compacted to the sorted form (n is exact)
  unsigned long long* ring_dst = nullptr;  // async: host-mapped word for (seq << 32 | |Δ'|)
  uint32_t ring_seq = 0;
  // max-mult direct words (kernels.cuh MxEnc): witness field WB = wrb + wT bits,
  // round stamps in the SB = 34 - WB bits above it when they hold every round
  int wT = 0, wrb = 0, wWB = 0;
  bool stamp_mode = false;
  unsigned long long smax = 0;
  int64_t cand_bound = 0;         // upper bound on slots dirtied this round
  DBuf<float> dfp;
  DBuf<uint32_t> dfw, dfbits, dkey32, ckey32, ckey32b;
  DBuf<uint64_t> ckey, ckey2, cv64, cv64b;
  DBuf<uint32_t> cv32, cv32b;
  int64_t nc = 0;
  Staged in;
  // outputs
  bool out_dev_ready = false, out_host_ready = false;
  DBuf<int32_t> o_sid, o_cols;
  DBuf<int64_t> o_soff;
  HBuf<int32_t> h_sid, h_cols;
  HBuf<float> h_p;
  HBuf<int64_t> h_soff, h_goff, h_gfid;
  HBuf<float> h_gval;
  std::vector<const int32_t*> col_ptrs;
  bool has_grad = false;
  DBuf<int64_t> goff, gfid;
  DBuf<float> gval;
  int64_t ng = 0;
  // micro-batched runs: `output` relations accumulated over sample chunks
  bool retained = true;
  DBuf<int32_t> acc_sid, acc_col[MAXARITY];
  DBuf<float> acc_p, acc_gval;
  DBuf<int64_t> acc_goff, acc_gfid;
  int64_t acc_n = 0, acc_ng = 0;
  // diff-top-1-proofs: proof index (keys = the stored tuples, offset + length
  // into the pool of fact ids) and this round's Δ' proof handles
  DBuf<uint64_t> pkey, pof, pkey2, pof2, dof;
  DBuf<uint32_t> pln, pln2, dln, pool, pool2;
  int64_t npx = 0, pool_n = 0;

  void bind(cudaStream_t st) {
    for (auto* b : {&key, &key2, &dkey, &okey, &ckey, &ckey2, &cv64, &cv64b}) b->bind(st);
    for (auto* b : {&p, &p2, &dp, &op, &gval}) b->bind(st);
    for (auto* b : {&w, &w2, &dw, &ow, &cv32, &cv32b, &dfw, &dfbits, &dkey32, &ckey32, &ckey32b, &dirty})
      b->bind(st);
    dfp.bind(st);
    dirf.bind(st);
    for (auto* b : {&fid, &o_sid, &o_cols}) b->bind(st);
    for (auto* b : {&o_soff, &goff, &gfid}) b->bind(st);
    dctr.bind(st);
    ndev.bind(st);
    ectr.bind(st);
    for (auto& c : in.cols) c.bind(st);
    for (auto& c : acc_col) c.bind(st);
    acc_sid.bind(st);
    acc_p.bind(st);
    acc_gval.bind(st);
    acc_goff.bind(st);
    acc_gfid.bind(st);
    for (auto* b : {&pkey, &pof, &pkey2, &pof2, &dof}) b->bind(st);
    for (auto* b : {&pln, &pln2, &dln, &pool, &pool2}) b->bind(st);
    in.sid.bind(st);
    in.p.bind(st);
    in.fid.bind(st);
  }
};

// Sorted index over one relation version: key = [sample][order...], prefix =
// sample + the first nbound columns of `order`.
struct Index {
  const uint64_t* key = nullptr;
  const float* p = nullptr;
  int64_t n = 0;
  DBuf<uint64_t> own_key, tmp_key;
  DBuf<float> own_p, tmp_p;
  DBuf<int64_t> off;
  const int64_t* offp = nullptr;
  DBuf<uint4> rec;                 // fan-out <= 4: per-prefix 32-B records (kernels.cuh JoinPlan::brec)
  const uint4* recp = nullptr;
  int64_t nprefix = 0;
  int free_bits = 0, prefix_bits = 0;
  int64_t maxdeg = -1;  // max rows per prefix (static CSR indexes), -1 unknown

  bool has_sample = false;
  int sshift = 0, sbits = 0;
  std::vector<int> col_shift, col_bits;
};

struct Table {  // probe side of a join step
  const void* key = nullptr;
  bool k32 = false;  // u32 keys (Δ of a dense relation)
  int64_t n = 0;
  std::vector<const float*> tags;
  std::vector<int> tag_atom;
  bool has_sample = true;
  int sshift = 0, sbits = 0;
  std::vector<int> vshift, vbits;  // per var id, -1 unbound
};

enum Version { V_EXT = 0, V_NEW = 1, V_OLD = 2, V_DELTA = 3 };

struct Ctx {
  lobster_options opt{};
  int32_t sample_base = 0;  // first global sample id of this context's shard (world_size > 1)
  cudaStream_t st = nullptr;
  std::string err;
  bool sticky = false;
  bool loaded = false, ran = false, dirty = false;
  int semi = 0;
  bool omin = false;  // diff-max-min-prob (semi == S_MAXMULT internally)
  bool top1 = false;  // diff-top-1-proofs (semi == S_MAXMULT internally; sorted stores, k_top1.cu)
  bool dadd = false;  // diff-add-mult-prob (semi == S_ADDMULT internally; adjoint-program gradients)
  bool unbounded_tags = false;  // internal child contexts: pushed tags are unclamped add-mult values
  std::string program_text;
  DBuf<int32_t> fact_group;  // top-1-proof exclusion group per fact (-1: none)
  bool has_groups = false;
  Program prog;
  std::vector<std::unique_ptr<RelState>> rels;
  int64_t next_fact = 0;
  Arena arena;
  int64_t* hbuf = nullptr;  // pinned
  std::map<std::pair<int, std::vector<int>>, std::unique_ptr<Index>> static_idx;
  std::vector<int64_t> class_min, class_max;
  std::vector<int> rule_bits;
  std::vector<std::vector<int>> wshift, wbits;  // per rule, per nonhead var
  DBuf<float> fact_p;
  lobster_run_stats stats{};
  unsigned long long* d_ncand = nullptr;  // device counter of fused-join candidates
  // bit-sliced frontier (k_slice.cu): relation / round bits, Δ triples, per-rule CSR
  struct SliceBufs {
    DBuf<uint32_t> Rb, Nb, dt, dwi, dbits, deg, pos, cnt, scan;
    std::vector<std::unique_ptr<DBuf<uint32_t>>> off, nbr;
    DBuf<unsigned long long> tup;
  } sl;
  bool no_slice = getenv("LOBSTER_NO_SLICE") != nullptr;  // A/B: per-sample bitmap rounds
  bool fj_prefetch = !getenv("LOBSTER_FJ_PREFETCH") || atoi(getenv("LOBSTER_FJ_PREFETCH")) != 0;
  bool force_slot_join = getenv("LOBSTER_SLOT_JOIN") != nullptr;  // A/B: slot-balanced join only
  int max_iters = 100000;
  // key-partitioned evaluation of one database (lobster_partition; SURVEY §8(f)
  // NEXT-3): every IDB tuple lives on the rank its key hashes to
  Xfer* xfer = nullptr;
  int part_rank = 0;
  int64_t* hx = nullptr;  // pinned: per-peer counts (3 x 64)
  int32_t batch_cur = 1;  // samples of the (micro-)batch being evaluated
  bool micro = false;     // the last run was split into sample chunks
  int log_level = getenv("LOBSTER_LOG") ? atoi(getenv("LOBSTER_LOG")) : 0;  // 1: per-run timing line, 2: + rounds
  std::vector<std::array<int64_t, 4>> trace;  // per round: first event index, fused probe rows, |Δ'|, stratum
  std::vector<std::pair<const char*, cudaEvent_t>> marks;  // LOBSTER_LOG>=1: GPU timeline sections of a run
  void mark(const char* what) {
    if (log_level < 1) return;
    cudaEvent_t e = get_event();
    cudaEventRecord(e, st);
    marks.push_back({what, e});
  }
  double host_ms[8] = {};
  struct HostTimer {  // accumulates host wall time of a scope (diagnostics)
    double& acc;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    bool on = true;
    explicit HostTimer(double& a) : acc(a) {}
    void stop() {
      if (on) acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      on = false;
    }
    ~HostTimer() { stop(); }
  };
  bool force_sorted = getenv("LOBSTER_SORTED_STORE") != nullptr;      // A/B: merge-based store
  bool force_sort_dedup = getenv("LOBSTER_SORT_DEDUP") != nullptr;    // A/B: radix sort + seg ⊕ on dense
  bool sorted_delta = getenv("LOBSTER_SORTED_DELTA") != nullptr;      // A/B: fully slot-ordered Δ' (2 launches)
  bool eager_compact = getenv("LOBSTER_EAGER_COMPACT") != nullptr;    // A/B: compact direct stores at stratum end
  // time every k-th fused join launch (LOBSTER_JOIN_TIMING_EVERY, default 4; 1 = all).
  // Other phases keep an event pair per launch: sampling them by round was tried and
  // rejected — rounds are too uneven (C4: 9 rounds, two of them hold most of the
  // work), and their sums feed the fixpoint-phase roofline of the non-fused configs.
  // That timing costs ~2 ms of a 32 ms C3 step and 0.25 ms of C1's 0.95 ms.
  int join_timing_every = getenv("LOBSTER_JOIN_TIMING_EVERY") ? std::max(1, atoi(getenv("LOBSTER_JOIN_TIMING_EVERY"))) : 4;
  uint64_t fj_seq = 0;
  std::set<int> timed_rounds;  // async rounds of the current stratum whose fused join is timed
  int64_t num_facts_db = 0;
  // timing
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  size_t ev_used = 0;
  std::vector<cudaEvent_t> ev_pool;

  // ------------------------------------------------------------------ util
  void sync() { cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"); }
  void kcheck(const char* what) { cuda_check(cudaGetLastError(), what); }
  template <typename T>
  T read_dev(const T* d) {
    cuda_check(cudaMemcpyAsync(hbuf, d, sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
    sync();
    T v;
    std::memcpy(&v, hbuf, sizeof(T));
    return v;
  }
  cudaEvent_t get_event() {
    if (ev_used < ev_pool.size()) return ev_pool[ev_used++];
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    ev_pool.push_back(e);
    ev_used++;
    return e;
  }
  struct Phase {
    Ctx* c;
    int id;
    cudaEvent_t a = nullptr;
    Phase(Ctx* cc, int i, bool on = true) : c(cc), id(i) {
      if (!on) return;
      a = c->get_event();
      cudaEventRecord(a, c->st);
    }
    ~Phase() {
      if (!a) return;
      cudaEvent_t b = c->get_event();
      cudaEventRecord(b, c->st);
      c->ev.push_back({id, {a, b}});
    }
  };
  // async sections: one event pair around all their rounds; their settle time is
  // the section's span minus its (individually timed) fused joins — per-launch
  // event pairs for the extraction would cost ~1 µs of host time each at
  // finish_run (hundreds per run)
  struct Section {
    cudaEvent_t a, b;
    size_t ev0, ev1;
  };
  std::vector<Section> sections;

  ~Ctx() {
    for (auto& r : rels) r.reset();
    static_idx.clear();
    arena.free_all();
    fact_p.release();
    if (st) cudaStreamSynchronize(st);
    if (d_ncand) cudaFree(d_ncand);
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (hbuf) cudaFreeHost(hbuf);
    if (hx) cudaFreeHost(hx);
    if (hplan) cudaFreeHost(hplan);
    if (hring) cudaFreeHost(hring);
  }

  // --------------------------------------------------------------- create
  void create(const lobster_options* o) {
    if (o) opt = *o;
    if (opt.batch_size < 1) opt.batch_size = 1;
    // Sharded batch: batch_size is the GLOBAL batch and this
    // context owns the contiguous shard [lo, hi) of `rank`; sample ids cross the
    // ABI as global ids and are rebased to the shard inside.
    if (opt.world_size > 1) {
      if (opt.rank < 0 || opt.rank >= opt.world_size) throw Failure(LOBSTER_E_INVALID_ARG, "rank outside [0, world_size)");
      const int64_t B = opt.batch_size, W = opt.world_size, base = B / W, extra = B % W;
      const int64_t lo = opt.rank * base + std::min<int64_t>(opt.rank, extra);
      const int64_t hi = lo + base + (opt.rank < extra ? 1 : 0);
      if (hi <= lo) throw Failure(LOBSTER_E_INVALID_ARG, "world_size larger than the batch");
      sample_base = (int32_t)lo;
      opt.batch_size = (int32_t)(hi - lo);
    }
    max_iters = opt.max_iters > 0 ? opt.max_iters : 100000;
    int ndev = 0;
    cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (opt.device < 0 || opt.device >= ndev) throw Failure(LOBSTER_E_CUDA, "no such CUDA device");
    cuda_check(cudaSetDevice(opt.device), "cudaSetDevice");
    st = reinterpret_cast<cudaStream_t>(opt.cuda_stream);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, opt.device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cuda_check(cudaMallocHost(&hbuf, 64), "cudaMallocHost");
    arena.bind(st);
    fact_p.bind(st);
    fact_group.bind(st);
    for (auto* b : {&sl.Rb, &sl.Nb, &sl.dt, &sl.dwi, &sl.dbits, &sl.deg, &sl.pos, &sl.cnt, &sl.scan}) b->bind(st);
    sl.tup.bind(st);
    if (opt.arena_bytes > 0) arena.reserve_initial((size_t)opt.arena_bytes);
  }

  // ---------------------------------------------------------- program load
  void load(const char* text, int semiring) {
    if (loaded) throw Failure(LOBSTER_E_STATE, "program already loaded");
    if (semiring < 0 || semiring > 6) throw Failure(LOBSTER_E_INVALID_ARG, "bad semiring");
    if (!text) throw Failure(LOBSTER_E_INVALID_ARG, "program text is NULL");
    prog = parse_program(text);
    // diff-max-min-prob runs on the max-mult machinery (packed (p, stamp,
    // witness) words, strict improvement, tie rules 8a/8b) with ⊗ = min and a
    // one-hot gradient (reading "diff-max-min")
    omin = semiring == LOBSTER_DIFF_MAX_MIN_PROB;
    top1 = semiring == LOBSTER_DIFF_TOP1_PROOFS;
    // diff-add-mult-prob: the forward fixpoint is add-mult; gradients come from
    // the adjoint program (dadd_gradients)
    dadd = semiring == LOBSTER_DIFF_ADD_MULT_PROB;
    if (dadd)
      for (auto& R : prog.rules) {
        bool arith = false;
        for (auto& e : R.head_expr) arith |= e.op != 0;
        for (auto& c : R.cmps) arith |= c.is_expr;
        if (arith) throw Failure(LOBSTER_E_PARSE, "diff-add-mult-prob with arithmetic (eval) rules is not supported");
      }
    semi = (omin || top1) ? S_MAXMULT : (dadd ? S_ADDMULT : semiring);
    program_text = text;
    for (auto& r : prog.rels)
      if (r.arity > MAXARITY) throw Failure(LOBSTER_E_PARSE, "relation " + r.name + ": arity above 8 is unsupported");
    for (auto& R : prog.rules) {
      if ((int)R.body.size() > MAXT) throw Failure(LOBSTER_E_PARSE, "rule with more than 6 body atoms is unsupported");
      if (R.var_names.size() > 9) throw Failure(LOBSTER_E_PARSE, "rule with more than 9 variables is unsupported");
    }
    rels.clear();
    for (size_t i = 0; i < prog.rels.size(); ++i) {
      rels.emplace_back(new RelState());
      rels.back()->bind(st);
    }
    // relations that need an "old" version: local atoms placed after another
    // local atom of the same stratum in some rule body (B_k^old)
    for (auto& R : prog.rules) {
      int s = prog.rels[R.head_rel].stratum;
      int seen = 0;
      for (auto& a : R.body) {
        if (!prog.rels[a.rel].input && prog.rels[a.rel].stratum == s) {
          if (seen) rels[a.rel]->need_old = true;
          seen++;
        }
      }
      if (seen >= 2)
        for (auto& a : R.body)
          if (!prog.rels[a.rel].input && prog.rels[a.rel].stratum == s) rels[a.rel]->build_local = true;
    }
    rule_bits.assign(prog.rels.size(), 0);
    for (size_t r = 0; r < prog.rels.size(); ++r)
      rule_bits[r] = prog.rels[r].nrules > 1 ? bits_for((uint64_t)prog.rels[r].nrules - 1) : 0;
    loaded = true;
  }

  // ------------------------------------------------------------ facts push
  void new_database() {
    for (auto& r : rels) {
      r->in.n = 0;
      r->n = r->nd = r->no = r->nc = 0;
      r->lazy = false;
      r->out_dev_ready = r->out_host_ready = false;
      r->has_grad = false;
    }
    static_idx.clear();
    next_fact = 0;
    has_groups = false;
    ran = false;
  }

  // top-1-proof exclusion groups of facts [first, first + n)
  void set_groups(int64_t first, int64_t n, const int32_t* groups) {
    if (!loaded) throw Failure(LOBSTER_E_STATE, "facts_groups before program_load");
    if (n < 0 || first < 0 || first + n > next_fact || (n > 0 && !groups))
      throw Failure(LOBSTER_E_INVALID_ARG, "group range outside the pushed facts");
    if (ran) throw Failure(LOBSTER_E_STATE, "facts_groups after run (push the next database first)");
    if (n == 0) return;
    cuda_check(cudaMemcpyAsync(fact_group.ptr() + first, groups, n * 4, cudaMemcpyDefault, st), "push groups");
    has_groups = true;
    dirty = true;
  }

  // key-partitioned evaluation of this context's database as `rank` of the group
  void set_partition(Xfer* x, int rank) {
    if (!loaded) throw Failure(LOBSTER_E_STATE, "partition before program_load");
    if (x && (rank < 0 || rank >= x->world)) throw Failure(LOBSTER_E_INVALID_ARG, "rank outside the group");
    if (x && opt.world_size > 1)
      throw Failure(LOBSTER_E_INVALID_ARG, "key partitioning and batch sharding (world_size > 1) are exclusive");
    if (x && (semi == S_MAXMULT || dadd))
      throw Failure(LOBSTER_E_INVALID_ARG, "key partitioning supports unit, max-min and add-mult (no gradients)");
    if (x)
      for (const Rule& R : prog.rules) {
        const int s = prog.rels[R.head_rel].stratum;
        int nloc = 0;
        for (auto& a : R.body) nloc += (!prog.rels[a.rel].input && prog.rels[a.rel].stratum == s) ? 1 : 0;
        if (nloc > 1)
          throw Failure(LOBSTER_E_SCHEMA, "key partitioning: a rule for " + prog.rels[R.head_rel].name +
                                              " reads its own stratum twice (linear recursion only)");
      }
    xfer = x;
    part_rank = x ? rank : 0;
  }

  void push(const char* relname, int64_t n, const int32_t* const* columns, const int32_t* sample_ids,
            const float* probs, int64_t* first) {
    if (!loaded) throw Failure(LOBSTER_E_STATE, "facts_push before program_load");
    if (!relname) throw Failure(LOBSTER_E_INVALID_ARG, "relation name is NULL");
    auto it = prog.rel_id.find(relname);
    if (it == prog.rel_id.end() || !prog.rels[it->second].input)
      throw Failure(LOBSTER_E_SCHEMA, std::string("unknown input relation ") + relname);
    if (n < 0) throw Failure(LOBSTER_E_INVALID_ARG, "negative row count");
    const Relation& R = prog.rels[it->second];
    if (R.arity > 0 && n > 0 && !columns) throw Failure(LOBSTER_E_INVALID_ARG, "columns is NULL");
    if (!R.shared && n > 0 && !sample_ids)
      throw Failure(LOBSTER_E_SCHEMA, std::string("relation ") + relname + " is batched: sample ids required");
    if (ran) new_database();
    RelState& S = *rels[it->second];
    const int64_t base = S.in.n;
    if (next_fact + n > INT32_MAX) throw Failure(LOBSTER_E_RANGE, "more than 2^31 facts");
    for (int c = 0; c < R.arity; ++c) {
      if (!columns[c] && n > 0) throw Failure(LOBSTER_E_INVALID_ARG, "column pointer is NULL");
      S.in.cols[c].reserve(base + n, base);
    }
    S.in.sid.reserve(base + n, base);
    S.in.p.reserve(base + n, base);
    S.in.fid.reserve(base + n, base);
    if (n > 0) {
      for (int c = 0; c < R.arity; ++c)
        cuda_check(cudaMemcpyAsync(S.in.cols[c].ptr() + base, columns[c], n * sizeof(int32_t), cudaMemcpyDefault, st),
                   "push columns");
      if (!R.shared)
        cuda_check(cudaMemcpyAsync(S.in.sid.ptr() + base, sample_ids, n * sizeof(int32_t), cudaMemcpyDefault, st),
                   "push sample ids");
      if (probs && semi != S_UNIT)
        cuda_check(cudaMemcpyAsync(S.in.p.ptr() + base, probs, n * sizeof(float), cudaMemcpyDefault, st), "push probs");
      else
        launch_fill_f32(S.in.p.ptr() + base, n, 1.0f, st);
      launch_iota_i32(S.in.fid.ptr() + base, n, (int32_t)next_fact, st);
      fact_group.reserve(next_fact + n, next_fact);  // no exclusion group until lobster_facts_groups
      cuda_check(cudaMemsetAsync(fact_group.ptr() + next_fact, 0xff, n * 4, st), "memset");
      // validation (reading: S:46 range errors)
      uint32_t* flags = reinterpret_cast<uint32_t*>(hbuf);
      uint32_t* dflag = arena.get<uint32_t>(1);
      cuda_check(cudaMemsetAsync(dflag, 0, 4, st), "memset");
      if (sample_base && !R.shared) launch_add_i32(S.in.sid.ptr() + base, n, -sample_base, st);
      launch_validate((probs && semi != S_UNIT && !unbounded_tags) ? S.in.p.ptr() + base : nullptr,
                      R.shared ? nullptr : S.in.sid.ptr() + base, n, opt.batch_size, dflag, st);
      kcheck("validate");
      cuda_check(cudaMemcpyAsync(flags, dflag, 4, cudaMemcpyDeviceToHost, st), "D2H");
      sync();
      arena.reset();
      if (*flags & 1u) throw Failure(LOBSTER_E_RANGE, std::string("relation ") + relname + ": probability NaN or outside [0,1]");
      if (*flags & 2u) throw Failure(LOBSTER_E_RANGE, std::string("relation ") + relname + ": sample id out of range");
    }
    S.in.n = base + n;
    *first = next_fact;
    next_fact += n;
    dirty = true;
  }

  // ---------------------------------------------------------------- layout
  Layout make_layout(int r) {
    const Relation& R = prog.rels[r];
    Layout L;
    L.has_sample = !R.shared;
    L.sbits = L.has_sample ? bits_for((uint64_t)batch_cur - 1) : 0;
    int pos = 0;
    L.bits.assign(R.arity, 0);
    L.shift.assign(R.arity, 0);
    L.mins.assign(R.arity, 0);
    for (int c = R.arity - 1; c >= 0; --c) {
      int cl = R.col_class[c];
      L.bits[c] = bits_for((uint64_t)(class_max[cl] - class_min[cl]));
      L.mins[c] = (int32_t)class_min[cl];
      L.shift[c] = pos;
      pos += L.bits[c];
    }
    L.sshift = pos;
    L.total = pos + L.sbits;
    if (L.total > 63)
      throw Failure(LOBSTER_E_RANGE, "packed key of relation " + R.name + " needs " + std::to_string(L.total) +
                                         " bits (> 63)");
    return L;
  }

  // ----------------------------------------------------------------- ingest
  void ingest_domains() {
    const int nr = (int)prog.rels.size();
    // A0: per-column min/max of every input relation -> domain classes
    std::vector<std::pair<int, int>> cols;
    for (int r = 0; r < nr; ++r)
      if (prog.rels[r].input)
        for (int c = 0; c < prog.rels[r].arity; ++c) cols.push_back({r, c});
    std::vector<int32_t> mm(cols.size() * 2);
    int32_t* dmm = arena.get<int32_t>((int64_t)mm.size() + 2);
    for (size_t i = 0; i < cols.size(); ++i) {
      mm[2 * i] = INT32_MAX;
      mm[2 * i + 1] = INT32_MIN;
    }
    if (!mm.empty()) {
      cuda_check(cudaMemcpyAsync(dmm, mm.data(), mm.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
      for (size_t i = 0; i < cols.size(); ++i) {
        RelState& S = *rels[cols[i].first];
        launch_minmax(S.in.cols[cols[i].second].ptr(), S.in.n, dmm + 2 * i, st);
      }
      kcheck("minmax");
      cuda_check(cudaMemcpyAsync(mm.data(), dmm, mm.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
      sync();
    }
    class_min.assign(prog.nclasses, INT64_MAX);
    class_max.assign(prog.nclasses, INT64_MIN);
    for (size_t i = 0; i < cols.size(); ++i) {
      if (rels[cols[i].first]->in.n == 0) continue;
      int cl = prog.rels[cols[i].first].col_class[cols[i].second];
      class_min[cl] = std::min<int64_t>(class_min[cl], mm[2 * i]);
      class_max[cl] = std::max<int64_t>(class_max[cl], mm[2 * i + 1]);
    }
    for (int cl = 0; cl < prog.nclasses; ++cl) {
      if (prog.class_has_const[cl]) {
        class_min[cl] = std::min(class_min[cl], prog.class_cmin[cl]);
        class_max[cl] = std::max(class_max[cl], prog.class_cmax[cl]);
      }
    }
    computed_domains();
    for (int cl = 0; cl < prog.nclasses; ++cl)
      if (class_min[cl] > class_max[cl]) class_min[cl] = class_max[cl] = 0;
  }

  // Domains of computed head columns (arithmetic): interval
  // arithmetic over the operand variables' domain classes, unioned into the
  // column's class until nothing grows.  An expression over its own column's
  // class (a value feeding its own domain) is refused.
  void computed_domains() {
    struct Iv { int64_t lo, hi; bool empty; };
    auto clamp32 = [](Iv v) {
      if (v.lo < INT32_MIN || v.hi > INT32_MAX) v.lo = INT32_MIN, v.hi = INT32_MAX;  // int32 wrap: anything
      return v;
    };
    for (int iter = 0;; ++iter) {
      bool grew = false;
      for (const Rule& R : prog.rules)
        for (size_t c = 0; c < R.head_expr.size(); ++c) {
          if (!R.head_expr[c].op) continue;
          const int tcl = prog.rels[R.head_rel].col_class[c];
          std::function<Iv(const Expr&)> iv = [&](const Expr& e) -> Iv {
            if (e.op == '#') return {e.cst, e.cst, false};
            if (e.op == 'v') {
              const int cl = R.var_class[e.var];
              if (cl == tcl)
                throw Failure(LOBSTER_E_RANGE, "a computed column of " + prog.rels[R.head_rel].name +
                                                   " feeds its own domain (unsupported)");
              return {class_min[cl], class_max[cl], class_min[cl] > class_max[cl]};
            }
            const Iv a = iv(e.kids[0]);
            if (e.op == 'n') return clamp32({-a.hi, -a.lo, a.empty});
            const Iv b = iv(e.kids[1]);
            const bool em = a.empty || b.empty;
            switch (e.op) {
              case '+': return clamp32({a.lo + b.lo, a.hi + b.hi, em});
              case '-': return clamp32({a.lo - b.hi, a.hi - b.lo, em});
              case '*': {
                const int64_t p[4] = {a.lo * b.lo, a.lo * b.hi, a.hi * b.lo, a.hi * b.hi};
                return clamp32({*std::min_element(p, p + 4), *std::max_element(p, p + 4), em});
              }
              case '/': {  // |x / y| <= |x| for |y| >= 1
                const int64_t m = std::max(std::llabs(a.lo), std::llabs(a.hi));
                return clamp32({a.lo >= 0 ? 0 : -m, a.hi <= 0 ? 0 : m, em});
              }
              default: {  // % : |r| < |y|, |r| <= |x|, sign of x
                const int64_t m = std::min(std::max(std::llabs(a.lo), std::llabs(a.hi)),
                                           std::max(std::llabs(b.lo), std::llabs(b.hi)) - 1);
                return {a.lo >= 0 ? 0 : -std::max<int64_t>(m, 0), a.hi <= 0 ? 0 : std::max<int64_t>(m, 0), em};
              }
            }
          };
          const Iv v = iv(R.head_expr[c]);
          if (v.empty) continue;  // an operand class without values: the rule derives nothing
          if (v.lo < class_min[tcl]) { class_min[tcl] = v.lo; grew = true; }
          if (v.hi > class_max[tcl]) { class_max[tcl] = v.hi; grew = true; }
        }
      if (!grew) return;
      if (iter >= 64) throw Failure(LOBSTER_E_RANGE, "domains of computed columns do not settle");
    }
  }

  // Per-chunk part of A0: layouts for the current (micro-)batch, witness
  // layouts, then pack + sort + ⊕-merge the facts of samples [s_lo, s_hi)
  // (rebased to 0) of every input relation; shared relations whole.
  void ingest_chunk(int32_t s_lo, int32_t s_hi) {
    const int nr = (int)prog.rels.size();
    for (int r = 0; r < nr; ++r) rels[r]->L = make_layout(r);
    // witness layouts (diff-max-mult): rule index in the top bits, non-head
    // variables below, first variable most significant (tie order, reading 8b)
    wshift.assign(prog.rules.size(), {});
    wbits.assign(prog.rules.size(), {});
    for (size_t ri = 0; ri < prog.rules.size(); ++ri) {
      const Rule& R = prog.rules[ri];
      int tot = 0;
      for (int v : R.nonhead) {
        int cl = R.var_class[v];
        int b = bits_for((uint64_t)(class_max[cl] - class_min[cl]));
        wbits[ri].push_back(b);
        tot += b;
      }
      if (semi == S_MAXMULT && tot > 32 - rule_bits[R.head_rel])
        throw Failure(LOBSTER_E_RANGE, "witness of a rule for " + prog.rels[R.head_rel].name + " needs " +
                                           std::to_string(tot + rule_bits[R.head_rel]) + " bits (> 32)");
      int pos = tot;
      for (size_t i = 0; i < R.nonhead.size(); ++i) {
        pos -= wbits[ri][i];
        wshift[ri].push_back(pos);
      }
    }
    // pack + sort + ⊕-merge duplicates of every input relation (A0)
    for (int r = 0; r < nr; ++r) {
      if (!prog.rels[r].input) continue;
      RelState& S = *rels[r];
      const int64_t n = S.in.n;
      S.n = 0;
      if (n == 0) continue;
      PackPlan pp{};
      pp.ncols = prog.rels[r].arity;
      for (int c = 0; c < pp.ncols; ++c) {
        pp.col[c] = S.in.cols[c].ptr();
        pp.min[c] = S.L.mins[c];
        pp.shift[c] = (uint8_t)S.L.shift[c];
      }
      pp.sample = S.L.has_sample ? S.in.sid.ptr() : nullptr;
      pp.sshift = (uint8_t)S.L.sshift;
      pp.s_lo = s_lo;
      pp.s_hi = s_hi;
      uint64_t* k0 = arena.get<uint64_t>(n);
      uint64_t* k1 = arena.get<uint64_t>(n);
      uint32_t* r0 = arena.get<uint32_t>(n);
      uint32_t* r1 = arena.get<uint32_t>(n);
      void* stmp = arena.alloc(sort_tmp_bytes(n));
      launch_pack(pp, n, k0, r0, st);
      int which = radix_sort(k0, r0, k1, r1, n, S.L.total + 1, stmp, st);  // +1: dead rows last
      uint64_t* ks = which ? k1 : k0;
      uint32_t* rs = which ? r1 : r0;
      float* ps = arena.get<float>(n);
      int32_t* fs = arena.get<int32_t>(n);
      launch_gather_f32(S.in.p.ptr(), rs, ps, n, st);
      launch_gather_i32(S.in.fid.ptr(), rs, fs, n, st);
      uint32_t* fl = arena.get<uint32_t>(n);
      uint32_t* pos = arena.get<uint32_t>(n);
      uint32_t* tot = arena.get<uint32_t>(1);
      launch_heads(ks, n, fl, st);
      exclusive_scan<uint32_t>(fl, pos, n, tot, arena.alloc(scan_tmp_bytes<uint32_t>(n)), st);
      kcheck("ingest");
      const int64_t nu = read_dev(tot);
      S.key.reserve(nu);
      S.p.reserve(nu);
      S.fid.reserve(nu);
      launch_edb_reduce(ks, ps, fs, pos, n, semi, S.key.ptr(), S.p.ptr(), S.fid.ptr(), st);
      kcheck("edb reduce");
      S.n = nu;
      arena.reset();
    }
    num_facts_db = next_fact;
    if (semi == S_MAXMULT) {
      fact_p.reserve(next_fact + 1);
      for (int r = 0; r < nr; ++r) {
        if (!prog.rels[r].input || rels[r]->in.n == 0) continue;
        RelState& S = *rels[r];
        // facts of one relation carry ids in push order: scatter p by id
        scatter_fact_p(S.in.fid.ptr(), S.in.p.ptr(), S.in.n);
      }
    }
  }

  void scatter_fact_p(const int32_t* fid, const float* p, int64_t n);

  // ------------------------------------------------------------------ index
  // Build (or alias) an index of relation r's version (key, p, n) with column
  // order `order`, prefix = sample + first nbound columns.
  void layout_index(Index& ix, const Layout& L, const std::vector<int>& order, int nbound) {
    ix.has_sample = L.has_sample;
    ix.sbits = L.sbits;
    ix.col_shift.assign(L.bits.size(), 0);
    ix.col_bits = L.bits;
    int pos = 0;
    for (int i = (int)order.size() - 1; i >= 0; --i) {
      ix.col_shift[order[i]] = pos;
      pos += L.bits[order[i]];
      if (i == nbound) ix.free_bits = pos;
    }
    if (nbound == (int)order.size()) ix.free_bits = 0;
    ix.sshift = pos;
    ix.prefix_bits = pos - ix.free_bits + ix.sbits;
  }

  static bool is_natural(const std::vector<int>& order) {
    for (size_t i = 0; i < order.size(); ++i)
      if (order[i] != (int)i) return false;
    return true;
  }

  // build into ix from a version's data; persistent=true uses ix.own_* buffers
  void build_index(Index& ix, const Layout& L, const std::vector<int>& order, int nbound, const uint64_t* key,
                   const float* p, int64_t n, bool persistent, bool want_offsets) {
    layout_index(ix, L, order, nbound);
    ix.n = n;
    if (is_natural(order)) {
      ix.key = key;
      ix.p = p;
    } else {
      std::vector<Move> mv;
      if (L.has_sample && L.sbits) mv.push_back({0, (uint8_t)L.sshift, (uint8_t)L.sbits, (uint8_t)ix.sshift});
      for (size_t c = 0; c < L.bits.size(); ++c)
        if (L.bits[c]) mv.push_back({0, (uint8_t)L.shift[c], (uint8_t)L.bits[c], (uint8_t)ix.col_shift[c]});
      uint64_t *k0, *k1;
      float *p0 = nullptr, *p1 = nullptr;
      if (persistent) {
        ix.own_key.bind(st); ix.tmp_key.bind(st); ix.own_p.bind(st); ix.tmp_p.bind(st);
        ix.own_key.reserve(n); ix.tmp_key.reserve(n);
        k0 = ix.own_key.ptr(); k1 = ix.tmp_key.ptr();
        if (p) { ix.own_p.reserve(n); ix.tmp_p.reserve(n); p0 = ix.own_p.ptr(); p1 = ix.tmp_p.ptr(); }
      } else {
        k0 = arena.get<uint64_t>(n); k1 = arena.get<uint64_t>(n);
        if (p) { p0 = arena.get<float>(n); p1 = arena.get<float>(n); }
      }
      launch_rekey(key, n, mv.data(), (int)mv.size(), k0, st);
      if (p) cuda_check(cudaMemcpyAsync(p0, p, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "index p");
      void* stmp = arena.alloc(sort_tmp_bytes(n));
      int which;
      if (p) which = radix_sort(k0, (uint32_t*)p0, k1, (uint32_t*)p1, n, L.total, stmp, st);
      else which = radix_sort<uint64_t, void>(k0, nullptr, k1, nullptr, n, L.total, stmp, st);
      ix.key = which ? k1 : k0;
      ix.p = p ? (which ? p1 : p0) : nullptr;
      kcheck("index build");
    }
    ix.offp = nullptr;
    if (want_offsets && ix.prefix_bits <= 26 && ((int64_t)1 << ix.prefix_bits) <= 4 * n + 4096) {
      ix.nprefix = (int64_t)1 << ix.prefix_bits;
      int64_t* off;
      if (persistent) {
        ix.off.bind(st);
        ix.rec.bind(st);
        ix.off.reserve(ix.nprefix + 1);
        off = ix.off.ptr();
      } else {
        off = arena.get<int64_t>(ix.nprefix + 1);
      }
      launch_build_offsets(ix.key, n, ix.free_bits, ix.nprefix, off, st);
      kcheck("offsets");
      ix.offp = off;
      if (persistent) {  // fan-out bound: selects the row-centric fused join
        unsigned long long* d = arena.get<unsigned long long>(1);
        cuda_check(cudaMemsetAsync(d, 0, 8, st), "memset");
        launch_max_degree(off, ix.nprefix, d, st);
        ix.maxdeg = (int64_t)read_dev(d);
        // fan-out <= 4 with index keys < 2^31: one 32-B record per prefix (keys + tags in one
        // sector) replaces the offsets -> keys -> tags loads of the fused join
        ix.recp = nullptr;
        if (ix.maxdeg <= 4 && ix.prefix_bits + ix.free_bits <= 31 && !getenv("LOBSTER_NO_REC")) {
          ix.rec.reserve(2 * ix.nprefix);
          launch_build_rec4(off, ix.key, ix.p, ix.nprefix, ix.rec.ptr(), st);
          kcheck("rec4");
          ix.recp = ix.rec.ptr();
        }
      }
    }
  }

  Index* static_index(int r, const std::vector<int>& order, int nbound) {
    auto key = std::make_pair(r, order);
    key.second.push_back(1000 + nbound);
    auto it = static_idx.find(key);
    if (it != static_idx.end()) return it->second.get();
    std::unique_ptr<Index> ix(new Index());
    RelState& S = *rels[r];
    ensure_sorted(S);
    build_index(*ix, S.L, order, nbound, S.key.ptr(), semi == S_UNIT ? nullptr : S.p.ptr(), S.n, true, true);
    Index* raw = ix.get();
    static_idx[key] = std::move(ix);
    return raw;
  }

  // ------------------------------------------------------------ rule eval
  struct VerData {
    const void* key;
    const float* p;
    int64_t n;
    bool k32;
  };
  VerData version_data(int rel, Version v) {
    RelState& S = *rels[rel];
    const bool tag = semi != S_UNIT;
    switch (v) {
      case V_DELTA:
        if (S.dense) return {S.dkey32.ptr(), tag ? S.dp.ptr() : nullptr, S.nd, true};
        return {S.dkey.ptr(), tag ? S.dp.ptr() : nullptr, S.nd, false};
      case V_OLD: return {S.okey.ptr(), tag ? S.op.ptr() : nullptr, S.no, false};
      default:
        ensure_sorted(S);
        return {S.key.ptr(), tag ? S.p.ptr() : nullptr, S.n, false};
    }
  }

  int32_t class_base(int cl) const { return (int32_t)class_min[cl]; }

  // atom k binds every variable of the rule: all other atoms are point lookups
  static bool covers_rule(const Rule& R, int k) {
    std::vector<char> b(R.var_names.size(), 0);
    for (auto& t : R.body[k].args)
      if (t.is_var()) b[t.var] = 1;
    for (char x : b)
      if (!x) return false;
    return true;
  }

  // Evaluate one rule (variant) and append its candidates to the head's buffer.
  void eval_rule(const Rule& R, const std::vector<Version>& ver, int start) {
    round_other++;  // moved to round_fused if this evaluation takes the fused direct join
    const int na = (int)R.body.size();
    const int nv = (int)R.var_names.size();
    RelState& H = *rels[R.head_rel];
    // join order: start atom, then most bound columns, natural prefix, size
    std::vector<int> order{start};
    std::vector<char> bound(nv, 0), used(na, 0);
    used[start] = 1;
    for (auto& t : R.body[start].args) if (t.is_var()) bound[t.var] = 1;
    for (int s = 1; s < na; ++s) {
      int best = -1;
      std::tuple<int, int, int64_t, int> bkey{};
      for (int a = 0; a < na; ++a) {
        if (used[a]) continue;
        int nb = 0;
        std::vector<char> isb;
        for (auto& t : R.body[a].args) {
          bool b = !t.is_var() || bound[t.var];
          isb.push_back(b);
          nb += b;
        }
        int natural = 1;
        for (int c = 0; c < (int)isb.size(); ++c) if ((c < nb) != (bool)isb[c]) natural = 0;
        int64_t sz = version_data(R.body[a].rel, ver[a]).n;
        auto k = std::make_tuple(nb, natural, -sz, -a);
        if (best < 0 || k > bkey) { best = a; bkey = k; }
      }
      order.push_back(best);
      used[best] = 1;
      for (auto& t : R.body[best].args) if (t.is_var()) bound[t.var] = 1;
    }
    // probe table = start atom
    Table T;
    const BodyAtom& A0 = R.body[start];
    const Layout& L0 = rels[A0.rel]->L;
    // a lazily compacted direct store probed by a lookup chain: probe its slot
    // words directly (slot index = packed key; absent slots are skipped)
    RelState& S0 = *rels[A0.rel];
    const bool dense_probe = S0.lazy && ver[start] == V_EXT && na >= 2 && covers_rule(R, start) && !force_slot_join;
    if (dense_probe && S0.n == 0) return;
    VerData d0 = dense_probe ? VerData{nullptr, nullptr, S0.nslots, true} : version_data(A0.rel, ver[start]);
    if (d0.n == 0) return;
    T.key = d0.key;
    T.k32 = d0.k32;
    T.n = d0.n;
    if (semi != S_UNIT) { T.tags.push_back(d0.p); T.tag_atom.push_back(start); }
    T.has_sample = L0.has_sample;
    T.sshift = L0.sshift;
    T.sbits = L0.sbits;
    T.vshift.assign(nv, -1);
    T.vbits.assign(nv, 0);
    std::vector<Cmp> pending_start;  // constants / repeated vars of the start atom
    for (int c = 0; c < (int)A0.args.size(); ++c) {
      const Term& t = A0.args[c];
      Operand f{0, (uint8_t)L0.shift[c], (uint8_t)L0.bits[c], L0.mins[c]};
      if (!t.is_var()) {
        Operand k{2, 0, 0, t.cst};
        pending_start.push_back({f, k, 0});
      } else if (T.vshift[t.var] >= 0) {
        Operand g{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], class_base(R.var_class[t.var])};
        pending_start.push_back({f, g, 0});
      } else {
        T.vshift[t.var] = L0.shift[c];
        T.vbits[t.var] = L0.bits[c];
      }
    }
    if (!T.has_sample) throw Failure(LOBSTER_E_STATE, "internal: join must start from a batched atom");
    std::vector<char> cmp_done(R.cmps.size(), 0);
    auto var_bound = [&](const Term& t, const std::vector<int>& vs) { return !t.is_var() || vs[t.var] >= 0; };

    if (na >= 2 && covers_rule(R, start) && !force_slot_join) {  // lookup chain
      LookupPlan lp{};
      lp.pkey = T.key;
      lp.pk32 = T.k32;
      lp.np = T.n;
      lp.ptag = semi != S_UNIT ? T.tags[0] : nullptr;
      if (dense_probe) lp.pdir = S0.dirf.get();
      std::vector<int> tag_atoms{start};
      for (int a = 0; a < na; ++a) {
        if (a == start) continue;
        const BodyAtom& A = R.body[a];
        const Layout& L = rels[A.rel]->L;
        std::vector<int> order(A.args.size());
        std::iota(order.begin(), order.end(), 0);
        Index* ix;
        Index local_ix;
        if (ver[a] == V_EXT) {
          ix = static_index(A.rel, order, (int)order.size());
        } else {
          VerData vd = version_data(A.rel, ver[a]);
          build_index(local_ix, L, order, (int)order.size(), (const uint64_t*)vd.key, vd.p, vd.n, false, true);
          ix = &local_ix;
        }
        if (ix->n == 0) return;
        if (lp.nlk >= MAXL) throw Failure(LOBSTER_E_PARSE, "too many lookup atoms in one rule");
        Lookup& K = lp.lk[lp.nlk++];
        if (L.has_sample && L.sbits) K.prem[K.nprem++] = Move{0, (uint8_t)T.sshift, (uint8_t)T.sbits, (uint8_t)ix->sshift};
        for (int c = 0; c < (int)A.args.size(); ++c) {
          const Term& t = A.args[c];
          if (!t.is_var()) {
            const int64_t f = (int64_t)t.cst - L.mins[c];
            if (f < 0 || f >= ((int64_t)1 << L.bits[c])) return;  // constant outside the domain: no match
            K.cprefix |= (uint64_t)f << ix->col_shift[c];
          } else if (L.bits[c]) {
            if (K.nprem >= MAXM) throw Failure(LOBSTER_E_PARSE, "lookup atom too wide");
            K.prem[K.nprem++] = Move{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], (uint8_t)ix->col_shift[c]};
          }
        }
        merge_moves(K.prem, K.nprem);
        K.bkey = ix->key;
        K.btag = semi != S_UNIT ? ix->p : nullptr;
        K.nb = ix->n;
        K.boff = ix->offp;
        K.nprefix = ix->nprefix;
        tag_atoms.push_back(a);
      }
      for (auto& c : pending_start) lp.cmp[lp.ncmp++] = c;
      for (size_t i = 0; i < R.cmps.size(); ++i) {
        auto op = [&](const Term& t) -> Operand {
          if (!t.is_var()) return Operand{2, 0, 0, t.cst};
          return Operand{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], class_base(R.var_class[t.var])};
        };
        if (lp.ncmp >= MAXC) throw Failure(LOBSTER_E_PARSE, "too many comparisons in one rule");
        lp.cmp[lp.ncmp++] = Cmp{op(R.cmps[i].a), op(R.cmps[i].b), R.cmps[i].rel};
      }
      head_moves(R, H, T, nullptr, lp.om, lp.nom, lp.cout);
      witness_moves(R, T, nullptr, lp.wm, lp.nwm, lp.wconst);
      merge_moves(lp.om, lp.nom);
      merge_moves(lp.wm, lp.nwm);
      lp.semi = semi;
      lp.omin = omin ? 1 : 0;
      if (semi != S_UNIT) {
        lp.ntag = na;
        for (int k = 0; k < na; ++k)
          for (size_t q = 0; q < tag_atoms.size(); ++q)
            if (tag_atoms[q] == k) lp.tag_order[k] = (int8_t)q;
      }
      if (H.direct) {
        direct_target(H, lp.direct, lp.fdir, lp.dirty, lp.aggregate, lp.mx);
      } else {
        reserve_candidates(H, H.nc + T.n);
        lp.ok32 = c32(H);
        lp.okey = cand_key(H);
        lp.oval32 = semi == S_MAXMIN || semi == S_ADDMULT ? H.cv32.ptr() + H.nc : nullptr;
        lp.oval64 = semi == S_MAXMULT ? H.cv64.ptr() + H.nc : nullptr;
      }
      {
        Phase ph(this, 0);
        launch_lookup_chain(lp, d_ncand, st);
        kcheck("lookup chain");
      }
      H.nc += T.n;  // live candidates are counted on the device (d_ncand)
      H.cand_bound += T.n;
      return;
    }

    if (na == 1) {  // projection
      ProjectPlan pp{};
      pp.key = T.key;
      pp.pk32 = T.k32;
      pp.ok32 = c32(H);
      pp.tag = semi != S_UNIT ? T.tags[0] : nullptr;
      pp.n = T.n;
      for (auto& c : pending_start) pp.cmp[pp.ncmp++] = c;
      for (size_t i = 0; i < R.cmps.size(); ++i) {
        const Compare& cm = R.cmps[i];
        if (cm.is_expr) continue;  // bytecode filters (below)
        auto op = [&](const Term& t) -> Operand {
          if (!t.is_var()) return Operand{2, 0, 0, t.cst};
          return Operand{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], class_base(R.var_class[t.var])};
        };
        if (pp.ncmp >= MAXC) throw Failure(LOBSTER_E_PARSE, "too many comparisons in one rule");
        pp.cmp[pp.ncmp++] = Cmp{op(cm.a), op(cm.b), cm.rel};
      }
      head_moves(R, H, T, nullptr, pp.om, pp.nom, pp.cout);
      // arithmetic (P:707-712 eval): head expressions and expression filters as bytecode
      for (size_t c = 0; c < R.head_expr.size(); ++c) {
        if (!R.head_expr[c].op) continue;
        if (pp.nbh >= MAXBH) throw Failure(LOBSTER_E_PARSE, "too many computed head columns in one rule");
        BcHead& b = pp.bh[pp.nbh++];
        compile_expr(R, R.head_expr[c], T, b.e);
        b.dshift = (uint8_t)H.L.shift[c];
        b.bits = (uint8_t)H.L.bits[c];
        b.base = H.L.mins[c];
      }
      for (const Compare& cm : R.cmps) {
        if (!cm.is_expr) continue;
        if (pp.nbf >= MAXBF) throw Failure(LOBSTER_E_PARSE, "too many expression comparisons in one rule");
        BcFilter& f = pp.bf[pp.nbf++];
        compile_expr(R, cm.ea, T, f.lhs);
        compile_expr(R, cm.eb, T, f.rhs);
        f.rel = cm.rel;
      }
      pp.semi = semi;
      witness_moves(R, T, nullptr, pp.wm, pp.nwm, pp.wconst);
      if (H.direct) {
        direct_target(H, pp.direct, pp.fdir, pp.dirty, pp.aggregate, pp.mx);
      } else {
        reserve_candidates(H, H.nc + T.n);
        pp.okey = cand_key(H);
        pp.oval32 = H.cv32.ptr() ? H.cv32.ptr() + H.nc : nullptr;
        pp.oval64 = H.cv64.ptr() ? H.cv64.ptr() + H.nc : nullptr;
      }
      merge_moves(pp.om, pp.nom);
      merge_moves(pp.wm, pp.nwm);
      launch_project(pp, st);
      kcheck("project");
      H.nc += T.n;
      H.cand_bound += T.n;
      stats.candidates += T.n;
      return;
    }

    for (int s = 1; s < na; ++s) {
      const int ai = order[s];
      const BodyAtom& A = R.body[ai];
      const Relation& AR = prog.rels[A.rel];
      RelState& AS = *rels[A.rel];
      const Layout& L = AS.L;
      // bound / free columns
      std::vector<int> bcols, fcols;
      for (int c = 0; c < (int)A.args.size(); ++c) {
        if (var_bound(A.args[c], T.vshift)) bcols.push_back(c); else fcols.push_back(c);
      }
      std::vector<int> iorder = bcols;
      iorder.insert(iorder.end(), fcols.begin(), fcols.end());
      const int nbound = (int)bcols.size();
      Index* ix;
      Index local_ix;
      if (ver[ai] == V_EXT) {
        ix = static_index(A.rel, iorder, nbound);
      } else {
        VerData vd = version_data(A.rel, ver[ai]);
        build_index(local_ix, L, iorder, nbound, (const uint64_t*)vd.key, vd.p, vd.n, false, true);
        ix = &local_ix;
      }
      if (ix->n == 0) return;
      JoinPlan jp{};
      jp.pkey = T.key;
      jp.pk32 = T.k32;
      jp.np = T.n;
      jp.npt = (int)T.tags.size();
      for (int k = 0; k < jp.npt; ++k) jp.ptag[k] = T.tags[k];
      // prefix moves (probe -> prefix coordinates)
      bool impossible = false;
      if (L.has_sample && L.sbits)
        jp.prem[jp.nprem++] = Move{0, (uint8_t)T.sshift, (uint8_t)T.sbits, (uint8_t)(ix->sshift - ix->free_bits)};
      for (int c : bcols) {
        const Term& t = A.args[c];
        const int dsh = ix->col_shift[c] - ix->free_bits;
        if (!t.is_var()) {
          int64_t f = (int64_t)t.cst - L.mins[c];
          if (f < 0 || f >= ((int64_t)1 << L.bits[c])) impossible = true;
          else jp.cprefix |= (uint64_t)f << dsh;
        } else if (L.bits[c]) {
          jp.prem[jp.nprem++] = Move{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], (uint8_t)dsh};
        }
      }
      if (impossible) return;
      jp.bkey = ix->key;
      jp.btag = semi != S_UNIT ? ix->p : nullptr;
      jp.nb = ix->n;
      jp.boff = ix->offp;
      jp.nprefix = ix->nprefix;
      jp.free_bits = ix->free_bits;
      // new variables from free columns; repeated free vars -> equality
      std::vector<int> nshift(nv, -1), nbits(nv, 0);  // build-side fields of new vars
      for (int c : fcols) {
        const Term& t = A.args[c];
        if (nshift[t.var] >= 0) {
          if (jp.nfeq >= 2) throw Failure(LOBSTER_E_PARSE, "too many repeated variables in one atom");
          jp.feq[jp.nfeq++] = Move{1, (uint8_t)ix->col_shift[c], (uint8_t)L.bits[c], (uint8_t)nshift[t.var]};
        } else {
          nshift[t.var] = ix->col_shift[c];
          nbits[t.var] = L.bits[c];
        }
      }
      // comparisons whose variables are all bound after this step
      auto operand = [&](const Term& t) -> Operand {
        if (!t.is_var()) return Operand{2, 0, 0, t.cst};
        if (T.vshift[t.var] >= 0)
          return Operand{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], class_base(R.var_class[t.var])};
        return Operand{1, (uint8_t)nshift[t.var], (uint8_t)nbits[t.var], class_base(R.var_class[t.var])};
      };
      auto avail = [&](const Term& t) { return !t.is_var() || T.vshift[t.var] >= 0 || nshift[t.var] >= 0; };
      if (s == 1)
        for (auto& c : pending_start) jp.cmp[jp.ncmp++] = c;
      for (size_t i = 0; i < R.cmps.size(); ++i) {
        if (cmp_done[i] || !avail(R.cmps[i].a) || !avail(R.cmps[i].b)) continue;
        if (jp.ncmp >= MAXC) throw Failure(LOBSTER_E_PARSE, "too many comparisons in one rule");
        jp.cmp[jp.ncmp++] = Cmp{operand(R.cmps[i].a), operand(R.cmps[i].b), R.cmps[i].rel};
        cmp_done[i] = 1;
      }
      jp.semi = semi;
      jp.omin = omin ? 1 : 0;
      jp.prefetch = fj_prefetch ? 1 : 0;
      const bool last = s == na - 1;
      jp.final_step = last ? 1 : 0;
      // fused row-centric join + direct ⊕: bounded fan-out, one probe tag
      if (last && H.direct && (H.L.total - H.L.sbits) > 8 && T.tags.size() <= 1 && na == 2 && ix->offp &&
          ix->maxdeg >= 0 && ix->maxdeg <= 8 && jp.nfeq == 0 && !force_slot_join) {
        head_moves(R, H, T, &nshift, jp.om, jp.nom, jp.cout, &nbits);
        witness_moves(R, T, &nshift, jp.wm, jp.nwm, jp.wconst, &nbits);
        if (semi != S_UNIT) {
          jp.ntag = 2;
          jp.tag_order[0] = (int8_t)(start < ai ? 0 : 1);
          jp.tag_order[1] = (int8_t)(start < ai ? 1 : 0);
        }
        direct_target(H, jp.direct, jp.fdir, jp.dirty, jp.aggregate, jp.mx);
        if (rels[A0.rel]->async) jp.np_dev = rels[A0.rel]->ndev.ptr();
        if (ix->maxdeg <= 4 && jp.pk32) jp.brec = ix->recp;
        merge_moves(jp.prem, jp.nprem);
        merge_moves(jp.om, jp.nom);
        merge_moves(jp.wm, jp.nwm);
        // every join_timing_every-th launch is timed with a CUDA event pair (its candidates
        // count into d_ncand[2]): each event pair costs ~4 µs of issue / GPU bubble, ~2.5 ms
        // per C2 step if every launch were timed
        const bool timed = (fj_seq++ % join_timing_every) == 0;
        {
          Phase ph(this, 5, timed);
          // async: Δ size unknown here; grid from the last size the host saw (any grid is
          // correct: the kernel strides over the device-side count)
          launch_join_rows_direct(jp, (int)ix->maxdeg, d_ncand + (timed ? 2 : 1), st,
                                  jp.np_dev ? 8 * async_nd0 + 1 : jp.np);
          kcheck("join rows direct");
        }
        stats.fj_launches++;
        if (timed) stats.fj_timed_launches++;
        round_other--;
        round_fused++;
        if (!H.async) {
          stats.fj_probe_rows += T.n;
          if (timed) stats.fj_timed_probe_rows += T.n;
        } else if (timed) {
          timed_rounds.insert(cur_round);  // its probe rows are learnt when the previous round drains
        }
        H.nc += T.n;  // candidates counted on the device (d_ncand[1])
        H.cand_bound += T.n * ix->maxdeg;
        return;
      }
      // count + scan (A3-A4)
      int64_t* count = arena.get<int64_t>(T.n);
      int64_t* start_ = arena.get<int64_t>(T.n);
      int64_t* offs = arena.get<int64_t>(T.n);
      int64_t* tot = arena.get<int64_t>(1);
      {
        Phase ph(this, 0);
        merge_moves(jp.prem, jp.nprem);
        launch_join_count(jp, count, start_, st);
        exclusive_scan<int64_t>(count, offs, T.n, tot, arena.alloc(scan_tmp_bytes<int64_t>(T.n)), st);
        kcheck("join count");
      }
      const int64_t total = read_dev(tot);
      if (total == 0) return;
      Table N;  // next probe table (intermediate)
      if (last) {
        Table view = T;
        head_moves(R, H, T, &nshift, jp.om, jp.nom, jp.cout, &nbits);
        witness_moves(R, T, &nshift, jp.wm, jp.nwm, jp.wconst, &nbits);
        // ⊗ order: T = [probe tags..., build tag]
        if (semi != S_UNIT) {
          jp.ntag = na;
          for (int k = 0; k < na; ++k) {
            int idx = -1;
            for (size_t q = 0; q < T.tag_atom.size(); ++q) if (T.tag_atom[q] == k) idx = (int)q;
            if (k == ai) idx = jp.npt;
            jp.tag_order[k] = (int8_t)idx;
          }
        }
        if (H.direct) {
          direct_target(H, jp.direct, jp.fdir, jp.dirty, jp.aggregate, jp.mx);
        } else {
          reserve_candidates(H, H.nc + total);
          jp.ok32 = c32(H);
          jp.okey = cand_key(H);
          jp.oval32 = semi == S_MAXMIN || semi == S_ADDMULT ? H.cv32.ptr() + H.nc : nullptr;
          jp.oval64 = semi == S_MAXMULT ? H.cv64.ptr() + H.nc : nullptr;
        }
      } else {
        // intermediate layout: sample + all bound vars (var id order)
        N.has_sample = true;
        N.vshift.assign(nv, -1);
        N.vbits.assign(nv, 0);
        int pos = 0;
        for (int v = nv - 1; v >= 0; --v) {
          int b = T.vshift[v] >= 0 ? T.vbits[v] : (nshift[v] >= 0 ? nbits[v] : -1);
          if (b < 0) continue;
          N.vshift[v] = pos;
          N.vbits[v] = b;
          pos += b;
        }
        N.sshift = pos;
        N.sbits = T.sbits;
        if (pos + N.sbits > 63) throw Failure(LOBSTER_E_RANGE, "intermediate join key wider than 63 bits");
        if (T.sbits) jp.om[jp.nom++] = Move{0, (uint8_t)T.sshift, (uint8_t)T.sbits, (uint8_t)N.sshift};
        for (int v = 0; v < nv; ++v) {
          if (N.vshift[v] < 0 || N.vbits[v] == 0) continue;
          if (jp.nom >= MAXM) throw Failure(LOBSTER_E_PARSE, "too many variables in one rule");
          if (T.vshift[v] >= 0) jp.om[jp.nom++] = Move{0, (uint8_t)T.vshift[v], (uint8_t)T.vbits[v], (uint8_t)N.vshift[v]};
          else jp.om[jp.nom++] = Move{1, (uint8_t)nshift[v], (uint8_t)nbits[v], (uint8_t)N.vshift[v]};
        }
        N.key = arena.get<uint64_t>(total);
        N.k32 = false;
        N.n = total;
        jp.okey = const_cast<void*>(N.key);
        jp.ok32 = 0;
        if (semi != S_UNIT) {
          for (int k = 0; k <= jp.npt; ++k) {
            float* t = arena.get<float>(total);
            jp.otag[k] = t;
            N.tags.push_back(t);
          }
          N.tag_atom = T.tag_atom;
          N.tag_atom.push_back(ai);
        }
      }
      {
        Phase ph(this, 0);
        merge_moves(jp.om, jp.nom);
        merge_moves(jp.wm, jp.nwm);
        launch_join_write(jp, offs, start_, total, arena.get<int64_t>(join_write_tiles(total) + 1), st);
        kcheck("join write");
      }
      if (last) {
        H.nc += total;
        H.cand_bound += total;
        stats.candidates += total;
      } else {
        T = N;
      }
      (void)AR;
    }
  }

  // head key moves (src 0 = probe table T, src 1 = build fields given by nshift)
  // postfix bytecode of an expression over the probe key's variable fields
  void compile_expr(const Rule& R, const Expr& e, const Table& T, Bc& out) {
    out.n = 0;
    std::function<void(const Expr&)> emit = [&](const Expr& x) {
      if (out.n >= MAXBC) throw Failure(LOBSTER_E_PARSE, "expression too long (more than 16 operations)");
      for (auto& k : x.kids) emit(k);
      BcIns& i = out.ins[out.n++];
      i = BcIns{};
      switch (x.op) {
        case '#': i.op = BC_CONST; i.v = x.cst; break;
        case 'v':
          i.op = BC_FIELD;
          i.shift = (uint8_t)T.vshift[x.var];
          i.bits = (uint8_t)T.vbits[x.var];
          i.v = class_base(R.var_class[x.var]);
          break;
        case '+': i.op = BC_ADD; break;
        case '-': i.op = BC_SUB; break;
        case '*': i.op = BC_MUL; break;
        case '/': i.op = BC_DIV; break;
        case '%': i.op = BC_MOD; break;
        default: i.op = BC_NEG; break;
      }
    };
    emit(e);
  }

  void head_moves(const Rule& R, RelState& H, const Table& T, const std::vector<int>* nshift, Move* om, int& nom,
                  uint64_t& cout, const std::vector<int>* nbits = nullptr) {
    const Layout& HL = H.L;
    nom = 0;
    cout = 0;
    if (HL.has_sample && HL.sbits) om[nom++] = Move{0, (uint8_t)T.sshift, (uint8_t)T.sbits, (uint8_t)HL.sshift};
    for (size_t c = 0; c < R.head.size(); ++c) {
      const Term& t = R.head[c];
      if (c < R.head_expr.size() && R.head_expr[c].op) continue;  // computed by bytecode (project_k)
      if (!t.is_var()) {
        cout |= (uint64_t)((int64_t)t.cst - HL.mins[c]) << HL.shift[c];
        continue;
      }
      if (HL.bits[c] == 0) continue;
      if (nom >= MAXM) throw Failure(LOBSTER_E_PARSE, "head too wide");
      if (T.vshift[t.var] >= 0) om[nom++] = Move{0, (uint8_t)T.vshift[t.var], (uint8_t)T.vbits[t.var], (uint8_t)HL.shift[c]};
      else om[nom++] = Move{1, (uint8_t)(*nshift)[t.var], (uint8_t)(*nbits)[t.var], (uint8_t)HL.shift[c]};
    }
  }

  void witness_moves(const Rule& R, const Table& T, const std::vector<int>* nshift, Move* wm, int& nwm,
                     uint32_t& wconst, const std::vector<int>* nbits = nullptr) {
    nwm = 0;
    wconst = 0;
    if (semi != S_MAXMULT) return;
    const int rb = rule_bits[R.head_rel];
    // direct max-mult heads store the compressed witness (rule index just above
    // the variable fields, kernels.cuh MxEnc); other stores the 32-bit layout
    const RelState& H = *rels[R.head_rel];
    if (rb) wconst = (uint32_t)R.local_index << (H.direct ? H.wT : 32 - rb);
    const size_t ri = (size_t)R.global_index;
    for (size_t i = 0; i < R.nonhead.size(); ++i) {
      const int v = R.nonhead[i];
      if (wbits[ri][i] == 0) continue;
      if (nwm >= MAXM) throw Failure(LOBSTER_E_PARSE, "too many non-head variables");
      if (T.vshift[v] >= 0) wm[nwm++] = Move{0, (uint8_t)T.vshift[v], (uint8_t)T.vbits[v], (uint8_t)wshift[ri][i]};
      else wm[nwm++] = Move{1, (uint8_t)(*nshift)[v], (uint8_t)(*nbits)[v], (uint8_t)wshift[ri][i]};
    }
  }

  // u32 candidate keys whenever the head's packed key fits 31 bits (dense stores
  // always): the dead key ~0 still sorts last, and sorts move 4 B less per key
  bool c32(const RelState& H) const { return H.dense || (H.L.total <= 31 && !top1 && !getenv("LOBSTER_C64")); }

  void* cand_key(RelState& H) {
    return c32(H) ? (void*)(H.ckey32.ptr() + H.nc) : (void*)(H.ckey.ptr() + H.nc);
  }

  void reserve_candidates(RelState& H, int64_t n) {
    if (c32(H)) H.ckey32.reserve(n, H.nc);
    else H.ckey.reserve(n, H.nc);
    if (semi == S_MAXMIN || semi == S_ADDMULT) H.cv32.reserve(n, H.nc);
    if (semi == S_MAXMULT) H.cv64.reserve(n, H.nc);
  }

  // -------------------------------------------------- per-relation epilogue
  // Dense store: u32 keys; sort + segmented ⊕ (A6-A7), then one in-place
  // classify/apply pass over U against the direct-mapped F and a compaction
  // of Δ' (A8) — O(|C|) per round, no O(|F|) merge.
  int64_t settle_dense(RelState& S) {
    const int64_t nc = S.nc;
    S.nc = 0;
    if (nc == 0) { S.nd = 0; return 0; }
    const int tb = S.L.total + 1;  // +1 bit: dead key (all ones) sorts last
    S.ckey32b.reserve(nc);
    uint32_t* ks;
    const void* vs;
    {
      Phase ph(this, 1);
      void* stmp = arena.alloc(sort_tmp_bytes(nc));
      int which;
      if (semi == S_MAXMULT) {
        S.cv64b.reserve(nc);
        which = radix_sort(S.ckey32.ptr(), S.cv64.ptr(), S.ckey32b.ptr(), S.cv64b.ptr(), nc, tb, stmp, st);
        vs = which ? S.cv64b.ptr() : S.cv64.ptr();
      } else if (semi == S_UNIT) {
        which = radix_sort<uint32_t, void>(S.ckey32.ptr(), nullptr, S.ckey32b.ptr(), nullptr, nc, tb, stmp, st);
        vs = nullptr;
      } else {
        S.cv32b.reserve(nc);
        which = radix_sort(S.ckey32.ptr(), S.cv32.ptr(), S.ckey32b.ptr(), S.cv32b.ptr(), nc, tb, stmp, st);
        vs = which ? S.cv32b.ptr() : S.cv32.ptr();
      }
      ks = which ? S.ckey32b.ptr() : S.ckey32.ptr();
      kcheck("sort");
    }
    uint32_t* fl = arena.get<uint32_t>(nc);
    uint32_t* pos = arena.get<uint32_t>(nc);
    uint32_t* tot = arena.get<uint32_t>(1);
    {
      Phase ph(this, 2);
      launch_heads(ks, nc, fl, st);
      exclusive_scan<uint32_t>(fl, pos, nc, tot, arena.alloc(scan_tmp_bytes<uint32_t>(nc)), st);
      kcheck("heads");
    }
    const int64_t nu = read_dev(tot);
    uint32_t* ukey = arena.get<uint32_t>(nu);
    float* up = semi != S_UNIT ? arena.get<float>(nu) : nullptr;
    uint32_t* uw = semi == S_MAXMULT ? arena.get<uint32_t>(nu) : nullptr;
    {
      Phase ph(this, 2);
      launch_seg_reduce(ks, vs, pos, nc, nu, semi, ukey, up, uw, arena.get<uint32_t>(2 * nu + 2), st);
      kcheck("seg reduce");
    }
    uint64_t* flags = arena.get<uint64_t>(nu);
    uint64_t* offs = arena.get<uint64_t>(nu);
    uint64_t* t2 = arena.get<uint64_t>(1);
    {
      Phase ph(this, 3);
      launch_dense_diff(ukey, up, uw, nu, semi, S.dfp.ptr(), S.dfw.ptr(), S.dfbits.ptr(), flags, st);
      exclusive_scan<uint64_t>(flags, offs, nu, t2, arena.alloc(scan_tmp_bytes<uint64_t>(nu)), st);
      kcheck("dense diff");
    }
    const uint64_t tt = read_dev(t2);
    const int64_t nd = (int64_t)(tt & 0xffffffffull), nnew = (int64_t)(tt >> 32);
    stats.bytes_algorithmic += bytes_round(nc, nu, nd);
    S.n += nnew;
    S.nd = nd;
    if (nd == 0) return 0;
    Phase ph(this, 3);
    S.dkey32.reserve(nd);
    if (semi != S_UNIT) S.dp.reserve(nd);
    if (semi == S_MAXMULT) S.dw.reserve(nd);
    launch_dense_delta(ukey, up, uw, nu, flags, offs, semi, S.dkey32.ptr(), semi != S_UNIT ? S.dp.ptr() : nullptr,
                       semi == S_MAXMULT ? S.dw.ptr() : nullptr, st);
    kcheck("dense delta");
    return nd;
  }

  void ensure_sorted(RelState& S) {
    if (!S.lazy) return;
    S.lazy = false;
    dense_to_sorted(S);
  }

  // dense F -> sorted list (key, p, w) for later strata, outputs and the walk
  void dense_to_sorted(RelState& S, int64_t known_n = -1) {
    const int64_t ns = S.nslots;
    uint32_t* fl = arena.get<uint32_t>(ns);
    uint32_t* pos = arena.get<uint32_t>(ns);
    uint32_t* tot = arena.get<uint32_t>(1);
    if (S.direct) launch_direct_present(S.dirf.get(), ns, semi, fl, st);
    else launch_dense_present(S.dfp.ptr(), S.dfbits.ptr(), ns, semi, fl, st);
    exclusive_scan<uint32_t>(fl, pos, ns, tot, arena.alloc(scan_tmp_bytes<uint32_t>(ns)), st);
    kcheck("dense present");
    const int64_t n = known_n >= 0 ? known_n : (int64_t)read_dev(tot);  // (the tile kernel counts its tuples)
    S.key.reserve(n);
    if (semi != S_UNIT) S.p.reserve(n);
    if (semi == S_MAXMULT) S.w.reserve(n);
    if (S.direct)
      launch_direct_compact(S.dirf.get(), pos, ns, semi, S.key.ptr(), semi != S_UNIT ? S.p.ptr() : nullptr,
                            semi == S_MAXMULT ? S.w.ptr() : nullptr, mx_wmask(S), S.wT, S.wrb, st);
    else
      launch_dense_compact(S.dfp.ptr(), S.dfw.ptr(), S.dfbits.ptr(), pos, ns, semi, S.key.ptr(),
                           semi != S_UNIT ? S.p.ptr() : nullptr, semi == S_MAXMULT ? S.w.ptr() : nullptr, st);
    kcheck("dense compact");
    S.n = n;
  }

  // Store choice for a local relation: direct-mapped
  // when its packed key fits 30 bits, it is only ever probed through Δ (no
  // B^new / B^old index is needed) and the slot array fits half of free HBM.
  // direct ⊕ target for `n` more candidates of head H this round: dlist must
  // hold every slot improved so far (<= candidates so far) plus n.
  void direct_target(RelState& H, int& direct, void*& f, uint32_t*& dirty, int& aggregate, MxEnc& mx) {
    direct = 1;
    aggregate = (H.L.total - H.L.sbits) <= 8 ? 1 : 0;  // narrow head: many candidates per slot
    f = H.dirf.get();
    dirty = H.dirty.ptr();
    mx.wmask = mx_wmask(H);
    mx.stamp = H.stamp_mode ? (H.smax - (unsigned long long)cur_round) << H.wWB : 0ull;
  }

  static unsigned long long mx_wmask(const RelState& S) { return S.wWB >= 64 ? ~0ull : (1ull << S.wWB) - 1ull; }

  // max-mult direct word layout of head relation r: widest variable field of its
  // rules (wT), rule-index bits (wrb); stamps when 2^(34 - WB) - 1 exceeds max_iters
  void mx_layout(int r, RelState& S) {
    S.wT = 0;
    for (const Rule& R : prog.rules) {
      if (R.head_rel != r) continue;
      int tot = 0;
      for (int b : wbits[(size_t)R.global_index]) tot += b;
      S.wT = std::max(S.wT, tot);
    }
    S.wrb = rule_bits[r];
    S.wWB = S.wT + S.wrb;
    const int sb = 34 - S.wWB;
    S.smax = (1ull << sb) - 1ull;
    S.stamp_mode = !getenv("LOBSTER_NO_STAMPS") && S.smax > (unsigned long long)max_iters + 1;
  }

  void choose_store(RelState& S, int r) {
    S.dense = false;
    S.direct = false;
    S.lazy = false;
    if (S.build_local || S.L.total > 30 || force_sorted || top1 || xfer) return;
    if (semi != S_ADDMULT && !force_sort_dedup) {  // idempotent ⊕: fused direct store
      const int64_t ns = (int64_t)1 << S.L.total;
      const size_t bytes = semi == S_UNIT ? (size_t)((ns + 31) / 32) * 4 : (size_t)ns * (semi == S_MAXMULT ? 8 : 4);
      if (S.dirf.capacity() < bytes) {  // cudaMemGetInfo costs 0.2-11 ms: only when a new slot array is needed
        size_t fr = 0, tot = 0;
        HostTimer hm(host_ms[6]);
        cudaMemGetInfo(&fr, &tot);
        if ((double)bytes > 0.5 * (double)fr) return;
      }
      S.dense = S.direct = true;
      S.nslots = ns;
      if (semi == S_MAXMULT) mx_layout(r, S);
      S.dirf.reserve(bytes);
      launch_direct_fill(S.dirf.get(), ns, semi, st);
      S.dirty.reserve((ns + 31) / 32);
      S.ndev.reserve(1);
      S.dctr.reserve(1);
      if (S.ectr.bytes() < 8) {
        S.ectr.reserve(2);
        cuda_check(cudaMemsetAsync(S.ectr.ptr(), 0, 8, st), "memset");
      }
      cuda_check(cudaMemsetAsync(S.dctr.ptr(), 0, 8, st), "memset");
      S.cand_bound = 0;
      cuda_check(cudaMemsetAsync(S.dirty.ptr(), 0, (size_t)((ns + 31) / 32) * 4, st), "memset");
      return;
    }
    const int64_t ns = (int64_t)1 << S.L.total;
    const double bytes = semi == S_UNIT ? ns / 8.0 : (double)ns * (semi == S_MAXMULT ? 8 : 4);
    if ((double)S.dfp.bytes() < bytes) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      if (bytes > 0.5 * (double)fr) return;
    }
    S.dense = true;
    S.nslots = ns;
    if (semi == S_UNIT) {
      S.dfbits.reserve((ns + 31) / 32);
    } else {
      S.dfp.reserve(ns);
      if (semi == S_MAXMULT) S.dfw.reserve(ns);
    }
    launch_dense_fill(S.dfp.ptr(), S.dfbits.ptr(), ns, semi, st);
    kcheck("dense fill");
  }

  // Sorted store: sort + segmented ⊕ (A6-A7), diff + apply + merge (A8); returns |Δ'|
  // Direct store: the join already ⊕-ed every candidate into F; Δ' = the
  // improved slots with their round-final tags (re-settled for the next round).
  int64_t settle_direct(RelState& S) {
    const int64_t nc = S.nc;
    S.nc = 0;
    if (nc == 0 && !S.async) { S.nd = 0; return 0; }
    const int64_t nw = (S.nslots + 31) / 32;
    const int64_t cap = S.async ? S.nslots : std::min<int64_t>(std::max<int64_t>(S.cand_bound, 1), S.nslots);
    S.cand_bound = 0;
    S.dkey32.reserve(cap);
    if (semi != S_UNIT) S.dp.reserve(cap);
    {  // Δ' in slot order (two launches); dirty bits cleared, slots re-settled.  Joins read
       // Δ keys and p only (a candidate's witness comes from its own body), so no Δ' witness.
      Phase ph(this, 3, !S.async || log_level >= 2);  // per-round trace keeps them
      launch_direct_extract2(S.dirf.get(), S.dirty.ptr(), nw, semi, S.dkey32.ptr(),
                             semi != S_UNIT ? S.dp.ptr() : nullptr, nullptr,
                             sorted_delta ? arena.get<uint32_t>(direct_extract2_scratch(nw)) : nullptr, S.ndev.ptr(),
                             semi == S_MAXMULT && !S.stamp_mode ? S.smax << S.wWB : 0ull, mx_wmask(S),
                             S.async ? S.ring_dst : nullptr, S.ring_seq, sorted_delta ? nullptr : S.ectr.ptr(), st);
      kcheck("direct extract");
    }
    if (S.async) {  // |Δ'| stays on the device: the next join reads it, the host polls it later
      S.nd = S.nslots;
      return -1;
    }
    const int64_t nd = (int64_t)read_dev(S.ndev.ptr());
    stats.bytes_algorithmic += bytes_round_direct(nc, nd);
    S.nd = nd;
    return nd;
  }

  int64_t bytes_round_direct(int64_t nc, int64_t nd) const {
    // probe read is counted by the caller's Δ (|Δ| r_Δ of the previous round's Δ'):
    // one slot read-modify-write per candidate + Δ' write + Δ re-read next round
    const int64_t slot = semi == S_MAXMULT ? 8 : 4;
    const int64_t rD = 4 + (semi == S_UNIT ? 0 : (semi == S_MAXMULT ? 8 : 4));
    return nc * slot + nd * (slot + 2 * rD);
  }

  int64_t settle(int r) {
    RelState& S = *rels[r];
    if (S.direct) return settle_direct(S);
    if (S.need_old) {  // OLD = F before this round's update (B^old of the next round)
      S.okey.reserve(S.n);
      if (S.n) cuda_check(cudaMemcpyAsync(S.okey.ptr(), S.key.ptr(), S.n * 8, cudaMemcpyDeviceToDevice, st), "old");
      if (semi != S_UNIT) {
        S.op.reserve(S.n);
        if (S.n) cuda_check(cudaMemcpyAsync(S.op.ptr(), S.p.ptr(), S.n * 4, cudaMemcpyDeviceToDevice, st), "old");
      }
      S.no = S.n;
    }
    if (S.dense) return settle_dense(S);
    if (xfer) S.nc = part_exchange(S, S.nc);  // collective: every rank, every relation, every round
    const int64_t nc = S.nc;
    S.nc = 0;
    if (nc == 0) { S.nd = 0; return 0; }
    if (top1) top1_candidates(r, S, nc);
    const int tb = S.L.total + 1;  // +1 bit: KEY_DEAD sorts after every key
    if (c32(S)) return settle_sorted32(S, nc, tb);
    S.ckey2.reserve(nc);
    uint64_t* ks;
    const void* vs;
    {
      Phase ph(this, 1);
      void* stmp = arena.alloc(sort_tmp_bytes(nc));
      int which;
      if (semi == S_MAXMULT) {
        S.cv64b.reserve(nc);
        which = radix_sort(S.ckey.ptr(), S.cv64.ptr(), S.ckey2.ptr(), S.cv64b.ptr(), nc, tb, stmp, st);
        vs = which ? S.cv64b.ptr() : S.cv64.ptr();
      } else if (semi == S_UNIT) {
        which = radix_sort<uint64_t, void>(S.ckey.ptr(), nullptr, S.ckey2.ptr(), nullptr, nc, tb, stmp, st);
        vs = nullptr;
      } else {
        S.cv32b.reserve(nc);
        which = radix_sort(S.ckey.ptr(), S.cv32.ptr(), S.ckey2.ptr(), S.cv32b.ptr(), nc, tb, stmp, st);
        vs = which ? S.cv32b.ptr() : S.cv32.ptr();
      }
      ks = which ? S.ckey2.ptr() : S.ckey.ptr();
      kcheck("sort");
    }
    uint32_t* fl = arena.get<uint32_t>(nc);
    uint32_t* pos = arena.get<uint32_t>(nc);
    uint32_t* tot = arena.get<uint32_t>(1);
    {
      Phase ph(this, 2);
      launch_heads(ks, nc, fl, st);
      exclusive_scan<uint32_t>(fl, pos, nc, tot, arena.alloc(scan_tmp_bytes<uint32_t>(nc)), st);
      kcheck("heads");
    }
    const int64_t nu = read_dev(tot);
    uint64_t* ukey = arena.get<uint64_t>(nu);
    float* up = semi != S_UNIT ? arena.get<float>(nu) : nullptr;
    uint32_t* uw = semi == S_MAXMULT ? arena.get<uint32_t>(nu) : nullptr;
    {
      Phase ph(this, 2);
      launch_seg_reduce(ks, vs, pos, nc, nu, semi, ukey, up, uw, arena.get<uint32_t>(2 * nu + 2), st);
      kcheck("seg reduce");
    }
    return merge_unique(S, ukey, up, uw, nu, nc);
  }

  // Sorted store with u32 candidates: u32 radix sort + segmented ⊕, then the
  // unique keys widen to u64 for the diff / apply / merge against F.
  int64_t settle_sorted32(RelState& S, int64_t nc, int tb) {
    S.ckey32b.reserve(nc);
    uint32_t* ks;
    const void* vs;
    {
      Phase ph(this, 1);
      void* stmp = arena.alloc(sort_tmp_bytes(nc));
      int which;
      if (semi == S_MAXMULT) {
        S.cv64b.reserve(nc);
        which = radix_sort(S.ckey32.ptr(), S.cv64.ptr(), S.ckey32b.ptr(), S.cv64b.ptr(), nc, tb, stmp, st);
        vs = which ? S.cv64b.ptr() : S.cv64.ptr();
      } else if (semi == S_UNIT) {
        which = radix_sort<uint32_t, void>(S.ckey32.ptr(), nullptr, S.ckey32b.ptr(), nullptr, nc, tb, stmp, st);
        vs = nullptr;
      } else {
        S.cv32b.reserve(nc);
        which = radix_sort(S.ckey32.ptr(), S.cv32.ptr(), S.ckey32b.ptr(), S.cv32b.ptr(), nc, tb, stmp, st);
        vs = which ? S.cv32b.ptr() : S.cv32.ptr();
      }
      ks = which ? S.ckey32b.ptr() : S.ckey32.ptr();
      kcheck("sort");
    }
    uint32_t* fl = arena.get<uint32_t>(nc);
    uint32_t* pos = arena.get<uint32_t>(nc);
    uint32_t* tot = arena.get<uint32_t>(1);
    {
      Phase ph(this, 2);
      launch_heads(ks, nc, fl, st);
      exclusive_scan<uint32_t>(fl, pos, nc, tot, arena.alloc(scan_tmp_bytes<uint32_t>(nc)), st);
      kcheck("heads");
    }
    const int64_t nu = read_dev(tot);
    uint32_t* ukey32 = arena.get<uint32_t>(nu);
    uint64_t* ukey = arena.get<uint64_t>(nu);
    float* up = semi != S_UNIT ? arena.get<float>(nu) : nullptr;
    uint32_t* uw = semi == S_MAXMULT ? arena.get<uint32_t>(nu) : nullptr;
    {
      Phase ph(this, 2);
      launch_seg_reduce(ks, vs, pos, nc, nu, semi, ukey32, up, uw, arena.get<uint32_t>(2 * nu + 2), st);
      launch_widen_u32(ukey32, nu, ukey, st);
      kcheck("seg reduce");
    }
    return merge_unique(S, ukey, up, uw, nu, nc);
  }

  // A8 for the sorted store: classify U against F, write Δ' and apply in place,
  // merge the new tuples (U sorted, unique, u64 keys)
  int64_t merge_unique(RelState& S, const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu,
                       int64_t nc) {
    uint64_t* flags = arena.get<uint64_t>(nu);
    uint64_t* offs = arena.get<uint64_t>(nu);
    int64_t* fpos = arena.get<int64_t>(nu);
    uint64_t* t2 = arena.get<uint64_t>(1);
    {
      Phase ph(this, 3);
      launch_diff(ukey, up, uw, nu, S.key.ptr(), semi != S_UNIT ? S.p.ptr() : nullptr, S.n, semi, flags, fpos, st);
      exclusive_scan<uint64_t>(flags, offs, nu, t2, arena.alloc(scan_tmp_bytes<uint64_t>(nu)), st);
      kcheck("diff");
    }
    const uint64_t tt = read_dev(t2);
    const int64_t nd = (int64_t)(tt & 0xffffffffull), nnew = (int64_t)(tt >> 32);
    stats.bytes_algorithmic += bytes_round(nc, nu, nd);
    S.nd = nd;
    if (nd == 0) return 0;
    Phase ph(this, 3);
    S.dkey.reserve(nd);
    if (semi != S_UNIT) S.dp.reserve(nd);
    if (semi == S_MAXMULT) S.dw.reserve(nd);
    uint64_t* nkey = arena.get<uint64_t>(nnew);
    float* np_ = semi != S_UNIT ? arena.get<float>(nnew) : nullptr;
    uint32_t* nw = semi == S_MAXMULT ? arena.get<uint32_t>(nnew) : nullptr;
    launch_apply(ukey, up, uw, nu, flags, offs, fpos, semi, semi != S_UNIT ? S.p.ptr() : nullptr,
                 semi == S_MAXMULT ? S.w.ptr() : nullptr, S.dkey.ptr(), semi != S_UNIT ? S.dp.ptr() : nullptr,
                 semi == S_MAXMULT ? S.dw.ptr() : nullptr, nkey, np_, nw, st);
    kcheck("apply");
    if (nnew > 0) {
      const int64_t nn = S.n + nnew;
      S.key2.reserve(nn);
      if (semi != S_UNIT) S.p2.reserve(nn);
      if (semi == S_MAXMULT) S.w2.reserve(nn);
      launch_merge(S.key.ptr(), semi != S_UNIT ? S.p.ptr() : nullptr, semi == S_MAXMULT ? S.w.ptr() : nullptr, S.n,
                   nkey, np_, nw, nnew, S.key2.ptr(), semi != S_UNIT ? S.p2.ptr() : nullptr,
                   semi == S_MAXMULT ? S.w2.ptr() : nullptr, st);
      kcheck("merge");
      S.key.swap(S.key2);
      S.p.swap(S.p2);
      S.w.swap(S.w2);
      S.n = nn;
    }
    return nd;
  }

  int64_t bytes_round(int64_t nc, int64_t nu, int64_t nd) const {
    const int64_t rt = semi == S_UNIT ? 0 : (semi == S_MAXMULT ? 8 : 4);
    const int64_t rC = 8 + rt, rF = 8 + rt;
    return 2 * nc * rC + nu * rF + nd * 2 * rF;
  }

  // ------------------------------------------------------------------- run
  void run(lobster_run_stats* out) {
    if (!loaded) throw Failure(LOBSTER_E_STATE, "run before program_load");
    if (sticky) throw Failure(LOBSTER_E_CUDA, "context is in a failed state");
    stats = lobster_run_stats{};
    if (!d_ncand) cuda_check(cudaMalloc(&d_ncand, 24), "cudaMalloc");
    cuda_check(cudaMemsetAsync(d_ncand, 0, 24, st), "memset");
    fj_seq = 0;
    ev.clear();
    ev_used = 0;
    marks.clear();
    sections.clear();
    cudaEvent_t t0 = get_event();
    cudaEventRecord(t0, st);
    mark("start");
    for (auto& r : rels) {
      r->out_dev_ready = r->out_host_ready = false;
      r->has_grad = false;
    }
    static_idx.clear();
    arena.reset();
    for (double& h : host_ms) h = 0.0;
    {
      HostTimer ht(host_ms[0]);
      ingest_domains();
    }
    mark("domains");
    // Micro-batching (SURVEY §5 memory planner): samples are independent
    // databases, so the fixpoint runs over sample ranges whose
    // packed keys fit the direct-mapped store; `output` relations are
    // collected across ranges.
    const int32_t B = opt.batch_size;
    const int32_t mb = choose_micro_batch();
    micro = mb < B;
    for (auto& r : rels) {
      r->retained = true;
      r->acc_n = r->acc_ng = 0;
    }
    int64_t round_cap_hit = 0;
    for (int32_t s0 = 0; s0 < B && !round_cap_hit; s0 += mb) {
      const int32_t s1 = std::min<int32_t>(B, s0 + mb);
      batch_cur = micro ? s1 - s0 : B;
      {
        HostTimer ht(host_ms[0]);
        static_idx.clear();
        ingest_chunk(micro ? s0 : 0, micro ? s1 : B);
      }
      mark("ingest");
      round_cap_hit = run_strata();
      for (size_t r = 0; r < prog.rels.size(); ++r)
        if (!prog.rels[r].input && !prog.rels[r].internal) stats.tuples_derived += rels[r]->n;
      if (!round_cap_hit && (semi == S_MAXMULT || dadd)) {
        Phase ph(this, 4);
        HostTimer htg(host_ms[5]);
        gradients();
      }
      mark("gradients");
      if (micro) collect_outputs(s0);
    }
    batch_cur = B;
    if (micro) finalize_collected();
    // the three device counters in one read, landing with finish_run's sync
    cuda_check(cudaMemcpyAsync(hbuf, d_ncand, 24, cudaMemcpyDeviceToHost, st), "D2H");
    stats.fj_row_bytes = 4 + (semi == S_UNIT ? 0 : (semi == S_MAXMULT ? 8 : 4));
    finish_run(t0, round_cap_hit, out, true);
  }

  // largest power-of-two sample range whose dense-eligible relations fit 30 bits
  int32_t choose_micro_batch() {
    const int32_t B = opt.batch_size;
    if (dadd) return B;  // the adjoint program reads the pushed facts of the whole batch
    if (opt.micro_batch > 0) return std::min(opt.micro_batch, B);
    const int sb_full = bits_for((uint64_t)B - 1);
    int excess = 0;
    for (size_t r = 0; r < prog.rels.size(); ++r) {
      const Relation& R = prog.rels[r];
      if (R.input || R.shared || rels[r]->build_local) continue;
      int cols = 0;
      for (int c = 0; c < R.arity; ++c) {
        const int cl = R.col_class[c];
        cols += bits_for((uint64_t)(class_max[cl] - class_min[cl]));
      }
      excess = std::max(excess, cols + sb_full - 30);
    }
    if (excess <= 0) return B;
    const int sb = sb_full - excess;
    if (sb < 0) return B;  // does not fit even per sample: sorted store, whole batch
    return std::min<int32_t>(B, (int32_t)1 << sb);
  }

  // append this chunk's `output` relations (sample ids rebased by s0) to the accumulators
  void collect_outputs(int32_t s0) {
    for (size_t r = 0; r < prog.rels.size(); ++r) {
      const Relation& R = prog.rels[r];
      if (R.input) continue;
      RelState& S = *rels[r];
      if (R.output) ensure_sorted(S);
      if (!R.output) {
        S.retained = false;
        continue;
      }
      const int64_t n = S.n, a = S.acc_n, ar = R.arity;
      S.acc_sid.reserve(a + n, a);
      for (int c = 0; c < ar; ++c) S.acc_col[c].reserve(a + n, a);
      if (n > 0) {
        int32_t* tcols = arena.get<int32_t>(std::max<int64_t>(1, ar * n));
        uint8_t* dsh = arena.get<uint8_t>(64);
        std::vector<uint8_t> hb(48, 0);
        for (int c = 0; c < ar; ++c) { hb[c] = (uint8_t)S.L.shift[c]; hb[8 + c] = (uint8_t)S.L.bits[c]; }
        std::memcpy(hb.data() + 16, S.L.mins.data(), ar * 4);
        cuda_check(cudaMemcpyAsync(dsh, hb.data(), hb.size(), cudaMemcpyHostToDevice, st), "H2D");
        launch_unpack(S.key.ptr(), n, S.L.has_sample, (uint8_t)S.L.sshift, (int)ar, dsh, dsh + 8,
                      reinterpret_cast<int32_t*>(dsh + 16), S.acc_sid.ptr() + a, tcols, st);
        launch_add_i32(S.acc_sid.ptr() + a, n, s0, st);
        for (int c = 0; c < ar; ++c)
          cuda_check(cudaMemcpyAsync(S.acc_col[c].ptr() + a, tcols + (int64_t)c * n, n * 4, cudaMemcpyDeviceToDevice, st),
                     "collect");
        if (semi != S_UNIT) {
          S.acc_p.reserve(a + n, a);
          cuda_check(cudaMemcpyAsync(S.acc_p.ptr() + a, S.p.ptr(), n * 4, cudaMemcpyDeviceToDevice, st), "collect");
        }
      }
      if (S.has_grad) {
        S.acc_goff.reserve(a + n + 1, a);
        launch_add_i64(S.goff.ptr(), n + 1, S.acc_ng, S.acc_goff.ptr() + a, st);
        S.acc_gfid.reserve(S.acc_ng + S.ng, S.acc_ng);
        S.acc_gval.reserve(S.acc_ng + S.ng, S.acc_ng);
        if (S.ng) {
          cuda_check(cudaMemcpyAsync(S.acc_gfid.ptr() + S.acc_ng, S.gfid.ptr(), S.ng * 8, cudaMemcpyDeviceToDevice, st),
                     "collect");
          cuda_check(cudaMemcpyAsync(S.acc_gval.ptr() + S.acc_ng, S.gval.ptr(), S.ng * 4, cudaMemcpyDeviceToDevice, st),
                     "collect");
        }
        S.acc_ng += S.ng;
      }
      S.acc_n += n;
      kcheck("collect outputs");
    }
    sync();
    arena.reset();
  }

  // accumulated outputs become the relation's output views
  void finalize_collected() {
    for (size_t r = 0; r < prog.rels.size(); ++r) {
      const Relation& R = prog.rels[r];
      RelState& S = *rels[r];
      if (R.input || !S.retained) continue;
      const int64_t n = S.acc_n, ar = R.arity;
      S.n = n;
      S.o_sid.swap(S.acc_sid);
      S.o_cols.reserve(std::max<int64_t>(1, ar * n));
      for (int c = 0; c < ar; ++c)
        if (n) cuda_check(cudaMemcpyAsync(S.o_cols.ptr() + (int64_t)c * n, S.acc_col[c].ptr(), n * 4,
                                          cudaMemcpyDeviceToDevice, st), "finalize");
      S.o_soff.reserve(opt.batch_size + 1);
      launch_sample_offsets_i32(S.o_sid.ptr(), n, opt.batch_size, S.o_soff.ptr(), st);
      if (sample_base && S.L.has_sample) launch_add_i32(S.o_sid.ptr(), n, sample_base, st);
      if (semi != S_UNIT) S.p.swap(S.acc_p);
      if (S.has_grad) {
        S.goff.swap(S.acc_goff);
        S.gfid.swap(S.acc_gfid);
        S.gval.swap(S.acc_gval);
        S.ng = S.acc_ng;
      }
      S.out_dev_ready = true;
      kcheck("finalize outputs");
    }
  }

  // one (micro-)batch: every stratum to fixpoint; returns 1 if max_iters was hit
  // Async rounds (direct strata): ring of pinned |Δ'| slots, one event per slot.
  // The extraction kernel writes (seq << 32 | |Δ'|) straight into host-mapped pinned
  // memory (zero-copy): no copy or event call per round, the host polls the words.
  static constexpr int ARING = 64, AREL = 8, ALAG = 6;
  unsigned long long* hring = nullptr;   // host view
  unsigned long long* dring = nullptr;   // device view of the same words
  uint32_t ring_seq = 0;                 // sequence of async rounds over the context's life
  int round_fused = 0, round_other = 0;
  int cur_round = 0;      // round of the stratum being issued (max-mult stamps)
  int64_t async_nd0 = 0;  // Δ rows probed by the first async round
  int async_nrel = 0;     // relations of the async stratum (ring entries per round)

  // Δ buffers must hold every slot (sizes are no longer known on the host)
  bool async_ok(const std::vector<int>& strat) {
    if (getenv("LOBSTER_SYNC_ROUNDS")) return false;
    size_t need = 0;
    for (int r : strat) {
      RelState& S = *rels[r];
      if (!S.direct) return false;
      const size_t row = 4 + (semi == S_UNIT ? 0 : 4);
      if (S.dkey32.bytes() < (size_t)S.nslots * 4) need += (size_t)S.nslots * row;
    }
    if (need) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      if ((double)need > 0.4 * (double)fr) return false;
    }
    if (!hring) {
      cuda_check(cudaHostAlloc(&hring, ARING * AREL * 8, cudaHostAllocMapped), "cudaHostAlloc");
      std::memset(hring, 0, ARING * AREL * 8);
      cuda_check(cudaHostGetDevicePointer((void**)&dring, hring, 0), "cudaHostGetDevicePointer");
    }
    return true;
  }

  // Consume finished rounds from the ring (all of them if `all`, else block only on
  // rounds more than ALAG behind).  Returns the first round whose Σ|Δ'| is 0, or 0.
  bool ring_ready(uint32_t seq) const {
    const volatile unsigned long long* e = hring + (seq % ARING) * AREL;
    for (int q = 0; q < async_nrel; ++q)
      if ((uint32_t)(e[q] >> 32) != seq) return false;
    return true;
  }

  int64_t drain_async(std::deque<std::pair<int, uint32_t>>& pending, size_t trace_base, bool all) {
    const int newest = pending.empty() ? 0 : pending.back().first;
    while (!pending.empty()) {
      const int pr = pending.front().first;
      const uint32_t seq = pending.front().second;
      if (all || newest - pr >= ALAG) {
        for (uint64_t spin = 0; !ring_ready(seq); ++spin)
          if ((spin & 1023) == 1023) {  // a failed kernel never writes its word
            const cudaError_t q = cudaStreamQuery(st);
            if (q == cudaSuccess && !ring_ready(seq)) throw Failure(LOBSTER_E_CUDA, "async round count missing");
            if (q != cudaSuccess && q != cudaErrorNotReady) cuda_check(q, "async round");
          }
      } else if (!ring_ready(seq)) {
        break;
      }
      pending.pop_front();
      int64_t sum = 0;
      const volatile unsigned long long* ent = hring + (seq % ARING) * AREL;
      for (int q = 0; q < async_nrel; ++q) sum += (uint32_t)ent[q];
      const int64_t probe = async_nd0;
      async_nd0 = sum;  // Δ' of this round = probe rows of the next
      stats.fj_probe_rows += probe;
      if (timed_rounds.count(pr)) stats.fj_timed_probe_rows += probe;
      stats.bytes_algorithmic += bytes_round_direct(probe, sum);
      if (log_level >= 2 && trace_base + pr - 1 < trace.size()) {
        trace[trace_base + pr - 1][1] = probe;
        trace[trace_base + pr - 1][2] = sum;
      }
      if (sum == 0) return pr;
    }
    return 0;
  }

  // ------------------------------------------------ diff-top-1-proofs
  // (k_top1.cu).  Linear rules only: a rule reads at most
  // one relation of its own stratum, whose proofs are then those of Δ (the
  // relation's proof index at round start); every other atom is external.
  std::vector<WalkRule> top1_rules;
  std::vector<int> top1_base;
  void top1_begin_stratum(const std::vector<int>& strat) {
    std::set<int> local(strat.begin(), strat.end());
    for (const Rule& R : prog.rules) {
      if (!local.count(R.head_rel)) continue;
      int nloc = 0;
      for (auto& a : R.body) nloc += local.count(a.rel) ? 1 : 0;
      if (nloc > 1)
        throw Failure(LOBSTER_E_SCHEMA, "diff-top-1-proofs: a rule for " + prog.rels[R.head_rel].name +
                                            " reads its own stratum twice (linear recursion only on the GPU)");
    }
    for (int r : strat) {
      rels[r]->npx = 0;
      rels[r]->pool_n = 0;
    }
    if (top1_rules.empty()) build_walk_rules(top1_rules, top1_base);
  }

  // device tables of every relation's proof source (rebuilt per use: buffers move)
  ProofTables top1_tables() {
    const int nr = (int)prog.rels.size();
    std::vector<ProofRel> pr(nr);
    for (int r = 0; r < nr; ++r) {
      RelState& S = *rels[r];
      ProofRel& q = pr[r];
      std::memset(&q, 0, sizeof(q));
      if (prog.rels[r].input) {
        q.key = S.key.ptr();
        q.n = S.n;
        q.fid = S.fid.ptr();
      } else {
        q.key = S.pkey.ptr();
        q.n = S.npx;
        q.pof = S.pof.ptr();
        q.pln = S.pln.ptr();
        q.pool = S.pool.ptr();
      }
      q.has_sample = S.L.has_sample ? 1 : 0;
      q.sshift = (uint8_t)S.L.sshift;
      for (int c = 0; c < prog.rels[r].arity; ++c) {
        q.shift[c] = (uint8_t)S.L.shift[c];
        q.bits[c] = (uint8_t)S.L.bits[c];
        q.min[c] = S.L.mins[c];
      }
    }
    ProofTables T{};
    T.rels = arena.get<ProofRel>(nr);
    T.rules = arena.get<WalkRule>((int64_t)top1_rules.size());
    T.rule_base = arena.get<int>(nr);
    T.rule_bits = arena.get<int>(nr);
    cuda_check(cudaMemcpyAsync(T.rels, pr.data(), nr * sizeof(ProofRel), cudaMemcpyHostToDevice, st), "H2D");
    if (!top1_rules.empty())
      cuda_check(cudaMemcpyAsync(T.rules, top1_rules.data(), top1_rules.size() * sizeof(WalkRule),
                                 cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(T.rule_base, top1_base.data(), nr * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(T.rule_bits, rule_bits.data(), nr * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    T.fact_p = fact_p.ptr();
    T.group = has_groups ? fact_group.ptr() : nullptr;
    T.cap = 300;
    return T;
  }

  void top1_check(int* d_err) {
    const int e = read_dev(d_err);
    if (e & 8) throw Failure(LOBSTER_E_RANGE, "diff-top-1-proofs: a proof exceeds 300 facts (P:628)");
    if (e) throw Failure(LOBSTER_E_CUDA, "top-1-proof: inconsistent body tuple (code " + std::to_string(e) + ")");
  }

  // candidates: the union proof's p replaces the ⊗ of the body tags; conflicting
  // candidates are dropped (dead keys) before the sort
  void top1_candidates(int r, RelState& S, int64_t nc) {
    Phase ph(this, 2);
    ProofTables T = top1_tables();
    int* d_err = arena.get<int>(1);
    cuda_check(cudaMemsetAsync(d_err, 0, 4, st), "memset");
    launch_top1_cand(T, r, S.ckey.ptr(), S.cv64.ptr(), nc, d_err, st);
    kcheck("top1 candidates");
    top1_check(d_err);
  }

  // after every relation of the round settled: Δ' proofs appended to the
  // pools, proof indexes updated (in place for improved tuples, merged for new)
  void top1_commit(const std::vector<int>& strat) {
    ProofTables T = top1_tables();  // round-start indexes: all Δ' unions read them
    int* d_err = arena.get<int>(1);
    cuda_check(cudaMemsetAsync(d_err, 0, 4, st), "memset");
    std::vector<int64_t> need(strat.size(), 0);
    for (size_t q = 0; q < strat.size(); ++q) {  // proof lengths -> offsets in the pool
      RelState& S = *rels[strat[q]];
      const int64_t nd = S.nd;
      if (nd <= 0) continue;
      S.dln.reserve(nd);
      S.dof.reserve(nd + 1);
      launch_top1_delta(T, strat[q], S.dkey.ptr(), S.dw.ptr(), nd, S.dln.ptr(), nullptr, nullptr, d_err, st);
      uint64_t* len64 = arena.get<uint64_t>(nd);
      launch_widen_u32(S.dln.ptr(), nd, len64, st);
      exclusive_scan<uint64_t>(len64, S.dof.ptr(), nd, S.dof.ptr() + nd, arena.alloc(scan_tmp_bytes<uint64_t>(nd)), st);
      kcheck("top1 lengths");
    }
    for (size_t q = 0; q < strat.size(); ++q) {
      RelState& S = *rels[strat[q]];
      if (S.nd > 0) need[q] = (int64_t)read_dev(S.dof.ptr() + S.nd);
    }
    top1_check(d_err);
    for (size_t q = 0; q < strat.size(); ++q) {
      RelState& S = *rels[strat[q]];
      const int64_t nd = S.nd;
      if (nd <= 0) continue;
      // the pool grows x1.5 and keeps its contents; live proofs are re-packed
      // when the garbage (proofs of since-improved tuples) dominates
      S.pool.reserve(S.pool_n + need[q], S.pool_n);
      launch_add_i64(reinterpret_cast<const int64_t*>(S.dof.ptr()), nd, S.pool_n,
                     reinterpret_cast<int64_t*>(S.dof.ptr()), st);
      launch_top1_delta(T, strat[q], S.dkey.ptr(), S.dw.ptr(), nd, nullptr, S.dof.ptr(), S.pool.ptr(), d_err, st);
      S.pool_n += need[q];
      // proof index: improved tuples in place, new tuples merged by rank
      uint32_t* isnew = arena.get<uint32_t>(nd);
      uint32_t* pos = arena.get<uint32_t>(nd + 1);
      launch_top1_update(S.pkey.ptr(), S.npx, S.pof.ptr(), S.pln.ptr(), S.dkey.ptr(), S.dof.ptr(), S.dln.ptr(), nd,
                         isnew, st);
      exclusive_scan<uint32_t>(isnew, pos, nd, pos + nd, arena.alloc(scan_tmp_bytes<uint32_t>(nd)), st);
      const int64_t nnew = (int64_t)read_dev(pos + nd);
      if (nnew > 0) {
        uint64_t* nk = arena.get<uint64_t>(nnew);
        uint64_t* no = arena.get<uint64_t>(nnew);
        uint32_t* nl = arena.get<uint32_t>(nnew);
        launch_top1_compact(S.dkey.ptr(), S.dof.ptr(), S.dln.ptr(), isnew, pos, nd, nk, no, nl, st);
        const int64_t nn = S.npx + nnew;
        S.pkey2.reserve(nn);
        S.pof2.reserve(nn);
        S.pln2.reserve(nn);
        launch_top1_merge(S.pkey.ptr(), S.pof.ptr(), S.pln.ptr(), S.npx, nk, no, nl, nnew, S.pkey2.ptr(), S.pof2.ptr(),
                          S.pln2.ptr(), st);
        S.pkey.swap(S.pkey2);
        S.pof.swap(S.pof2);
        S.pln.swap(S.pln2);
        S.npx = nn;
      }
      kcheck("top1 commit");
      top1_maybe_compact(S);
    }
    top1_check(d_err);
  }

  void top1_maybe_compact(RelState& S) {
    if (S.pool_n < ((int64_t)1 << 20) || S.npx == 0) return;
    uint64_t* len64 = arena.get<uint64_t>(S.npx);
    uint64_t* noff = arena.get<uint64_t>(S.npx + 1);
    launch_widen_u32(S.pln.ptr(), S.npx, len64, st);
    exclusive_scan<uint64_t>(len64, noff, S.npx, noff + S.npx, arena.alloc(scan_tmp_bytes<uint64_t>(S.npx)), st);
    const int64_t live = (int64_t)read_dev(noff + S.npx);
    if (2 * live >= S.pool_n) return;
    S.pool2.reserve(live);
    launch_top1_gather(S.pool.ptr(), S.pof.ptr(), S.pln.ptr(), noff, S.npx, S.pool2.ptr(), st);
    cuda_check(cudaMemcpyAsync(S.pof.ptr(), noff, S.npx * 8, cudaMemcpyDeviceToDevice, st), "copy");
    S.pool.swap(S.pool2);
    S.pool_n = live;
    kcheck("top1 pool compaction");
  }

  // gradients of every output relation straight from its proofs
  void top1_gradients() {
    for (size_t r = 0; r < prog.rels.size(); ++r) {
      if (!prog.rels[r].output || prog.rels[r].input) continue;
      RelState& S = *rels[r];
      ensure_sorted(S);
      const int64_t n = S.n;
      if (n != S.npx) throw Failure(LOBSTER_E_CUDA, "top-1-proof: proof index out of step with the relation");
      S.goff.reserve(n + 1);
      uint64_t* len64 = arena.get<uint64_t>(n);
      uint64_t* noff = arena.get<uint64_t>(n + 1);
      if (n) launch_widen_u32(S.pln.ptr(), n, len64, st);
      exclusive_scan<uint64_t>(len64, noff, n, noff + n, arena.alloc(scan_tmp_bytes<uint64_t>(n)), st);
      const int64_t ng = n ? (int64_t)read_dev(noff + n) : 0;
      S.gfid.reserve(ng);
      S.gval.reserve(ng);
      double* scratch = arena.get<double>(ng);
      launch_top1_grad(S.pool.ptr(), S.pof.ptr(), S.pln.ptr(), noff, n, fact_p.ptr(), S.goff.ptr(), S.gfid.ptr(),
                       S.gval.ptr(), scratch, st);
      kcheck("top1 gradients");
      S.ng = ng;
      S.has_grad = true;
    }
  }

  // ------------------------------------------------ bit-sliced frontier
  // A stratum qualifies when: unit semiring; one batched unary relation R in a
  // direct (bitmap) store; every rule of R is either all-external (the seed
  // round, evaluated as usual) or R(u) :- R(v), E(.., ..) / E(.., ..), R(v)
  // with E a SHARED binary input whose columns are v and u (distinct
  // variables of R's domain class), no constants, no comparisons.
  struct SliceRule {
    int erel;      // the shared binary relation
    int ccol;      // its column joined with R's variable
    int hcol;      // its column projected to R's head
  };
  bool slice_ok(const std::vector<int>& strat, std::vector<SliceRule>& out) {
    out.clear();
    if (no_slice || semi != S_UNIT || strat.size() != 1) return false;
    const int r = strat[0];
    const Relation& RR = prog.rels[r];
    RelState& S = *rels[r];
    if (RR.arity != 1 || RR.shared || !S.direct || !S.L.has_sample || S.L.bits[0] > 24) return false;
    for (const Rule& R : prog.rules) {
      if (R.head_rel != r) continue;
      int nloc = 0;
      for (auto& a : R.body) nloc += a.rel == r;
      if (nloc == 0) continue;  // seed rule: already evaluated
      if (R.body.size() != 2 || nloc != 1 || !R.cmps.empty() || !R.head[0].is_var()) return false;
      const BodyAtom& ra = R.body[0].rel == r ? R.body[0] : R.body[1];
      const BodyAtom& ea = R.body[0].rel == r ? R.body[1] : R.body[0];
      const Relation& E = prog.rels[ea.rel];
      if (!E.input || !E.shared || E.arity != 2 || !ra.args[0].is_var()) return false;
      if (!ea.args[0].is_var() || !ea.args[1].is_var()) return false;
      const int v = ra.args[0].var, u = R.head[0].var;
      if (u == v) return false;
      SliceRule sr;
      if (ea.args[0].var == v && ea.args[1].var == u) { sr.ccol = 0; sr.hcol = 1; }
      else if (ea.args[1].var == v && ea.args[0].var == u) { sr.ccol = 1; sr.hcol = 0; }
      else return false;
      sr.erel = ea.rel;
      const Layout& EL = rels[ea.rel]->L;
      if (EL.mins[0] != S.L.mins[0] || EL.mins[1] != S.L.mins[0] || EL.bits[0] != S.L.bits[0] ||
          EL.bits[1] != S.L.bits[0] || rels[ea.rel]->n >= ((int64_t)1 << 32))
        return false;
      out.push_back(sr);
    }
    return !out.empty() && out.size() <= 4;
  }

  // Rounds 2.. of a qualifying stratum on bit-sliced words; R's bitmap holds
  // the seed round's tuples on entry and every tuple on exit.  Returns the
  // rounds run (the last one empty, as in the per-sample loop).
  int run_sliced(RelState& S, const std::vector<SliceRule>& srules) {
    const int tbits = S.L.bits[0];
    const int64_t T = (int64_t)1 << tbits;
    const int B = batch_cur;
    const int W = (B + 31) / 32;
    const int64_t nw = T * W;         // sliced words
    const int64_t ndw = (nw + 31) / 32;  // dirty-bitmap words
    while (sl.off.size() < srules.size()) {
      sl.off.emplace_back(new DBuf<uint32_t>());
      sl.nbr.emplace_back(new DBuf<uint32_t>());
      sl.off.back()->bind(st);
      sl.nbr.back()->bind(st);
    }
    sl.cnt.reserve(T + 4);
    sl.scan.reserve((int64_t)(scan_tmp_bytes<uint32_t>(std::max<int64_t>(T + 1, nw)) / 4 + 1));
    for (size_t q = 0; q < srules.size(); ++q) {  // per-rule CSR of E by its joined column
      const RelState& E = *rels[srules[q].erel];
      sl.off[q]->reserve(T + 1);
      sl.nbr[q]->reserve(std::max<int64_t>(E.n, 1));
      launch_slice_csr(E.key.ptr(), E.n, E.L.shift[srules[q].ccol], E.L.shift[srules[q].hcol], tbits, T,
                       sl.off[q]->ptr(), sl.cnt.ptr(), sl.nbr[q]->ptr(), sl.scan.ptr(), st);
    }
    sl.Rb.reserve(nw);
    sl.Nb.reserve(nw);
    sl.dt.reserve(nw);
    sl.dwi.reserve(nw);
    sl.dbits.reserve(nw);
    sl.deg.reserve(nw + 1);
    sl.pos.reserve(nw + 1);
    sl.tup.reserve(1);
    uint32_t* dirty = S.dirty.ptr();  // sized for B·T bits >= T·W bits; zero between rounds
    cuda_check(cudaMemsetAsync(sl.Rb.ptr(), 0, nw * 4, st), "memset");
    cuda_check(cudaMemsetAsync(sl.tup.ptr(), 0, 8, st), "memset");
    uint32_t* bm = reinterpret_cast<uint32_t*>(S.dirf.get());
    launch_slice_from_bitmap(bm, tbits, B, T, W, sl.Nb.ptr(), dirty, st);
    kcheck("slice from bitmap");
    // Δ of round 2 = the seed round's tuples
    uint32_t* count = sl.cnt.ptr() + ((T + 2) & ~(int64_t)1);  // two scratch words (8-B aligned) after the CSR counts
    // count[0] = |Δ'| (entries), count[1] = (edge, word) items of the round's joins
    int64_t items = 0;
    auto extract = [&]() -> int64_t {
      Phase ph(this, 3);
      cuda_check(cudaMemsetAsync(count, 0, 4, st), "memset");
      launch_slice_extract(dirty, ndw, sl.Nb.ptr(), sl.Rb.ptr(), W, sl.dt.ptr(), sl.dwi.ptr(), sl.dbits.ptr(), count,
                           sl.tup.ptr(), st);
      kcheck("slice extract");
      const uint64_t both = read_dev(reinterpret_cast<const uint64_t*>(count));
      items = (int64_t)(both >> 32);
      return (int64_t)(both & 0xffffffffu);
    };
    int64_t nd = extract();
    int rounds = 0;
    round_cap_hit_slice = false;
    while (nd > 0) {
      if (rounds + 1 >= max_iters) {  // the stratum's round 1 was the seed round
        round_cap_hit_slice = true;
        break;
      }
      ++rounds;
      {
        Phase ph(this, 0);
        for (size_t q = 0; q < srules.size(); ++q) {
          launch_slice_deg(sl.dt.ptr(), nd, sl.off[q]->ptr(), sl.deg.ptr(), st);
          exclusive_scan<uint32_t>(sl.deg.ptr(), sl.pos.ptr(), nd, sl.pos.ptr() + nd, sl.scan.ptr(), st);
          launch_slice_expand(sl.dt.ptr(), sl.dwi.ptr(), sl.dbits.ptr(), sl.pos.ptr(), nd, sl.pos.ptr() + nd,
                              sl.off[q]->ptr(), sl.nbr[q]->ptr(), sl.Rb.ptr(), sl.Nb.ptr(), W, dirty, d_ncand, st);
          // this rule's item total joins count[1] (read with |Δ'| after the extraction)
          launch_add_u32_dev(count + 1, sl.pos.ptr() + nd, q == 0, st);
        }
        kcheck("slice join");
      }
      // §8(d) bytes of the sliced round: Δ triples read (12 B), per (edge, word)
      // item the neighbour id and the target word (8 B), Δ' word update + triple (16 B)
      const int64_t nd_prev = nd;
      nd = extract();
      stats.bytes_algorithmic += nd_prev * 12 + items * 8 + nd * 16;
      sl_items += items;
    }
    // all tuples back into R's (s, t) bitmap (downstream strata, outputs, counting)
    cuda_check(cudaMemsetAsync(bm, 0, (size_t)((S.nslots + 31) / 32) * 4, st), "memset");
    launch_slice_to_bitmap(sl.Rb.ptr(), tbits, B, T, W, bm, st);
    kcheck("slice to bitmap");
    return rounds;
  }
  bool round_cap_hit_slice = false;
  int64_t sl_items = 0;  // (edge, word) items of the sliced joins in this run (diagnostics)

  // ------------------------------------------------ key-partitioned evaluation
  // (xfer.hpp).  Inputs are replicated, IDB tuples owned
  // by the hash of their packed key.  Seed-round candidates are derived on
  // every rank, so each keeps the ones it owns; later rounds derive each
  // candidate once (linear rules: the Δ atom's tuple lives on one rank) and
  // send it to its owner.  Buckets are stable (radix sort by owner), so a
  // receiver's candidate order is deterministic.
  int64_t* host_counts() {
    if (!hx) cuda_check(cudaMallocHost(&hx, 3 * 64 * sizeof(int64_t)), "cudaMallocHost");
    return hx;
  }

  int64_t part_exchange(RelState& S, int64_t nc) {
    const bool k32 = c32(S);
    void* keys = k32 ? (void*)S.ckey32.ptr() : (void*)S.ckey.ptr();
    const int W = xfer->world;
    if (cur_round == 1) {
      launch_part_keep(keys, k32, nc, (uint32_t)W, (uint32_t)part_rank, st);
      kcheck("part keep");
      return nc;
    }
    const int kb = k32 ? 4 : 8;
    const bool tags = semi != S_UNIT;
    uint32_t* dest = arena.get<uint32_t>(nc);
    uint32_t* idx = arena.get<uint32_t>(nc);
    uint32_t* dest2 = arena.get<uint32_t>(nc);
    uint32_t* idx2 = arena.get<uint32_t>(nc);
    unsigned long long* cnt = arena.get<unsigned long long>(W + 1);
    int64_t* h = host_counts();
    cuda_check(cudaMemsetAsync(cnt, 0, (W + 1) * 8, st), "memset");
    launch_part_dest(keys, k32, nc, (uint32_t)W, dest, idx, cnt, st);
    const int which = radix_sort(dest, idx, dest2, idx2, nc, bits_for((uint64_t)W), arena.alloc(sort_tmp_bytes(nc)), st);
    const uint32_t* perm = which ? idx2 : idx;
    cuda_check(cudaMemcpyAsync(h, cnt, (W + 1) * 8, cudaMemcpyDeviceToHost, st), "D2H");
    int64_t nsend = 0;
    void* sk = arena.alloc((size_t)std::max<int64_t>(nc, 1) * kb);
    void* sv = tags ? arena.alloc((size_t)std::max<int64_t>(nc, 1) * 4) : nullptr;
    sync();
    for (int d = 0; d < W; ++d) nsend += h[d];  // dead candidates (bucket W) are dropped
    launch_part_gather(keys, perm, sk, nsend, kb, st);
    if (tags) launch_part_gather(S.cv32.ptr(), perm, sv, nsend, 4, st);
    kcheck("part gather");
    int64_t* rc = h + 64;
    Phase ph(this, 6);
    xfer->counts(part_rank, h, rc, st);
    int64_t nr = 0;
    for (int d = 0; d < W; ++d) nr += rc[d];
    std::vector<int64_t> scnt(h, h + W), rcnt(rc, rc + W);
    reserve_candidates_for(S, nr);
    void* rk = k32 ? (void*)S.ckey32.ptr() : (void*)S.ckey.ptr();
    xfer->alltoallv(part_rank, sk, scnt.data(), rk, rcnt.data(), kb, st);
    if (tags) xfer->alltoallv(part_rank, sv, scnt.data(), S.cv32.ptr(), rcnt.data(), 4, st);
    return nr;
  }

  void reserve_candidates_for(RelState& S, int64_t n) {
    if (c32(S)) S.ckey32.reserve(n);
    else S.ckey.reserve(n);
    if (semi != S_UNIT) S.cv32.reserve(n);
  }

  int64_t part_sum(int64_t v) {
    int64_t* h = host_counts();
    const int W = xfer->world;
    for (int d = 0; d < W; ++d) h[d] = v;
    xfer->counts(part_rank, h, h + 64, st);
    int64_t s = 0;
    for (int d = 0; d < W; ++d) s += h[64 + d];
    return s;
  }

  bool read_later(int r, size_t si) const {
    for (const Rule& R : prog.rules) {
      if ((size_t)prog.rels[R.head_rel].stratum <= si) continue;
      for (auto& a : R.body)
        if (a.rel == r) return true;
    }
    return false;
  }

  // every rank gets the whole relation (sorted, keys disjoint across ranks)
  void part_gather(RelState& S) {
    ensure_sorted(S);
    const int W = xfer->world;
    int64_t* h = host_counts();
    for (int d = 0; d < W; ++d) h[d] = S.n;
    xfer->counts(part_rank, h, h + 64, st);
    int64_t nr = 0;
    for (int d = 0; d < W; ++d) nr += h[64 + d];
    std::vector<int64_t> scnt(h, h + W), rcnt(h + 64, h + 64 + W);
    const bool tags = semi != S_UNIT;
    uint64_t* sk = arena.get<uint64_t>(std::max<int64_t>(1, S.n * W));
    uint32_t* sv = tags ? arena.get<uint32_t>(std::max<int64_t>(1, S.n * W)) : nullptr;
    for (int d = 0; d < W && S.n; ++d) {
      cuda_check(cudaMemcpyAsync(sk + d * S.n, S.key.ptr(), S.n * 8, cudaMemcpyDeviceToDevice, st), "gather");
      if (tags) cuda_check(cudaMemcpyAsync(sv + d * S.n, S.p.ptr(), S.n * 4, cudaMemcpyDeviceToDevice, st), "gather");
    }
    uint64_t* k0 = arena.get<uint64_t>(nr);
    uint64_t* k1 = arena.get<uint64_t>(nr);
    uint32_t* v0 = tags ? arena.get<uint32_t>(nr) : nullptr;
    uint32_t* v1 = tags ? arena.get<uint32_t>(nr) : nullptr;
    xfer->alltoallv(part_rank, sk, scnt.data(), k0, rcnt.data(), 8, st);
    if (tags) xfer->alltoallv(part_rank, sv, scnt.data(), v0, rcnt.data(), 4, st);
    void* stmp = arena.alloc(sort_tmp_bytes(nr));
    int which;
    if (tags) which = radix_sort(k0, v0, k1, v1, nr, S.L.total, stmp, st);
    else which = radix_sort<uint64_t, void>(k0, nullptr, k1, nullptr, nr, S.L.total, stmp, st);
    S.key.reserve(nr);
    cuda_check(cudaMemcpyAsync(S.key.ptr(), which ? k1 : k0, nr * 8, cudaMemcpyDeviceToDevice, st), "gather");
    if (tags) {
      S.p.reserve(nr);
      cuda_check(cudaMemcpyAsync(S.p.ptr(), which ? v1 : v0, nr * 4, cudaMemcpyDeviceToDevice, st), "gather");
    }
    kcheck("part gather");
    S.n = nr;
  }

  // ------------------------------------------------ small dense strata (k_tile.cu)
  // A stratum qualifies when: unit / max-min / add-mult; every relation of it
  // batched with arity <= 4; every rule within the plan limits, the variable
  // that closes an atom appears once in it and has a domain <= 64; and the
  // stratum's S / Δ / U arrays plus fibers fit one CTA's shared memory.
  bool no_tile = getenv("LOBSTER_NO_TILE") != nullptr;  // A/B: the per-round path
  bool no_tile_compact = getenv("LOBSTER_NO_TILE_COMPACT") != nullptr;  // A/B: every head slot every round
  int64_t tile_max_slots = getenv("LOBSTER_TILE") ? INT64_MAX : 65536;
  TilePlan* hplan = nullptr;  // pinned
  int64_t class_dom(int cl) const { return class_max[cl] - class_min[cl] + 1; }

  bool tile_plan(const std::vector<int>& strat, TilePlan& P, std::vector<int>& prel) {
    if (no_tile || top1 || omin || semi == S_MAXMULT || xfer) return false;
    std::memset(&P, 0, sizeof(P));
    P.semi = semi;
    P.nsamples = batch_cur;
    P.max_iters = max_iters;
    std::set<int> local(strat.begin(), strat.end());
    prel.clear();
    auto plan_rel = [&](int r) -> int {
      for (size_t i = 0; i < prel.size(); ++i)
        if (prel[i] == r) return (int)i;
      if ((int)prel.size() >= TILE_MAXREL) return -1;
      const Relation& R = prog.rels[r];
      if (R.arity > TILE_MAXCOL) return -1;
      TileRel& T = P.rel[prel.size()];
      T.ncols = (int8_t)R.arity;
      T.local = local.count(r) ? 1 : 0;
      T.shared = R.shared ? 1 : 0;
      if (T.local && (R.shared || rels[r]->L.total > 30)) return -1;
      int64_t D = 1;
      for (int c = R.arity - 1; c >= 0; --c) {
        T.stride[c] = (int32_t)D;
        T.dom[c] = (int32_t)class_dom(R.col_class[c]);
        D *= T.dom[c];
        if (D > (1 << 20)) return -1;
      }
      T.D = (int32_t)D;
      for (int c = 0; c < TILE_MAXCOL; ++c) {
        for (int k = 0; k < 3; ++k) T.sm_tag[k] = T.sm_bits[k] = -1;
        T.sm_fib[0][c] = T.sm_fib[1][c] = -1;
      }
      prel.push_back(r);
      return (int)prel.size() - 1;
    };
    for (int r : strat) {
      const int i = plan_rel(r);
      if (i < 0 || !rels[r]->L.has_sample) return false;
      P.local_rel[P.nlocal++] = (int8_t)i;
    }
    for (const Rule& R : prog.rules) {
      if (!local.count(R.head_rel)) continue;
      if (P.nrule >= TILE_MAXRULE || (int)R.var_names.size() > TILE_MAXV || (int)R.nonhead.size() > TILE_MAXLEV ||
          (int)R.body.size() > MAXT || (int)R.cmps.size() > MAXC)
        return false;
      for (auto& e : R.head_expr)
        if (e.op) return false;  // arithmetic: the projection kernel's bytecode
      for (auto& c : R.cmps)
        if (c.is_expr) return false;
      TileRule& T = P.rule[P.nrule++];
      T.head = (int8_t)plan_rel(R.head_rel);
      std::vector<int> lev(R.var_names.size(), -1);
      for (size_t i = 0; i < R.nonhead.size(); ++i) {
        lev[R.nonhead[i]] = (int)i;
        T.lev_var[i] = (int8_t)R.nonhead[i];
      }
      T.nlev = (int8_t)R.nonhead.size();
      for (size_t v = 0; v < R.var_names.size(); ++v) {
        if (class_dom(R.var_class[v]) > 64) return false;  // values are packed 6 bits per variable
        T.vdom[v] = (int32_t)class_dom(R.var_class[v]);
        T.vmin[v] = (int32_t)class_min[R.var_class[v]];
      }
      const Relation& HR = prog.rels[R.head_rel];
      for (int c = 0; c < HR.arity; ++c) {
        T.hvar[c] = (int8_t)R.head[c].var;
        if (!R.head[c].is_var()) {
          const int64_t x = (int64_t)R.head[c].cst - class_min[HR.col_class[c]];
          T.hcst[c] = (x < 0 || x >= class_dom(HR.col_class[c])) ? -1 : (int32_t)x;
        }
      }
      T.natoms = (int8_t)R.body.size();
      std::vector<int> lpos;
      for (int a = 0; a < (int)R.body.size(); ++a) {
        const BodyAtom& B = R.body[a];
        const int pi = plan_rel(B.rel);
        if (pi < 0) return false;
        if (local.count(B.rel)) lpos.push_back(a);
        TileAtom& A = T.atom[a];
        A.rel = (int8_t)pi;
        A.level = -1;
        A.fcol = -1;
        for (int c = 0; c < (int)B.args.size(); ++c) {
          A.var[c] = (int8_t)B.args[c].var;
          if (!B.args[c].is_var()) {
            A.cst[c] = (int32_t)((int64_t)B.args[c].cst - class_min[prog.rels[B.rel].col_class[c]]);
          } else if (lev[B.args[c].var] > A.level) {
            A.level = (int8_t)lev[B.args[c].var];
            A.fcol = (int8_t)c;
          }
        }
        A.chk = -1;
        if (A.level >= 0)
          for (int c = 0; c < (int)B.args.size(); ++c)
            if (B.args[c].is_var() && c != A.fcol && lev[B.args[c].var] > A.chk) A.chk = (int8_t)lev[B.args[c].var];
        if (A.level >= 0) {  // the closing variable: one column, domain <= 64
          int occ = 0;
          for (auto& t : B.args) occ += t.is_var() && t.var == B.args[A.fcol].var;
          TileRel& TR = P.rel[pi];
          if (occ != 1 || TR.dom[A.fcol] > 64) return false;
          TR.nfib[A.fcol] = TR.D / TR.dom[A.fcol];
        }
      }
      if ((int)lpos.size() > TILE_MAXVAR) return false;
      if (lpos.empty()) {
        T.seed = 1;
        T.nvariant = 1;
        for (int a = 0; a < T.natoms; ++a) T.ver[0][a] = TV_EXT;
      } else {
        T.nvariant = (int8_t)lpos.size();
        for (size_t j = 0; j < lpos.size(); ++j) {
          for (int a = 0; a < T.natoms; ++a) T.ver[j][a] = TV_EXT;
          for (size_t q = 0; q < lpos.size(); ++q)
            T.ver[j][lpos[q]] = q == j ? TV_DELTA : (q < j ? TV_NEW : TV_OLD);
        }
      }
      // the composition shape (tile_device.cuh compose_head): H(a,x,z) :- H(b,x,y), H(c,y,z), T(b,c,a)
      T.shape = 0;
      if (R.body.size() == 3 && R.cmps.empty() && lpos.size() == 2 && lpos[0] == 0 && lpos[1] == 1 &&
          R.body[0].rel == R.head_rel && R.body[1].rel == R.head_rel && !local.count(R.body[2].rel) &&
          prog.rels[R.head_rel].arity == 3 && prog.rels[R.body[2].rel].arity == 3) {
        bool ok = true;
        for (auto& a : R.body)
          for (auto& t : a.args) ok &= t.is_var();
        for (auto& t : R.head) ok &= t.is_var();
        if (ok) {
          const int b = R.body[0].args[0].var, x = R.body[0].args[1].var, y = R.body[0].args[2].var;
          const int c = R.body[1].args[0].var, z = R.body[1].args[2].var, av = R.body[2].args[2].var;
          const std::set<int> distinct{b, x, y, c, z, av};
          ok = distinct.size() == 6 && R.body[1].args[1].var == y && R.body[2].args[0].var == b &&
               R.body[2].args[1].var == c && R.head[0].var == av && R.head[1].var == x && R.head[2].var == z;
        }
        if (ok) T.shape = 1;
      }
      T.ncmp = (int8_t)R.cmps.size();
      for (size_t i = 0; i < R.cmps.size(); ++i) {
        const Compare& c = R.cmps[i];
        TileCmp& t = T.cmp[i];
        t.va = (int8_t)c.a.var;
        t.vb = (int8_t)c.b.var;
        t.ca = c.a.cst;
        t.cb = c.b.cst;
        t.neq = c.rel;  // relational operator (program.hpp RelOp)
        t.level = (int8_t)std::max(c.a.is_var() ? lev[c.a.var] : -1, c.b.is_var() ? lev[c.b.var] : -1);
      }
    }
    P.nrel = (int)prel.size();
    // compacted composition rounds (tile_device.cuh compose_rounds): one local
    // relation whose only recursive rule is the composition shape.  (Fibers
    // along its middle column, to cut each lane's y walk to the y with a
    // candidate, measured slower: 13.8 vs 8.7 ms on C3 — the walk was uniform
    // across a warp's lanes, the cut one diverges.)
    P.cm_rule = -1;
    P.cm_off = 0;
    P.cm_nocert = getenv("LOBSTER_TILE_NO_CERT") ? 1 : 0;
    P.cm_nosplit = getenv("LOBSTER_TILE_NO_SPLIT") ? 1 : 0;
    if (P.nlocal == 1 && !no_tile_compact) {
      int cm = -1, nrec = 0;
      for (int i = 0; i < P.nrule; ++i) {
        if (P.rule[i].seed) continue;
        ++nrec;
        if (P.rule[i].shape == 1 && P.rule[i].head == P.local_rel[0]) cm = i;
      }
      if (nrec == 1 && cm >= 0) {
        P.cm_rule = cm;
        TileRel& H = P.rel[P.local_rel[0]];
        H.nfib[1] = H.D / H.dom[1];  // middle-column fibers (compose_bc32)
      }
    }
    // fiber strides (row-major over the other columns) and the shared-memory layout:
    // [fibers S, Δ | bits S, Δ] (zeroed per sample) then [bits U | tags S, Δ, U]
    int64_t off = 0;
    for (int i = 0; i < P.nrel; ++i) {
      TileRel& T = P.rel[i];
      for (int c = 0; c < T.ncols; ++c) {
        int64_t m = 1;
        for (int q = T.ncols - 1; q >= 0; --q) {
          if (q == c) continue;
          T.fstride[c][q] = (int32_t)m;
          m *= T.dom[q];
        }
      }
      if (!T.local) continue;
      for (int c = 0; c < T.ncols; ++c)
        for (int k = 0; k < 2 && T.nfib[c]; ++k) {
          T.sm_fib[k][c] = (int32_t)off;
          off += (int64_t)T.nfib[c] * 8;
        }
    }
    for (int i = 0; i < P.nrel; ++i) {
      TileRel& T = P.rel[i];
      if (!T.local) continue;
      for (int k = 0; k < 2; ++k) {
        T.sm_bits[k] = (int32_t)off;
        off += (int64_t)((T.D + 31) / 32) * 4;
      }
    }
    P.clear_words = (int32_t)(off / 4);
    for (int i = 0; i < P.nrel; ++i) {
      TileRel& T = P.rel[i];
      if (!T.local) continue;
      T.sm_bits[2] = (int32_t)off;
      off += (int64_t)((T.D + 31) / 32) * 4;
      if (semi != S_UNIT)
        for (int k = 0; k < 3; ++k) {
          T.sm_tag[k] = (int32_t)off;
          off += (int64_t)T.D * 4;
        }
    }
    if (P.cm_rule >= 0) {  // compacted composition rounds: masks + pair list
      const TileRel& H = P.rel[P.local_rel[0]];
      off = (off + 15) & ~int64_t(15);
      P.cm_off = (int32_t)off;
      off += 320 * 8 + 64 + (int64_t)H.dom[1] * H.dom[2] * 6 + 8 + (int64_t)TILE_CM_PARTS * 16;
    }
    if (off > 200 * 1024) return false;
    // Each round pulls every head slot of every sample through an interpreted
    // enumeration: a win for tiny problems (one launch instead of ~20 per
    // round and a host sync per join), a loss once the batch holds more than
    // ~64k head slots (measured: C3, 2M slots, 210 ms vs 32 ms per step).
    // LOBSTER_TILE=1 forces the path (parity tests at full size).
    int64_t slots = 0;
    for (int i = 0; i < P.nrel; ++i)
      if (P.rel[i].local) slots += (int64_t)P.rel[i].D * batch_cur;
    bool spelled = true;  // every recursive rule has a spelled-out shape (no interpretation)
    for (int i = 0; i < P.nrule; ++i) spelled &= P.rule[i].seed || P.rule[i].shape != 0;
    if (slots > tile_max_slots && !spelled) return false;
    P.smem_bytes = (int32_t)std::max<int64_t>(off, 16);
    return true;
  }

  // Run a qualifying stratum in one launch; its relations end in dense stores
  // (compacted by the caller).  Returns the stratum's rounds (max over samples).
  int run_tile(TilePlan& P, const std::vector<int>& prel, bool& cap) {
    const int B = batch_cur;
    for (int i = 0; i < P.nrel; ++i) {  // external relations -> dense per-sample arrays
      TileRel& T = P.rel[i];
      const int r = prel[i];
      RelState& S = *rels[r];
      if (T.local) {
        S.dense = true;
        S.direct = false;
        S.lazy = false;
        S.nslots = (int64_t)1 << S.L.total;
        if (semi == S_UNIT) S.dfbits.reserve((S.nslots + 31) / 32);
        else S.dfp.reserve(S.nslots);
        launch_dense_fill(S.dfp.ptr(), S.dfbits.ptr(), S.nslots, semi, st);
        T.dfp = semi == S_UNIT ? nullptr : S.dfp.ptr();
        T.dfbits = semi == S_UNIT ? S.dfbits.ptr() : nullptr;
        for (int c = 0; c < T.ncols; ++c) T.pshift[c] = (uint8_t)S.L.shift[c];
        T.psshift = (uint8_t)S.L.sshift;
        continue;
      }
      ensure_sorted(S);
      const int64_t ns = T.shared ? 1 : B;
      const int64_t nbw = (T.D + 31) / 32;
      int64_t nf = 0;
      for (int c = 0; c < T.ncols; ++c) nf += T.nfib[c];
      const size_t bytes = (size_t)ns * ((semi == S_UNIT ? 0 : (size_t)T.D * 4) + nbw * 4 + nf * 8);
      uint8_t* base = reinterpret_cast<uint8_t*>(arena.alloc(bytes));
      cuda_check(cudaMemsetAsync(base, 0, bytes, st), "memset");
      size_t o = 0;
      for (int c = 0; c < T.ncols; ++c) {
        T.fib[c] = T.nfib[c] ? reinterpret_cast<const unsigned long long*>(base + o) : nullptr;
        o += (size_t)ns * T.nfib[c] * 8;
      }
      T.bits = reinterpret_cast<const uint32_t*>(base + o);
      o += (size_t)ns * nbw * 4;
      T.tag = semi == S_UNIT ? nullptr : reinterpret_cast<const float*>(base + o);
      TileScatter sc{};
      sc.key = S.key.ptr();
      sc.p = semi == S_UNIT ? nullptr : S.p.ptr();
      sc.n = S.n;
      sc.has_sample = S.L.has_sample ? 1 : 0;
      sc.sshift = (uint8_t)S.L.sshift;
      sc.sbits = (uint8_t)S.L.sbits;
      sc.ncols = T.ncols;
      for (int c = 0; c < T.ncols; ++c) {
        sc.shift[c] = (uint8_t)S.L.shift[c];
        sc.bits[c] = (uint8_t)S.L.bits[c];
      }
      sc.rel = T;
      launch_tile_scatter(sc, st);
      stats.bytes_algorithmic += S.n * (8 + (semi == S_UNIT ? 0 : 4));
    }
    // [max rounds, cap hit, tuples of each local relation (u64), rounds per sample...]
    int* d = arena.get<int>(B + 2 + 2 * TILE_MAXREL);
    cuda_check(cudaMemsetAsync(d, 0, 8 + 8 * TILE_MAXREL, st), "memset");
    P.counts = reinterpret_cast<unsigned long long*>(d + 2);
    std::vector<uint32_t> htr;
    if (getenv("LOBSTER_TILE_TRACE")) {  // debug: per (sample, round) candidates and |Δ'|
      P.trace = arena.get<uint32_t>((int64_t)B * 256);
      cuda_check(cudaMemsetAsync(P.trace, 0, (size_t)B * 256 * 4, st), "memset");
    }
    {
      Phase ph(this, 0);
      if (!hplan) cuda_check(cudaMallocHost(&hplan, sizeof(TilePlan)), "cudaMallocHost");
      *hplan = P;  // pinned staging: the plan's H2D copy stays asynchronous (the previous one completed at its sync)
      launch_tile_fixpoint(*hplan, reinterpret_cast<TilePlan*>(arena.alloc(sizeof(TilePlan))),
                           d + 2 + 2 * TILE_MAXREL, d_ncand, d + 1, st);
      kcheck("tile fixpoint");
    }
    if (P.trace) {
      htr.resize((size_t)B * 256);
      cuda_check(cudaMemcpyAsync(htr.data(), P.trace, htr.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
      sync();
      for (int s = 0; s < B; ++s) {
        fprintf(stderr, "[tile] sample %d:", s);
        for (int r = 1; r < 64 && (htr[(s * 64 + r) * 4] || htr[(s * 64 + r) * 4 + 1]); ++r)
          fprintf(stderr, " r%d c%u d%u", r, htr[(s * 64 + r) * 4], htr[(s * 64 + r) * 4 + 1]);
        fprintf(stderr, "\n[tile] sample %d U phase / longest item (x16 cycles):", s);
        for (int r = 1; r < 64 && htr[(s * 64 + r) * 4 + 3]; ++r)
          fprintf(stderr, " r%d %u/%u", r, htr[(s * 64 + r) * 4 + 3], htr[(s * 64 + r) * 4 + 2]);
        fprintf(stderr, "\n");
      }
    }
    launch_max_i32(d + 2 + 2 * TILE_MAXREL, B, d, st);
    cuda_check(cudaMemcpyAsync(hbuf, d, 8 + 8 * TILE_MAXREL, cudaMemcpyDeviceToHost, st), "D2H");
    sync();
    const int* h = reinterpret_cast<const int*>(hbuf);
    cap = h[1] != 0;
    for (int li = 0; li < P.nlocal; ++li)  // exact tuple counts: compaction needs no second read
      rels[prel[P.local_rel[li]]]->n = (int64_t)reinterpret_cast<const unsigned long long*>(h + 2)[li];
    return h[0];
  }

  int64_t run_strata() {
    int64_t round_cap_hit = 0;
    for (size_t si = 0; si < prog.strata.size(); ++si) {
      const std::vector<int>& strat = prog.strata[si];
      std::set<int> local(strat.begin(), strat.end());
      if (top1) top1_begin_stratum(strat);
      TilePlan tplan;
      std::vector<int> tprel;
      const bool tiled = tile_plan(strat, tplan, tprel);
      for (int r : strat) {
        RelState& S = *rels[r];
        S.n = S.nd = S.no = S.nc = 0;
        S.key.reserve(1);
        if (semi != S_UNIT) S.p.reserve(1);
        if (semi == S_MAXMULT) S.w.reserve(1);
        HostTimer hts(host_ms[4]);
        if (!tiled) choose_store(S, r);
      }
      mark("store setup");
      int rounds = 0;
      bool first = true, first_round = true, async = false;
      int64_t done = 0;
      std::deque<std::pair<int, uint32_t>> pending;  // (round, ring sequence)
      timed_rounds.clear();
      const size_t trace_base = trace.size();
      async_nd0 = 0;
      if (tiled) {  // the whole stratum in one launch (k_tile.cu)
        bool cap = false;
        rounds = run_tile(tplan, tprel, cap);
        stats.tile_strata++;
        if (cap) round_cap_hit = 1;
      }
      for (; !tiled;) {
        if (rounds >= max_iters) {
          if (async && (done = drain_async(pending, trace_base, true)) > 0) { rounds = (int)done; break; }
          round_cap_hit = 1;
          break;
        }
        rounds++;
        cur_round = rounds;
        arena.reset();
        const int64_t probe0 = stats.fj_probe_rows;
        if (log_level >= 2) trace.push_back({(int64_t)ev.size(), 0, 0, (int64_t)si});
        round_fused = round_other = 0;
        HostTimer ht_rules(host_ms[1]);
        for (const Rule& R : prog.rules) {
          if (!local.count(R.head_rel)) continue;
          std::vector<int> lpos;
          for (int k = 0; k < (int)R.body.size(); ++k)
            if (local.count(R.body[k].rel)) lpos.push_back(k);
          if (lpos.empty()) {
            if (!first) continue;
            std::vector<Version> ver(R.body.size(), V_EXT);
            // start: a batched atom covering every variable (the rest become
            // point lookups: no intermediate), else the smallest batched atom
            int start = -1;
            int64_t best = INT64_MAX;
            for (int pass = 0; pass < 2 && start < 0; ++pass)
              for (int k = 0; k < (int)R.body.size(); ++k) {
                if (prog.rels[R.body[k].rel].shared) continue;
                if (pass == 0 && !(R.body.size() >= 2 && covers_rule(R, k))) continue;
                int64_t n = rels[R.body[k].rel]->n;
                if (n < best) { best = n; start = k; }
              }
            eval_rule(R, ver, start);
            continue;
          }
          if (first) continue;
          for (size_t j = 0; j < lpos.size(); ++j) {
            std::vector<Version> ver(R.body.size(), V_EXT);
            for (size_t q = 0; q < lpos.size(); ++q)
              ver[lpos[q]] = q == j ? V_DELTA : (q < j ? V_NEW : V_OLD);
            eval_rule(R, ver, lpos[j]);
          }
        }
        ht_rules.stop();
        first = false;
        int64_t changed = 0;
        {
          HostTimer ht(host_ms[2]);
          if (async) {  // this round's |Δ'| words (zero-copy ring entry per relation)
            ++ring_seq;
            for (size_t q = 0; q < strat.size(); ++q) {
              rels[strat[q]]->ring_dst = dring + (ring_seq % ARING) * AREL + q;
              rels[strat[q]]->ring_seq = ring_seq;
            }
          }
          for (int r : strat) changed += settle(r);
          if (xfer) changed = part_sum(changed);  // Σ|Δ'| over every rank (Alg. 1's test, globally)
          if (top1) top1_commit(strat);
        }
        if (async) {  // |Δ'| of this round -> pinned ring; poll earlier rounds without stalling the GPU
          pending.push_back({rounds, ring_seq});
          if ((done = drain_async(pending, trace_base, false)) > 0) { rounds = (int)done; break; }
          continue;
        }
        if (log_level >= 2) { trace.back()[1] = stats.fj_probe_rows - probe0; trace.back()[2] = changed; }
        if (changed == 0) break;
        if (first_round) {  // C4-shaped strata continue as a bit-sliced frontier (k_slice.cu)
          std::vector<SliceRule> srules;
          if (slice_ok(strat, srules)) {
            mark("seed round");
            rounds += run_sliced(*rels[strat[0]], srules);
            if (round_cap_hit_slice) round_cap_hit = 1;
            async = false;
            break;
          }
        }
        // every recursive rule took the fused direct join in this (non-seed) round: later
        // rounds need no host-side sizes, so they are issued without a sync (lagged stop test)
        if (first_round) mark("seed round");
        if (!first_round && round_other == 0 && round_fused > 0 && strat.size() <= (size_t)AREL && async_ok(strat)) {
          mark("sync rounds");
          async = true;
          sections.push_back({get_event(), nullptr, ev.size(), 0});
          cudaEventRecord(sections.back().a, st);
          async_nrel = (int)strat.size();
          for (int r : strat) rels[r]->async = true;
          for (int r : strat) async_nd0 += rels[r]->nd;
        }
        first_round = false;
      }
      mark(async ? "async rounds" : "sync rounds");
      if (async) {
        sections.back().b = get_event();
        cudaEventRecord(sections.back().b, st);
        sections.back().ev1 = ev.size();
        sync();
        if (log_level >= 2 && trace.size() > trace_base + rounds) trace.resize(trace_base + rounds);
        for (int r : strat) {
          rels[r]->async = false;
          rels[r]->nd = 0;
        }
        pending.clear();
      }
      HostTimer ht(host_ms[3]);
      // Finished direct stores are compacted on first use (ensure_sorted): a lookup
      // chain can probe the slot words directly, so e.g. C2's `path` (64M tuples)
      // is never copied out unless an output or a sorted index asks for it.
      for (int r : strat) {
        RelState& S = *rels[r];
        if (!S.dense) continue;
        if (S.direct && !eager_compact) {
          unsigned long long* c = arena.get<unsigned long long>(1);
          cuda_check(cudaMemsetAsync(c, 0, 8, st), "memset");
          launch_direct_count(S.dirf.get(), S.nslots, semi, c, st);
          kcheck("direct count");
          S.n = (int64_t)read_dev(c);
          S.lazy = true;
        } else {
          dense_to_sorted(S, tiled ? S.n : -1);
        }
      }
      mark("dense->sorted");
      if (xfer && !round_cap_hit)  // later strata read this stratum's relations whole
        for (int r : strat)
          if (read_later(r, si)) part_gather(*rels[r]);
      if (!prog.rels[strat[0]].internal) {  // __eval<k> strata are an implementation detail
        stats.rounds_total += rounds;
        stats.strata++;
      }
      if (round_cap_hit) break;
    }
    return round_cap_hit;
  }

  void finish_run(cudaEvent_t t0, int64_t round_cap_hit, lobster_run_stats* out, bool counters = false) {
    cudaEvent_t t1 = get_event();
    cudaEventRecord(t1, st);
    sync();
    if (counters) {  // run(): d_ncand was copied to hbuf before t1
      const unsigned long long* c = reinterpret_cast<const unsigned long long*>(hbuf);
      stats.fj_timed_candidates = (int64_t)c[2];
      stats.fj_candidates = (int64_t)c[1] + stats.fj_timed_candidates;
      stats.candidates += (int64_t)c[0] + stats.fj_candidates;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    stats.ms_total = ms;
    std::vector<float> evms(ev.size(), 0.0f);
    for (size_t q = 0; q < ev.size(); ++q) {
      auto& e = ev[q];
      float m = 0;
      cudaEventElapsedTime(&m, e.second.first, e.second.second);
      evms[q] = m;
      switch (e.first) {
        case 0: stats.ms_join += m; break;
        case 1: stats.ms_sort += m; break;
        case 2: stats.ms_reduce += m; break;
        case 3: stats.ms_merge += m; break;
        case 5:  // timed fused joins (every join_timing_every-th launch)
          stats.ms_fused_join += m;
          break;
        case 6: stats.ms_comm += m; break;  // key-partitioned exchange
        default: stats.ms_grad += m; break;
      }
    }
    // phase total of the fused joins: the timed launches scaled to all launches
    if (stats.fj_timed_launches)
      stats.ms_join += stats.ms_fused_join * (double)stats.fj_launches / (double)stats.fj_timed_launches;
    for (const Section& sc : sections) {  // async rounds: settle = span - fused joins
      if (!sc.b || log_level >= 2) continue;  // (LOBSTER_LOG=2 times every settle itself)
      float span = 0;
      cudaEventElapsedTime(&span, sc.a, sc.b);
      double joins = 0;
      for (size_t q = sc.ev0; q < sc.ev1 && q < ev.size(); ++q)
        if (ev[q].first == 5) joins += evms[q];
      // only every k-th join carries events: the section's join time is estimated as k x
      stats.ms_merge += std::max(0.0, (double)span - joins * join_timing_every);
    }
    sections.clear();
    if (log_level >= 1 && marks.size() > 1) {  // GPU timeline sections (includes idle gaps)
      std::string line = "[lobster] timeline ms:";
      for (size_t q = 1; q < marks.size(); ++q) {
        float m = 0;
        cudaEventElapsedTime(&m, marks[q - 1].second, marks[q].second);
        char b[96];
        snprintf(b, sizeof b, " %s %.2f |", marks[q].first, m);
        line += b;
      }
      fprintf(stderr, "%s\n", line.c_str());
    }
    if (log_level >= 2) {  // per-round trace: probe rows, |Δ'|, GPU ms of join / settle phases
      for (size_t t = 0; t < trace.size(); ++t) {
        const size_t e0 = (size_t)trace[t][0], e1 = t + 1 < trace.size() ? (size_t)trace[t + 1][0] : ev.size();
        double pj = 0, pm = 0;
        for (size_t q = e0; q < e1 && q < ev.size(); ++q) {
          float m = 0;
          cudaEventElapsedTime(&m, ev[q].second.first, ev[q].second.second);
          if (ev[q].first == 0 || ev[q].first == 5) pj += m; else pm += m;
        }
        fprintf(stderr, "[lobster] round %4zu stratum %lld probe %10lld delta' %10lld join %8.1f us settle %8.1f us\n", t,
                (long long)trace[t][3], (long long)trace[t][1], (long long)trace[t][2], pj * 1e3, pm * 1e3);
      }
    }
    trace.clear();
    ran = true;
    arena.reset();
    if (log_level >= 1)
      fprintf(stderr,
              "[lobster] run: %.2f ms (events) | host: ingest %.2f, rules %.2f, settle %.2f, dense->sorted %.2f | "
              "store setup %.2f (memgetinfo %.2f), gradients %.2f | phases: join %.2f (fused %.2f), sort %.2f, reduce %.2f, merge %.2f, grad %.2f | rounds %d\n",
              stats.ms_total, host_ms[0], host_ms[1], host_ms[2], host_ms[3], host_ms[4], host_ms[6], host_ms[5], stats.ms_join, stats.ms_fused_join,
              stats.ms_sort, stats.ms_reduce, stats.ms_merge, stats.ms_grad, stats.rounds_total);
    if (out) *out = stats;
    if (round_cap_hit) throw Failure(LOBSTER_E_ITER_CAP, "max_iters rounds reached");
  }

  // per relation, its rules in local order: how a (head key, witness) names
  // the body tuples of the derivation (witness walk, top-1-proof unions)
  void build_walk_rules(std::vector<WalkRule>& ordered, std::vector<int>& base) {
    const int nr = (int)prog.rels.size();
    base.assign(nr, 0);
    {
      std::vector<int> cnt(nr, 0);
      for (auto& R : prog.rules) cnt[R.head_rel]++;
      int acc = 0;
      for (int r = 0; r < nr; ++r) { base[r] = acc; acc += cnt[r]; }
    }
    ordered.assign(prog.rules.size(), WalkRule{});
    for (auto& R : prog.rules) {
      WalkRule wrl;
      std::memset(&wrl, 0, sizeof(wrl));
      wrl.natoms = (int)R.body.size();
      for (int a = 0; a < wrl.natoms; ++a) {
        wrl.atom[a].rel = R.body[a].rel;
        wrl.atom[a].ncols = (int)R.body[a].args.size();
        for (int c = 0; c < wrl.atom[a].ncols; ++c) {
          wrl.atom[a].var[c] = (int8_t)R.body[a].args[c].var;
          wrl.atom[a].cst[c] = R.body[a].args[c].cst;
        }
      }
      wrl.nvars = (int)R.var_names.size();
      for (int v = 0; v < 16; ++v) { wrl.head_col[v] = -1; wrl.wfield[v] = -1; }
      for (size_t c = 0; c < R.head.size(); ++c)
        if (R.head[c].is_var() && wrl.head_col[R.head[c].var] < 0) wrl.head_col[R.head[c].var] = (int8_t)c;
      for (size_t i = 0; i < R.nonhead.size(); ++i) {
        int v = R.nonhead[i];
        wrl.wfield[v] = (int8_t)i;
        wrl.wshift[v] = (uint8_t)wshift[R.global_index][i];
        wrl.wbits[v] = (uint8_t)wbits[R.global_index][i];
        wrl.wmin[v] = (int32_t)class_min[R.var_class[v]];
      }
      ordered[base[R.head_rel] + R.local_index] = wrl;
    }
  }

  // ------------------------------------------- diff-add-mult: adjoint program
  // Reverse mode over the final relations.  For an output relation O (arity k)
  // every relation X it depends on gets an adjoint __adj_X(o1..ok, x...) =
  // ∂O(o)/∂tag(X(x)); for each rule H(h) :- B1, .., Bn and each atom j:
  //   __adj_Bj(o, bj) :- __adj_H(o, h), __fwd_B1, .., (no Bj), .., __fwd_Bn, __dom_Bj(bj), filters
  // (__fwd_X: X's final tuples and tags; __dom_X: the same tuples, tag 1, so
  // every variable of Bj is bound and only existing tuples get adjoints), seeded
  // by __adj_O(o, o) = 1, and the input facts read their entries through
  //   __grad(o, f) :- __adj_E(o, e), __fid_E(e, f)
  // (duplicate facts are ⊕-merged by +, so each gets ∂ = 1 · adjoint).  The
  // program is evaluated by a child context under add-mult on this stream:
  // the same kernels, no CPU path.  On finite derivation sets the adjoint sums
  // equal the dual-number derivative of the add-mult result.
  static constexpr const char* kRelText[6] = {" == ", " != ", " < ", " <= ", " > ", " >= "};
  static std::string cols_decl(int n, const char* pfx) {
    std::string t;
    for (int c = 0; c < n; ++c) t += (c ? ", " : "") + std::string(pfx) + std::to_string(c) + ": i32";
    return t;
  }
  std::string term_text(const Rule& R, const Term& t) const {
    return t.is_var() ? R.var_names[t.var] : std::to_string(t.cst);
  }
  static std::string join_args(const std::vector<std::string>& v) {
    std::string t;
    for (size_t i = 0; i < v.size(); ++i) t += (i ? ", " : "") + v[i];
    return t;
  }
  std::string adjoint_program(int O, std::vector<int>& deps) const {
    const int nr = (int)prog.rels.size();
    std::vector<char> in(nr, 0);
    in[O] = 1;
    for (bool grew = true; grew;) {  // relations O depends on
      grew = false;
      for (const Rule& R : prog.rules)
        if (in[R.head_rel])
          for (auto& a : R.body)
            if (!in[a.rel]) in[a.rel] = grew = true;
    }
    deps.clear();
    for (int r = 0; r < nr; ++r)
      if (in[r]) deps.push_back(r);
    const int k = prog.rels[O].arity;
    std::vector<std::string> ov;
    for (int c = 0; c < k; ++c) ov.push_back("__o" + std::to_string(c));
    auto with_o = [&](const std::vector<std::string>& rest) {
      std::vector<std::string> v = ov;
      v.insert(v.end(), rest.begin(), rest.end());
      return join_args(v);
    };
    auto atom_args = [&](const Rule& R, const std::vector<Term>& ts) {
      std::vector<std::string> v;
      for (auto& t : ts) v.push_back(term_text(R, t));
      return v;
    };
    std::string t = "type __seed(" + cols_decl(k, "c") + ")\n";
    for (int r : deps) {
      const Relation& X = prog.rels[r];
      const std::string sh = X.shared ? "shared " : "";
      t += sh + "type __fwd_" + X.name + "(" + cols_decl(X.arity, "c") + ")\n";
      t += sh + "type __dom_" + X.name + "(" + cols_decl(X.arity, "c") + ")\n";
      if (X.input) t += sh + "type __fid_" + X.name + "(" + cols_decl(X.arity + 1, "c") + ")\n";
    }
    // seed: ∂O(o)/∂O(x) = [o == x]
    t += "rel __adj_" + prog.rels[O].name + "(" + with_o(ov) + ") :- __seed(" + join_args(ov) + ").\n";
    for (const Rule& R : prog.rules) {
      if (!in[R.head_rel]) continue;
      const std::vector<std::string> hargs = atom_args(R, R.head);
      for (size_t j = 0; j < R.body.size(); ++j) {
        const BodyAtom& Bj = R.body[j];
        const std::vector<std::string> bargs = atom_args(R, Bj.args);
        std::string body = "__adj_" + prog.rels[R.head_rel].name + "(" + with_o(hargs) + ")";
        for (size_t i = 0; i < R.body.size(); ++i)
          if (i != j)
            body += ", __fwd_" + prog.rels[R.body[i].rel].name + "(" + join_args(atom_args(R, R.body[i].args)) + ")";
        body += ", __dom_" + prog.rels[Bj.rel].name + "(" + join_args(bargs) + ")";
        for (const Compare& cp : R.cmps)
          body += ", " + term_text(R, cp.a) + kRelText[cp.rel] + term_text(R, cp.b);
        t += "rel __adj_" + prog.rels[Bj.rel].name + "(" + with_o(bargs) + ") :- " + body + ".\n";
      }
    }
    for (int r : deps) {
      const Relation& X = prog.rels[r];
      if (!X.input) continue;
      std::vector<std::string> e;
      for (int c = 0; c < X.arity; ++c) e.push_back("__e" + std::to_string(c));
      std::vector<std::string> ef = e;
      ef.push_back("__f");
      t += "rel __grad(" + with_o({"__f"}) + ") :- __adj_" + X.name + "(" + with_o(e) + "), __fid_" + X.name + "(" +
           join_args(ef) + ").\n";
    }
    return t;
  }

  // relation r's stored tuples unpacked (sample ids local to the batch, columns SoA)
  void unpack_local(RelState& S, int r, int32_t* sid, int32_t* cols) {
    ensure_sorted(S);
    const int ar = prog.rels[r].arity;
    uint8_t* dsh = arena.get<uint8_t>(3 * 8 + 64);
    std::vector<uint8_t> hb(16 + 32, 0);
    for (int c = 0; c < ar; ++c) { hb[c] = (uint8_t)S.L.shift[c]; hb[8 + c] = (uint8_t)S.L.bits[c]; }
    std::memcpy(hb.data() + 16, S.L.mins.data(), ar * 4);
    cuda_check(cudaMemcpyAsync(dsh, hb.data(), hb.size(), cudaMemcpyHostToDevice, st), "H2D");
    launch_unpack(S.key.ptr(), S.n, S.L.has_sample, (uint8_t)S.L.sshift, ar, dsh, dsh + 8,
                  reinterpret_cast<int32_t*>(dsh + 16), sid, cols, st);
    kcheck("unpack");
  }

  void dadd_gradients() {
    for (int O = 0; O < (int)prog.rels.size(); ++O) {
      const Relation& OR = prog.rels[O];
      if (!OR.output || OR.input) continue;
      std::vector<int> deps;
      const std::string text = adjoint_program(O, deps);
      if (log_level >= 2) fprintf(stderr, "[lobster] adjoint program of %s:\n%s", OR.name.c_str(), text.c_str());
      lobster_options o = opt;
      o.batch_size = batch_cur;
      o.world_size = 1;
      o.rank = 0;
      o.micro_batch = 0;
      o.arena_bytes = 0;
      std::unique_ptr<Ctx> ch(new Ctx());
      ch->create(&o);
      ch->unbounded_tags = true;
      ch->load(text.c_str(), LOBSTER_ADD_MULT_PROB);
      int64_t first = 0;
      auto push = [&](const std::string& name, int64_t n, int ar, const int32_t* cols, const int32_t* sid,
                      const float* p) {
        std::vector<const int32_t*> cp(std::max(ar, 1), nullptr);
        for (int c = 0; c < ar; ++c) cp[c] = cols + (int64_t)c * n;
        ch->push(name.c_str(), n, cp.data(), sid, p, &first);
      };
      for (int r : deps) {
        RelState& X = *rels[r];
        const Relation& XR = prog.rels[r];
        const int64_t n = (ensure_sorted(X), X.n);
        int32_t* sid = arena.get<int32_t>(n);
        int32_t* cols = arena.get<int32_t>(std::max<int64_t>(1, (int64_t)XR.arity * n));
        unpack_local(X, r, sid, cols);
        push("__fwd_" + XR.name, n, XR.arity, cols, XR.shared ? nullptr : sid, X.p.ptr());
        push("__dom_" + XR.name, n, XR.arity, cols, XR.shared ? nullptr : sid, nullptr);
        if (r == O) push("__seed", n, XR.arity, cols, sid, nullptr);  // O's tuples, tag 1
        if (XR.input) {  // every pushed fact with its id (duplicates included)
          const int64_t m = X.in.n;
          int32_t* fc = arena.get<int32_t>(std::max<int64_t>(1, (int64_t)(XR.arity + 1) * m));
          for (int c = 0; c < XR.arity && m; ++c)
            cuda_check(cudaMemcpyAsync(fc + (int64_t)c * m, X.in.cols[c].ptr(), m * 4, cudaMemcpyDeviceToDevice, st), "fid");
          if (m) cuda_check(cudaMemcpyAsync(fc + (int64_t)XR.arity * m, X.in.fid.ptr(), m * 4, cudaMemcpyDeviceToDevice, st), "fid");
          push("__fid_" + XR.name, m, XR.arity + 1, fc, XR.shared ? nullptr : X.in.sid.ptr(), nullptr);
        }
      }
      ch->run(nullptr);
      lobster_output g{};
      const auto git = ch->prog.rel_id.find("__grad");
      RelState& S = *rels[O];
      const int k = OR.arity;
      const int64_t n = S.n;
      S.goff.reserve(n + 1);
      if (git == ch->prog.rel_id.end() || !n) {  // no input facts reach O
        cuda_check(cudaMemsetAsync(S.goff.ptr(), 0, (n + 1) * 8, st), "memset");
        S.ng = 0;
        S.gfid.reserve(1);
        S.gval.reserve(1);
      } else {
        ch->output_get("__grad", 1, &g);
        int32_t* osid = arena.get<int32_t>(n);
        int32_t* ocols = arena.get<int32_t>(std::max<int64_t>(1, (int64_t)k * n));
        unpack_local(S, O, osid, ocols);
        S.ng = g.n;
        S.gfid.reserve(std::max<int64_t>(1, g.n));
        S.gval.reserve(std::max<int64_t>(1, g.n));
        launch_grad_rows(osid, ocols, n, k, g.sample_ids, g.columns[0], g.n, S.goff.ptr(), st);
        launch_widen_i32(g.columns[k], g.n, S.gfid.ptr(), st);
        if (g.n) cuda_check(cudaMemcpyAsync(S.gval.ptr(), g.probs, g.n * 4, cudaMemcpyDeviceToDevice, st), "grad");
        kcheck("adjoint rows");
      }
      sync();  // the child's buffers are released with it
      S.has_grad = true;
      stats.candidates += ch->stats.candidates;
    }
  }

  // --------------------------------------------------------- gradients (A11)
  void gradients() {
    if (top1) return top1_gradients();
    if (dadd) return dadd_gradients();
    const int nr = (int)prog.rels.size();
    for (int r = 0; r < nr; ++r)  // walks start from the output relations' sorted rows
      if (prog.rels[r].output) ensure_sorted(*rels[r]);
    std::vector<WalkRel> wr(nr);
    for (int r = 0; r < nr; ++r) {
      RelState& S = *rels[r];
      WalkRel& w = wr[r];
      std::memset(&w, 0, sizeof(w));
      w.key = S.key.ptr();
      w.p = S.p.ptr();
      w.w = S.w.ptr();
      w.fid = S.fid.ptr();
      if (prog.rels[r].input) {  // an index aliasing the rows, with CSR offsets: O(1) + a short scan
        for (auto& kv : static_idx) {
          const Index& ix = *kv.second;
          if (kv.first.first != r || ix.key != S.key.ptr() || !ix.offp || ix.maxdeg < 0 || ix.maxdeg > 64) continue;
          w.off = ix.offp;
          w.nprefix = ix.nprefix;
          w.pshift = ix.free_bits;
          break;
        }
      }
      if (S.direct && semi == S_MAXMULT) {  // O(1) hops through the store's final words
        w.dir = reinterpret_cast<const unsigned long long*>(S.dirf.get());
        w.wmask = mx_wmask(S);
        w.wT = S.wT;
        w.wrb = S.wrb;
      }
      w.n = S.n;
      w.input = prog.rels[r].input ? 1 : 0;
      w.has_sample = S.L.has_sample ? 1 : 0;
      w.sshift = (uint8_t)S.L.sshift;
      w.ncols = prog.rels[r].arity;
      for (int c = 0; c < w.ncols; ++c) {
        w.shift[c] = (uint8_t)S.L.shift[c];
        w.bits[c] = (uint8_t)S.L.bits[c];
        w.min[c] = S.L.mins[c];
      }
    }
    std::vector<WalkRule> ordered;
    std::vector<int> base;
    build_walk_rules(ordered, base);
    WalkRel* d_rels = arena.get<WalkRel>(nr);
    WalkRule* d_rules = arena.get<WalkRule>((int64_t)ordered.size());
    int* d_base = arena.get<int>(nr);
    int* d_rb = arena.get<int>(nr);
    int* d_err = arena.get<int>(1);
    cuda_check(cudaMemcpyAsync(d_rels, wr.data(), nr * sizeof(WalkRel), cudaMemcpyHostToDevice, st), "H2D");
    if (!ordered.empty())
      cuda_check(cudaMemcpyAsync(d_rules, ordered.data(), ordered.size() * sizeof(WalkRule), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(d_base, base.data(), nr * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(d_rb, rule_bits.data(), nr * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemsetAsync(d_err, 0, sizeof(int), st), "memset");
    WalkTables T{d_rels, d_rules, d_base, d_rb, nr};
    for (int r = 0; r < nr; ++r) {
      if (!prog.rels[r].output || prog.rels[r].input) continue;
      RelState& S = *rels[r];
      const int64_t n = S.n;
      S.goff.reserve(n + 1);
      if (n == 0) {
        cuda_check(cudaMemsetAsync(S.goff.ptr(), 0, 8, st), "memset");
        S.ng = 0;
        S.has_grad = true;
        continue;
      }
      int64_t* cnt = arena.get<int64_t>(n);
      int64_t* loff = arena.get<int64_t>(n + 1);
      // Proofs whose pending IDB atoms outgrow the in-register stack (deep
      // non-linear trees; linear recursion never does) are re-walked with a
      // global spill region per thread, doubling it until every stack fits.
      uint64_t* gkey = nullptr;
      int* grel = nullptr;
      int64_t gcap = 0, gthreads = 0;
      auto free_spill = [&]() {
        if (gkey) cudaFreeAsync(gkey, st);
        if (grel) cudaFreeAsync(grel, st);
        gkey = nullptr;
        grel = nullptr;
      };
      int64_t nleaf = 0;
      for (;;) {
        launch_walk(T, r, n, 0, nullptr, cnt, nullptr, d_err, gkey, grel, gcap, gthreads, st);
        exclusive_scan<int64_t>(cnt, loff, n, loff + n, arena.alloc(scan_tmp_bytes<int64_t>(n)), st);
        kcheck("walk");
        nleaf = read_dev(loff + n);
        const int e = read_dev(d_err);
        if (e == 0) break;
        if (e & ~2) { free_spill(); throw Failure(LOBSTER_E_CUDA, "witness walk failed (code " + std::to_string(e) + ")"); }
        free_spill();
        gcap = gcap ? 2 * gcap : 1024;
        gthreads = std::min<int64_t>(n, 148 * 64);
        while (gthreads > 148 && gthreads * gcap * 12 > ((int64_t)1 << 30)) gthreads /= 2;
        if (gthreads * gcap * 12 > ((int64_t)4 << 30)) {
          throw Failure(LOBSTER_E_RANGE, "witness walk: a proof needs more than " + std::to_string(gcap / 2) +
                                             " pending IDB atoms");
        }
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&gkey), gthreads * gcap * 8, st), "walk spill");
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&grel), gthreads * gcap * 4, st), "walk spill");
        cuda_check(cudaMemsetAsync(d_err, 0, sizeof(int), st), "memset");
      }
      uint64_t* k0 = arena.get<uint64_t>(nleaf);
      uint64_t* k1 = arena.get<uint64_t>(nleaf);
      launch_walk(T, r, n, 1, loff, nullptr, reinterpret_cast<int64_t*>(k0), d_err, gkey, grel, gcap, gthreads, st);
      free_spill();
      // leaf keys: tuple << 32 | fact, sorted -> unique (tuple, fact) runs
      tag_leaves(k0, loff, n, nleaf);
      const int tbits = 32 + bits_for((uint64_t)n);
      int which = radix_sort<uint64_t, void>(k0, nullptr, k1, nullptr, nleaf, tbits, arena.alloc(sort_tmp_bytes(nleaf)), st);
      uint64_t* ks = which ? k1 : k0;
      if (omin) {
        S.gfid.reserve(n);
        S.gval.reserve(n);
        launch_grad_onehot(ks, nleaf, fact_p.ptr(), n, loff, S.goff.ptr(), S.gfid.ptr(), S.gval.ptr(), st);
        kcheck("grad one-hot");
        S.ng = n;
        S.has_grad = true;
        continue;
      }
      uint32_t* fl = arena.get<uint32_t>(nleaf);
      uint32_t* pos = arena.get<uint32_t>(nleaf);
      uint32_t* tot = arena.get<uint32_t>(1);
      launch_leaf_heads(ks, nleaf, fl, st);
      exclusive_scan<uint32_t>(fl, pos, nleaf, tot, arena.alloc(scan_tmp_bytes<uint32_t>(nleaf)), st);
      kcheck("leaf heads");
      const int64_t nuniq = read_dev(tot);
      S.gfid.reserve(nuniq);
      S.gval.reserve(nuniq);
      double* scratch = arena.get<double>(nuniq);
      launch_grad(ks, pos, nleaf, nuniq, fact_p.ptr(), n, loff, S.goff.ptr(), S.gfid.ptr(), S.gval.ptr(), scratch, st);
      kcheck("grad");
      S.ng = nuniq;
      S.has_grad = true;
    }
  }

  void tag_leaves(uint64_t* k, const int64_t* loff, int64_t n, int64_t nleaf);

  // ------------------------------------------------------------- outputs
  void output_get(const char* relname, int where, lobster_output* out) {
    if (!relname || !out) throw Failure(LOBSTER_E_INVALID_ARG, "NULL argument");
    if (where != 0 && where != 1) throw Failure(LOBSTER_E_INVALID_ARG, "where must be 0 (host) or 1 (device)");
    auto it = prog.rel_id.find(relname);
    if (it == prog.rel_id.end()) throw Failure(LOBSTER_E_INVALID_ARG, std::string("unknown relation ") + relname);
    if (!ran) throw Failure(LOBSTER_E_STATE, "output_get before a successful run");
    const int r = it->second;
    RelState& S = *rels[r];
    if (!S.retained)
      throw Failure(LOBSTER_E_INVALID_ARG, std::string("relation ") + relname +
                                               " was not retained by a micro-batched run (declare it `output`)");
    ensure_sorted(S);
    const int ar = prog.rels[r].arity;
    const int64_t n = S.n;
    if (!S.out_dev_ready) {
      S.o_sid.reserve(n);
      S.o_cols.reserve((int64_t)ar * n);
      S.o_soff.reserve(opt.batch_size + 1);
      uint8_t* dsh = arena.get<uint8_t>(3 * 8 + 64);
      std::vector<uint8_t> hb(16 + 32, 0);
      for (int c = 0; c < ar; ++c) { hb[c] = (uint8_t)S.L.shift[c]; hb[8 + c] = (uint8_t)S.L.bits[c]; }
      std::memcpy(hb.data() + 16, S.L.mins.data(), ar * 4);
      cuda_check(cudaMemcpyAsync(dsh, hb.data(), hb.size(), cudaMemcpyHostToDevice, st), "H2D");
      launch_unpack(S.key.ptr(), n, S.L.has_sample, (uint8_t)S.L.sshift, ar, dsh, dsh + 8,
                    reinterpret_cast<int32_t*>(dsh + 16), S.o_sid.ptr(), S.o_cols.ptr(), st);
      launch_sample_offsets(S.key.ptr(), n, opt.batch_size, (uint8_t)S.L.sshift, S.L.has_sample, S.o_soff.ptr(), st);
      if (sample_base && S.L.has_sample) launch_add_i32(S.o_sid.ptr(), n, sample_base, st);
      kcheck("unpack");
      sync();
      arena.reset();
      S.out_dev_ready = true;
    }
    std::memset(out, 0, sizeof(*out));
    out->n = n;
    out->arity = ar;
    out->on_device = where;
    if (where == 1) {
      S.col_ptrs.assign(ar, nullptr);
      for (int c = 0; c < ar; ++c) S.col_ptrs[c] = S.o_cols.ptr() + (int64_t)c * n;
      out->sample_ids = S.o_sid.ptr();
      out->columns = S.col_ptrs.data();
      out->probs = semi != S_UNIT ? S.p.ptr() : nullptr;
      out->sample_offsets = S.o_soff.ptr();
      if (S.has_grad) {
        out->grad_offsets = S.goff.ptr();
        out->grad_fact_ids = S.gfid.ptr();
        out->grad_values = S.gval.ptr();
      }
      return;
    }
    if (!S.out_host_ready) {
      S.h_sid.resize(n);
      S.h_cols.resize((size_t)ar * n);
      S.h_soff.resize(opt.batch_size + 1);
      if (n) {
        cuda_check(cudaMemcpyAsync(S.h_sid.data(), S.o_sid.ptr(), n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        if (ar) cuda_check(cudaMemcpyAsync(S.h_cols.data(), S.o_cols.ptr(), (size_t)ar * n * 4, cudaMemcpyDeviceToHost, st), "D2H");
      }
      cuda_check(cudaMemcpyAsync(S.h_soff.data(), S.o_soff.ptr(), (opt.batch_size + 1) * 8, cudaMemcpyDeviceToHost, st), "D2H");
      if (semi != S_UNIT) {
        S.h_p.resize(n);
        if (n) cuda_check(cudaMemcpyAsync(S.h_p.data(), S.p.ptr(), n * 4, cudaMemcpyDeviceToHost, st), "D2H");
      }
      if (S.has_grad) {
        S.h_goff.resize(n + 1);
        S.h_gfid.resize(S.ng);
        S.h_gval.resize(S.ng);
        cuda_check(cudaMemcpyAsync(S.h_goff.data(), S.goff.ptr(), (n + 1) * 8, cudaMemcpyDeviceToHost, st), "D2H");
        if (S.ng) {
          cuda_check(cudaMemcpyAsync(S.h_gfid.data(), S.gfid.ptr(), S.ng * 8, cudaMemcpyDeviceToHost, st), "D2H");
          cuda_check(cudaMemcpyAsync(S.h_gval.data(), S.gval.ptr(), S.ng * 4, cudaMemcpyDeviceToHost, st), "D2H");
        }
      }
      sync();
      S.out_host_ready = true;
    }
    S.col_ptrs.assign(ar, nullptr);
    for (int c = 0; c < ar; ++c) S.col_ptrs[c] = S.h_cols.data() + (size_t)c * n;
    out->sample_ids = S.h_sid.data();
    out->columns = S.col_ptrs.data();
    out->probs = semi != S_UNIT ? S.h_p.data() : nullptr;
    out->sample_offsets = S.h_soff.data();
    if (S.has_grad) {
      out->grad_offsets = S.h_goff.data();
      out->grad_fact_ids = S.h_gfid.data();
      out->grad_values = S.h_gval.data();
    }
  }

  void backward(const char* relname, const float* upstream, float* grad_facts) {
    if (!relname || !upstream || !grad_facts) throw Failure(LOBSTER_E_INVALID_ARG, "NULL argument");
    auto it = prog.rel_id.find(relname);
    if (it == prog.rel_id.end()) throw Failure(LOBSTER_E_INVALID_ARG, std::string("unknown relation ") + relname);
    if (!ran) throw Failure(LOBSTER_E_STATE, "backward before a successful run");
    RelState& S = *rels[it->second];
    if ((semi != S_MAXMULT && !dadd) || !S.has_grad)
      throw Failure(LOBSTER_E_INVALID_ARG, "no gradients for this relation");
    const int64_t nf = num_facts_db;
    cuda_check(cudaMemsetAsync(grad_facts, 0, nf * sizeof(float), st), "memset");
    const int64_t ng = S.ng;
    if (ng > 0) {
      uint64_t* k0 = arena.get<uint64_t>(ng);
      uint64_t* k1 = arena.get<uint64_t>(ng);
      uint32_t* v0 = arena.get<uint32_t>(ng);
      uint32_t* v1 = arena.get<uint32_t>(ng);
      launch_grad_contrib(S.goff.ptr(), S.gfid.ptr(), S.gval.ptr(), upstream, S.n, ng, k0, v0, st);
      int which = radix_sort(k0, v0, k1, v1, ng, bits_for((uint64_t)nf), arena.alloc(sort_tmp_bytes(ng)), st);
      launch_dense_sum(which ? k1 : k0, which ? v1 : v0, nullptr, ng, grad_facts, st);
      kcheck("backward");
    }
    sync();
    arena.reset();
  }
};

}  // namespace lob

// ============================================================================
// small kernels used only by the driver
// ============================================================================
namespace lob {
namespace {
__global__ void scatter_p_k(const int32_t* __restrict__ fid, const float* __restrict__ p, int64_t n,
                            float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[fid[i]] = p[i];
}
__global__ void tag_leaves_k(uint64_t* __restrict__ k, const int64_t* __restrict__ loff, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  for (int64_t i = loff[t]; i < loff[t + 1]; ++i) k[i] = ((uint64_t)t << 32) | (uint64_t)(uint32_t)k[i];
}
int gridn(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}
}  // namespace
void Ctx::scatter_fact_p(const int32_t* fid, const float* p, int64_t n) {
  if (n > 0) {
    note_launch();
    scatter_p_k<<<gridn(n), 256, 0, st>>>(fid, p, n, fact_p.ptr());
  }
  kcheck("scatter p");
}
void Ctx::tag_leaves(uint64_t* k, const int64_t* loff, int64_t n, int64_t nleaf) {
  (void)nleaf;
  if (n > 0) {
    note_launch();
    tag_leaves_k<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(k, loff, n);
  }
  kcheck("tag leaves");
}
}  // namespace lob

// ============================================================================
// C ABI
// ============================================================================
struct lobster_ctx {
  lob::Ctx c;
};

struct lobster_group {
  std::unique_ptr<lob::Xfer> x;
};

namespace {
template <typename F>
lobster_status guarded(lobster_ctx* ctx, F&& f) {
  if (!ctx) return LOBSTER_E_INVALID_ARG;
  try {
    f();
    ctx->c.err.clear();
    return LOBSTER_OK;
  } catch (lob::Failure& e) {
    ctx->c.err = e.what();
    if (e.code == LOBSTER_E_CUDA) ctx->c.sticky = true;
    return (lobster_status)e.code;
  } catch (std::exception& e) {
    ctx->c.err = e.what();
    return LOBSTER_E_INVALID_ARG;
  }
}
}  // namespace

extern "C" {

lobster_status lobster_create(const lobster_options* options, lobster_ctx** out) {
  if (!out) return LOBSTER_E_INVALID_ARG;
  *out = nullptr;
  lobster_ctx* ctx = nullptr;
  try {
    ctx = new lobster_ctx();
    ctx->c.create(options);
  } catch (lob::Failure& e) {
    delete ctx;
    return (lobster_status)e.code;
  } catch (std::exception&) {
    delete ctx;
    return LOBSTER_E_CUDA;
  }
  *out = ctx;
  return LOBSTER_OK;
}

void lobster_destroy(lobster_ctx* ctx) { delete ctx; }

const char* lobster_last_error(const lobster_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "NULL context"; }

lobster_status lobster_program_load(lobster_ctx* ctx, const char* text, lobster_semiring semiring) {
  return guarded(ctx, [&]() { ctx->c.load(text, (int)semiring); });
}

lobster_status lobster_facts_push(lobster_ctx* ctx, const char* relation, int64_t n, const int32_t* const* columns,
                                  const int32_t* sample_ids, const float* probs, int64_t* first_fact_id) {
  int64_t dummy = 0;
  return guarded(ctx, [&]() {
    ctx->c.push(relation, n, columns, sample_ids, probs, first_fact_id ? first_fact_id : &dummy);
  });
}

lobster_status lobster_run(lobster_ctx* ctx, lobster_run_stats* stats) {
  return guarded(ctx, [&]() { ctx->c.run(stats); });
}

lobster_status lobster_output_get(lobster_ctx* ctx, const char* relation, int32_t where, lobster_output* out) {
  return guarded(ctx, [&]() { ctx->c.output_get(relation, where, out); });
}

lobster_status lobster_output_backward(lobster_ctx* ctx, const char* relation, const float* upstream,
                                       float* grad_facts) {
  return guarded(ctx, [&]() { ctx->c.backward(relation, upstream, grad_facts); });
}

int64_t lobster_num_facts(const lobster_ctx* ctx) { return ctx ? ctx->c.next_fact : 0; }

lobster_status lobster_facts_groups(lobster_ctx* ctx, int64_t first_fact_id, int64_t n, const int32_t* group_ids) {
  return guarded(ctx, [&]() { ctx->c.set_groups(first_fact_id, n, group_ids); });
}

int64_t lobster_kernel_launches(void) { return lob::g_launches.load(); }

lobster_status lobster_group_local(int32_t world_size, lobster_group** out) {
  if (!out || world_size < 1 || world_size > 64) return LOBSTER_E_INVALID_ARG;
  *out = new lobster_group{std::unique_ptr<lob::Xfer>(new lob::LocalXfer(world_size))};
  return LOBSTER_OK;
}

lobster_status lobster_nccl_id(uint8_t* id) {
  if (!id) return LOBSTER_E_INVALID_ARG;
  try {
    lob::NcclXfer::unique_id(id);
  } catch (lob::Failure& e) {
    return (lobster_status)e.code;
  }
  return LOBSTER_OK;
}

lobster_status lobster_group_nccl(const uint8_t* id, int32_t rank, int32_t world_size, int32_t device,
                                  lobster_group** out) {
  if (!out || !id || world_size < 1 || world_size > 64 || rank < 0 || rank >= world_size) return LOBSTER_E_INVALID_ARG;
  try {
    *out = new lobster_group{std::unique_ptr<lob::Xfer>(new lob::NcclXfer(id, rank, world_size, device))};
  } catch (lob::Failure& e) {
    return (lobster_status)e.code;
  }
  return LOBSTER_OK;
}

void lobster_group_destroy(lobster_group* g) { delete g; }

lobster_status lobster_partition(lobster_ctx* ctx, lobster_group* group, int32_t rank) {
  return guarded(ctx, [&]() { ctx->c.set_partition(group ? group->x.get() : nullptr, rank); });
}

}  // extern "C"
