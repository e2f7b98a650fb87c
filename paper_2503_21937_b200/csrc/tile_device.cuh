// tile_device.cuh — device code of the one-launch small-domain strata (see
// k_tile.cu for the algorithm).  Include-free (needs tile_plan.h and the
// fixed-width integer types).  TILE_JIT selects a compile-time plan `kPlan`
// (every plan-driven loop unrolled, every field folded).  A run-time NVRTC
// specialisation built on it was measured and rejected: on C3 the unrolled
// kernel took 262 ms per step against 210 ms for this interpreted one (code
// growth; the enumeration's cost is its divergent mask work, not plan reads)
// and each plan took ~10 s to compile.
#pragma once

namespace lob {

#ifdef TILE_JIT
#define TP(F) ::lob::kPlan
#define TILE_UNROLL _Pragma("unroll")
#else
#define TP(F) (*(F).P)
#define TILE_UNROLL
#endif

template <int SEMI>
__device__ __forceinline__ float tile_otimes(float a, float b) {
  if constexpr (SEMI == TILE_S_MAXMIN) return a < b ? a : b;
  else return __fmul_rn(a, b);  // one IEEE op, no contraction (reading 9)
}

__device__ __forceinline__ bool tbit(const uint32_t* b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

template <int SEMI>
__device__ __forceinline__ float oplus_state(float s, float b) {
  if constexpr (SEMI == TILE_S_ADDMULT) return (float)__dadd_rn((double)s, (double)b);
  else return b > s ? b : s;  // max-min (unit has no tags)
}

// Per-thread enumeration state.  Variable values (domains <= 64) are packed
// 6 bits each into one register word so that nothing is indexed dynamically:
// the whole enumeration stays in registers (arrays indexed by runtime
// variable ids or levels went to local memory, which thrashed through L2).
struct Frame {
  const TilePlan* P;   // structure of the plan (the constexpr kPlan when specialised)
  const TilePlan* Q;   // the plan as launched: pointers, sample count, iteration cap
  const uint8_t* sm;
  int s;
  unsigned long long vals;
  double acc;
  double aabs;  // Σ|t| of add-mult terms (split composition items: the rounding certificate)
  float mx;
  bool any;
  uint32_t ncand;
};

__device__ __forceinline__ int getv(unsigned long long vals, int v) { return (int)((vals >> (6 * v)) & 63ull); }
__device__ __forceinline__ void setv(unsigned long long& vals, int v, int x) {
  vals = (vals & ~(63ull << (6 * v))) | ((unsigned long long)x << (6 * v));
}

__device__ __forceinline__ int32_t arg_coord(const TileAtom& A, int c, unsigned long long vals) {
  return A.var[c] >= 0 ? getv(vals, A.var[c]) : A.cst[c];
}

__device__ __forceinline__ unsigned long long fiber(const Frame& F, const TileAtom& A, int ver) {
  const TileRel& T = TP(F).rel[A.rel];
  const TileRel& TQ = F.Q->rel[A.rel];
  const int c = A.fcol;
  int f = 0;
  TILE_UNROLL
  for (int q = 0; q < T.ncols; ++q)
    if (q != c) f += arg_coord(A, q, F.vals) * T.fstride[c][q];
  if (!T.local) return __ldg(TQ.fib[c] + (T.shared ? 0 : (int64_t)F.s * T.nfib[c]) + f);
  const unsigned long long* S = reinterpret_cast<const unsigned long long*>(F.sm + T.sm_fib[0][c]);
  const unsigned long long* D = reinterpret_cast<const unsigned long long*>(F.sm + T.sm_fib[1][c]);
  return ver == TV_OLD ? S[f] : (ver == TV_DELTA ? D[f] : (S[f] | D[f]));
}

__device__ __forceinline__ int atom_slot(const TileRel& T, const TileAtom& A, unsigned long long vals) {
  int slot = 0;
  TILE_UNROLL
  for (int q = 0; q < T.ncols; ++q) slot += arg_coord(A, q, vals) * T.stride[q];
  return slot;
}

__device__ __forceinline__ bool present(const Frame& F, const TileAtom& A, int ver) {
  const TileRel& T = TP(F).rel[A.rel];
  const TileRel& TQ = F.Q->rel[A.rel];
  const int slot = atom_slot(T, A, F.vals);
  if (!T.local) return tbit(TQ.bits + (T.shared ? 0 : (int64_t)F.s * ((T.D + 31) >> 5)), slot);
  const uint32_t* Sb = reinterpret_cast<const uint32_t*>(F.sm + T.sm_bits[0]);
  const uint32_t* Db = reinterpret_cast<const uint32_t*>(F.sm + T.sm_bits[1]);
  if (ver == TV_OLD) return tbit(Sb, slot);
  if (ver == TV_DELTA) return tbit(Db, slot);
  return tbit(Sb, slot) || tbit(Db, slot);
}

template <int SEMI>
__device__ __forceinline__ float atom_tag(const Frame& F, const TileAtom& A, int ver) {
  const TileRel& T = TP(F).rel[A.rel];
  const TileRel& TQ = F.Q->rel[A.rel];
  const int slot = atom_slot(T, A, F.vals);
  if (!T.local) return __ldg(TQ.tag + (T.shared ? 0 : (int64_t)F.s * T.D) + slot);
  const float* St = reinterpret_cast<const float*>(F.sm + T.sm_tag[0]);
  const float* Dt = reinterpret_cast<const float*>(F.sm + T.sm_tag[1]);
  if (ver == TV_OLD) return St[slot];
  if (ver == TV_DELTA) return Dt[slot];
  const uint32_t* Sb = reinterpret_cast<const uint32_t*>(F.sm + T.sm_bits[0]);
  const uint32_t* Db = reinterpret_cast<const uint32_t*>(F.sm + T.sm_bits[1]);
  const bool sp = tbit(Sb, slot), dp = tbit(Db, slot);
  return sp ? (dp ? oplus_state<SEMI>(St[slot], Dt[slot]) : St[slot]) : Dt[slot];
}

__device__ __forceinline__ int32_t cmp_value(int8_t v, int32_t c, const TileRule& R, unsigned long long vals) {
  return v >= 0 ? getv(vals, v) + R.vmin[v] : c;
}

__device__ __forceinline__ bool cmps_ok(const TileRule& R, int level, unsigned long long vals) {
  TILE_UNROLL
  for (int i = 0; i < R.ncmp; ++i) {
    const TileCmp& c = R.cmp[i];
    if (c.level != level) continue;
    const int32_t a = cmp_value(c.va, c.ca, R, vals), b = cmp_value(c.vb, c.cb, R, vals);
    // c.neq: relation 0 ==, 1 !=, 2 <, 3 <=, 4 >, 5 >=
    const bool ok = c.neq == 0 ? a == b : c.neq == 1 ? a != b : c.neq == 2 ? a < b : c.neq == 3 ? a <= b
                  : c.neq == 4 ? a > b : a >= b;
    if (!ok) return false;
  }
  return true;
}

// leaf: every alive variant in order; ⊗ left-deep in body order (reading 9)
template <int SEMI>
__device__ __forceinline__ void leaf(Frame& F, const TileRule& R, uint32_t alive) {
  TILE_UNROLL
  for (int j = 0; j < R.nvariant; ++j) {
    if (!((alive >> j) & 1u)) continue;
    F.any = true;
    F.ncand++;
    if constexpr (SEMI != TILE_S_UNIT) {
      float t = atom_tag<SEMI>(F, R.atom[0], R.ver[j][0]);
      TILE_UNROLL
      for (int a = 1; a < R.natoms; ++a) t = tile_otimes<SEMI>(t, atom_tag<SEMI>(F, R.atom[a], R.ver[j][a]));
      if constexpr (SEMI == TILE_S_ADDMULT) F.acc = __dadd_rn(F.acc, (double)t);
      else F.mx = (F.ncand == 1 || t > F.mx) ? t : F.mx;
    }
  }
}

// Semi-join pruning: an atom whose other variables are all bound at level L
// (chk == L) but which closes later needs a non-empty fiber in each variant's
// version, else that variant has no candidate below this value.
__device__ __forceinline__ uint32_t prune(const Frame& F, const TileRule& R, int L, uint32_t al) {
  TILE_UNROLL
  for (int a = 0; a < R.natoms && al; ++a) {
    const TileAtom& A = R.atom[a];
    if (A.chk != L || A.level <= L) continue;
    TILE_UNROLL
    for (int j = 0; j < R.nvariant; ++j)
      if (((al >> j) & 1u) && !fiber(F, A, R.ver[j][a])) al &= ~(1u << j);
  }
  return al;
}

// Level L of the canonical enumeration (non-head variables by first
// appearance, ascending values; reading 8b): per variant, the values of the
// level's variable are the AND of the fibers of the atoms it closes.  NLEV is
// a compile-time bound so every per-level mask stays in registers.
template <int SEMI, int L, int NLEV>
__device__ __forceinline__ void level(Frame& F, const TileRule& R, uint32_t alive) {
  if constexpr (L == NLEV) {
    leaf<SEMI>(F, R, alive);
  } else {
    const int v = R.lev_var[L];
    const unsigned long long full = R.vdom[v] >= 64 ? ~0ull : ((1ull << R.vdom[v]) - 1ull);
    unsigned long long m[TILE_MAXVAR];
#pragma unroll
    for (int j = 0; j < TILE_MAXVAR; ++j) {
      unsigned long long x = 0;
      if (j < R.nvariant && ((alive >> j) & 1u)) {
        x = full;
        TILE_UNROLL
        for (int a = 0; a < R.natoms && x; ++a)
          if (R.atom[a].level == L) x &= fiber(F, R.atom[a], R.ver[j][a]);
      }
      m[j] = x;
    }
    unsigned long long rem = m[0] | m[1] | m[2] | m[3];
    while (rem) {
      const int b = __ffsll((long long)rem) - 1;
      rem &= rem - 1;
      setv(F.vals, v, b);
      if (!cmps_ok(R, L, F.vals)) continue;
      uint32_t al = 0;
#pragma unroll
      for (int j = 0; j < TILE_MAXVAR; ++j) al |= (uint32_t)((m[j] >> b) & 1ull) << j;
      al = prune(F, R, L, al);
      if (al) level<SEMI, L + 1, NLEV>(F, R, al);
    }
  }
}

// MAXL: deepest enumeration compiled in (the 1024-thread variant keeps only
// shallow seed rules, the host checks R.nlev <= MAXL)
template <int SEMI, int MAXL>
__device__ __forceinline__ void enumerate(Frame& F, const TileRule& R, uint32_t alive) {
  switch (R.nlev) {
    case 0: level<SEMI, 0, 0>(F, R, alive); break;
    case 1: level<SEMI, 0, 1>(F, R, alive); break;
    default:
      if constexpr (MAXL <= 2) {
        level<SEMI, 0, 2>(F, R, alive);
      } else {
        switch (R.nlev) {
          case 2: level<SEMI, 0, 2>(F, R, alive); break;
          case 3: level<SEMI, 0, 3>(F, R, alive); break;
          case 4: level<SEMI, 0, 4>(F, R, alive); break;
          default: level<SEMI, 0, 5>(F, R, alive); break;
        }
      }
  }
}

// The composition rule (CLUTRR-shaped kinship)
//     H(a, x, z) :- K(b, x, y), K(c, y, z), T(b, c, a)      (K = H local, T external)
// enumerated with its structure spelled out: the same canonical order
// (b, y, c, variant) and the same fibers as the generic levels, without
// interpreting the plan (the generic path spent ~200 instructions per
// candidate on plan reads and atom loops).  Variant 0 reads Δ(b,x,y),
// OLD(c,y,z); variant 1 NEW(b,x,y), Δ(c,y,z).
//
// ys_s / ys_d: the y values z can be reached from through OLD(·, y, z) /
// Δ(·, y, z) (all ones when unknown).  A y outside (Δ(b,x,·) ∩ ys_s) ∪
// (NEW(b,x,·) ∩ ys_d) has no candidate in either variant, so skipping it
// leaves the candidates and their order unchanged.
template <int SEMI>
__device__ __forceinline__ void compose_core(Frame& F, const TileRule& R, int a, int x, int z,
                                             unsigned long long ys_s, unsigned long long ys_d,
                                             unsigned long long bs) {
  const TileRel& K = TP(F).rel[R.atom[0].rel];
  const TileRel& T = TP(F).rel[R.atom[2].rel];
  const TileRel& TQ = F.Q->rel[R.atom[2].rel];
  const int RB = K.dom[0];
  const unsigned long long* Sf2 = reinterpret_cast<const unsigned long long*>(F.sm + K.sm_fib[0][2]);
  const unsigned long long* Df2 = reinterpret_cast<const unsigned long long*>(F.sm + K.sm_fib[1][2]);
  const unsigned long long* Sf0 = reinterpret_cast<const unsigned long long*>(F.sm + K.sm_fib[0][0]);
  const unsigned long long* Df0 = reinterpret_cast<const unsigned long long*>(F.sm + K.sm_fib[1][0]);
  const float* St = reinterpret_cast<const float*>(F.sm + K.sm_tag[0]);
  const float* Dt = reinterpret_cast<const float*>(F.sm + K.sm_tag[1]);
  const uint32_t* Sb = reinterpret_cast<const uint32_t*>(F.sm + K.sm_bits[0]);
  const unsigned long long* Tf = TQ.fib[1] + (T.shared ? 0 : (int64_t)F.s * T.nfib[1]);
  const float* Tt = TQ.tag ? TQ.tag + (T.shared ? 0 : (int64_t)F.s * T.D) : nullptr;
  (void)RB;
  while (bs) {  // b with NEW(b, x, ·) non-empty (a superset: all ones when unknown)
    const int b = __ffsll((long long)bs) - 1;
    bs &= bs - 1;
    const int fbx = b * K.fstride[2][0] + x * K.fstride[2][1];
    const unsigned long long d0 = Df2[fbx], n0 = Sf2[fbx] | d0;  // y with Δ / NEW (b, x, y)
    unsigned long long ys = (d0 & ys_s) | (n0 & ys_d);
    if (!ys) continue;
    const unsigned long long tf = __ldg(Tf + b * T.fstride[1][0] + a * T.fstride[1][2]);  // c with T(b, c, a)
    if (!tf) continue;
    while (ys) {
      const int y = __ffsll((long long)ys) - 1;
      ys &= ys - 1;
      const int fyz = y * K.fstride[0][1] + z * K.fstride[0][2];
      const unsigned long long m0 = ((d0 >> y) & 1ull) ? (Sf0[fyz] & tf) : 0ull;  // v0: Δ(b,x,y) OLD(c,y,z)
      const unsigned long long m1 = Df0[fyz] & tf;                                // v1: NEW(b,x,y) Δ(c,y,z)
      unsigned long long cs = m0 | m1;
      if (!cs) continue;
      const int sbxy = b * K.stride[0] + x * K.stride[1] + y * K.stride[2];
      float nbxy = 0.0f, dbxy = 0.0f;
      if constexpr (SEMI != TILE_S_UNIT) {
        dbxy = Dt[sbxy];
        const bool sp = tbit(Sb, sbxy), dp = (d0 >> y) & 1ull;
        nbxy = sp ? (dp ? oplus_state<SEMI>(St[sbxy], dbxy) : St[sbxy]) : dbxy;
      }
      while (cs) {
        const int c = __ffsll((long long)cs) - 1;
        cs &= cs - 1;
        const int scyz = c * K.stride[0] + y * K.stride[1] + z * K.stride[2];
        const float tc = (SEMI != TILE_S_UNIT && Tt) ? __ldg(Tt + b * T.stride[0] + c * T.stride[1] + a * T.stride[2]) : 1.0f;
        if ((m0 >> c) & 1ull) {
          F.any = true;
          F.ncand++;
          if constexpr (SEMI != TILE_S_UNIT) {
            const float t = tile_otimes<SEMI>(tile_otimes<SEMI>(dbxy, St[scyz]), tc);
            if constexpr (SEMI == TILE_S_ADDMULT) F.acc = __dadd_rn(F.acc, (double)t);
            else F.mx = (F.ncand == 1 || t > F.mx) ? t : F.mx;
          }
        }
        if ((m1 >> c) & 1ull) {
          F.any = true;
          F.ncand++;
          if constexpr (SEMI != TILE_S_UNIT) {
            const float t = tile_otimes<SEMI>(tile_otimes<SEMI>(nbxy, Dt[scyz]), tc);
            if constexpr (SEMI == TILE_S_ADDMULT) F.acc = __dadd_rn(F.acc, (double)t);
            else F.mx = (F.ncand == 1 || t > F.mx) ? t : F.mx;
          }
        }
      }
    }
  }
}

// compose_core with 32-bit masks (relation-type and entity domains <= 32, the
// low words of the 64-bit fibers), the T tag row and the (y, z) slot part
// hoisted out of the candidate loop: the same candidates in the same order.
template <int SEMI, bool ABS = false>
__device__ __forceinline__ void compose_core32(Frame& F, const TileRule& R, int a, int x, int z, uint32_t ys_s,
                                               uint32_t ys_d, uint32_t bs) {
  const TileRel& K = TP(F).rel[R.atom[0].rel];
  const TileRel& T = TP(F).rel[R.atom[2].rel];
  const TileRel& TQ = F.Q->rel[R.atom[2].rel];
  const uint32_t* Sf2 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[0][2]);  // low words: [2 f]
  const uint32_t* Df2 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[1][2]);
  const uint32_t* Sf0 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[0][0]);
  const uint32_t* Df0 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[1][0]);
  const float* St = reinterpret_cast<const float*>(F.sm + K.sm_tag[0]);
  const float* Dt = reinterpret_cast<const float*>(F.sm + K.sm_tag[1]);
  const uint32_t* Sb = reinterpret_cast<const uint32_t*>(F.sm + K.sm_bits[0]);
  const uint32_t* Tf = reinterpret_cast<const uint32_t*>(TQ.fib[1] + (T.shared ? 0 : (int64_t)F.s * T.nfib[1]));
  const float* Tt = TQ.tag ? TQ.tag + (T.shared ? 0 : (int64_t)F.s * T.D) : nullptr;
  const int ks0 = K.stride[0], zs = z * K.stride[2], xs = x * K.stride[1];
  const int f2x = x * K.fstride[2][1], f2b = K.fstride[2][0], f0y = K.fstride[0][1], f0z = z * K.fstride[0][2];
  const int tfb = T.fstride[1][0], tfa = a * T.fstride[1][2], ts0 = T.stride[0], ts1 = T.stride[1];
  const int ta = a * T.stride[2];
  double acc = F.acc, aabs = F.aabs;
  float mx = F.mx;
  uint32_t nc = F.ncand;
  while (bs) {
    const int b = __ffs(bs) - 1;
    bs &= bs - 1;
    const int fbx = b * f2b + f2x;
    const uint32_t d0 = Df2[2 * fbx], n0 = Sf2[2 * fbx] | d0;
    uint32_t ys = (d0 & ys_s) | (n0 & ys_d);
    if (!ys) continue;
    const uint32_t tf = __ldg(Tf + 2 * (b * tfb + tfa));
    if (!tf) continue;
    const float* Ttb = Tt ? Tt + b * ts0 + ta : nullptr;
    const int bx = b * ks0 + xs;
    while (ys) {
      const int y = __ffs(ys) - 1;
      ys &= ys - 1;
      const int fyz = y * f0y + f0z;
      const uint32_t dy = (d0 >> y) & 1u;
      const uint32_t m0 = dy ? (Sf0[2 * fyz] & tf) : 0u;  // v0: Δ(b,x,y) OLD(c,y,z)
      const uint32_t m1 = Df0[2 * fyz] & tf;              // v1: NEW(b,x,y) Δ(c,y,z)
      uint32_t cs = m0 | m1;
      if (!cs) continue;
      float nbxy = 0.0f, dbxy = 0.0f;
      if constexpr (SEMI != TILE_S_UNIT) {
        const int sbxy = bx + y * K.stride[2];
        dbxy = Dt[sbxy];
        const bool sp = tbit(Sb, sbxy);
        nbxy = sp ? (dy ? oplus_state<SEMI>(St[sbxy], dbxy) : St[sbxy]) : dbxy;
      }
      const int yz = y * K.stride[1] + zs;
      while (cs) {
        const int c = __ffs(cs) - 1;
        cs &= cs - 1;
        const int scyz = c * ks0 + yz;
        const float tc = (SEMI != TILE_S_UNIT && Ttb) ? __ldg(Ttb + c * ts1) : 1.0f;
        if ((m0 >> c) & 1u) {
          ++nc;
          if constexpr (SEMI != TILE_S_UNIT) {
            const float t = tile_otimes<SEMI>(tile_otimes<SEMI>(dbxy, St[scyz]), tc);
            if constexpr (SEMI == TILE_S_ADDMULT) {
              acc = __dadd_rn(acc, (double)t);
              if constexpr (ABS) aabs = __dadd_rn(aabs, fabs((double)t));
            } else {
              mx = (nc == 1 || t > mx) ? t : mx;
            }
          }
        }
        if ((m1 >> c) & 1u) {
          ++nc;
          if constexpr (SEMI != TILE_S_UNIT) {
            const float t = tile_otimes<SEMI>(tile_otimes<SEMI>(nbxy, Dt[scyz]), tc);
            if constexpr (SEMI == TILE_S_ADDMULT) {
              acc = __dadd_rn(acc, (double)t);
              if constexpr (ABS) aabs = __dadd_rn(aabs, fabs((double)t));
            } else {
              mx = (nc == 1 || t > mx) ? t : mx;
            }
          }
        }
      }
    }
  }
  F.acc = acc;
  F.aabs = aabs;
  F.mx = mx;
  F.any = F.any || nc != F.ncand;
  F.ncand = nc;
}

template <int SEMI>
__device__ __forceinline__ void compose_head(Frame& F, const TileRule& R) {
  compose_core<SEMI>(F, R, getv(F.vals, R.atom[2].var[2]), getv(F.vals, R.atom[0].var[1]),
                     getv(F.vals, R.atom[1].var[2]), ~0ull, ~0ull,
                     TP(F).rel[R.atom[0].rel].dom[0] >= 64 ? ~0ull : (1ull << TP(F).rel[R.atom[0].rel].dom[0]) - 1ull);
}

// The candidates of one head (a, x, z) enumerated from T's side, in the
// order (b, c, y, variant): for each b with NEW(b, x, ·) and each c of
// T(b, ·, a), the y are the AND of the fibers Δ(b,x,·) ∧ OLD(c,·,z)
// (variant 0) and NEW(b,x,·) ∧ Δ(c,·,z) (variant 1) — K's middle-column
// fibers — so no y without a candidate is visited.  The terms are the same
// fp32 values as the canonical walk; only their summation order differs, so
// the caller certifies the fp32 rounding (add-mult) or needs no certificate
// (max-min: max is exact; unit).
template <int SEMI>
__device__ __forceinline__ void compose_bc32(Frame& F, const TileRule& R, int a, int x, int z, uint32_t bs) {
  const TileRel& K = TP(F).rel[R.atom[0].rel];
  const TileRel& T = TP(F).rel[R.atom[2].rel];
  const TileRel& TQ = F.Q->rel[R.atom[2].rel];
  const uint32_t* Sf2 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[0][2]);  // low words: [2 f]
  const uint32_t* Df2 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[1][2]);
  const uint32_t* Sf1 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[0][1]);
  const uint32_t* Df1 = reinterpret_cast<const uint32_t*>(F.sm + K.sm_fib[1][1]);
  const float* St = reinterpret_cast<const float*>(F.sm + K.sm_tag[0]);
  const float* Dt = reinterpret_cast<const float*>(F.sm + K.sm_tag[1]);
  const uint32_t* Sb = reinterpret_cast<const uint32_t*>(F.sm + K.sm_bits[0]);
  const uint32_t* Tf = reinterpret_cast<const uint32_t*>(TQ.fib[1] + (T.shared ? 0 : (int64_t)F.s * T.nfib[1]));
  const float* Tt = TQ.tag ? TQ.tag + (T.shared ? 0 : (int64_t)F.s * T.D) : nullptr;
  const int ks0 = K.stride[0], ks1 = K.stride[1], ks2 = K.stride[2], zs = z * ks2, xs = x * ks1;
  const int f2x = x * K.fstride[2][1], f2b = K.fstride[2][0], f1c = K.fstride[1][0], f1z = z * K.fstride[1][2];
  const int tfb = T.fstride[1][0], tfa = a * T.fstride[1][2], ts0 = T.stride[0], ts1 = T.stride[1];
  const int ta = a * T.stride[2];
  double acc = F.acc, aabs = F.aabs;
  float mx = F.mx;
  uint32_t nc = F.ncand;
  while (bs) {
    const int b = __ffs(bs) - 1;
    bs &= bs - 1;
    uint32_t cc = __ldg(Tf + 2 * (b * tfb + tfa));  // c with T(b, c, a)
    if (!cc) continue;
    const int fbx = b * f2b + f2x;
    const uint32_t d0 = Df2[2 * fbx], n0 = Sf2[2 * fbx] | d0;
    const float* Ttb = Tt ? Tt + b * ts0 + ta : nullptr;
    const int bx = b * ks0 + xs;
    while (cc) {
      const int c = __ffs(cc) - 1;
      cc &= cc - 1;
      const int fcz = c * f1c + f1z;
      uint32_t m0 = d0 & Sf1[2 * fcz], m1 = n0 & Df1[2 * fcz];
      if (!(m0 | m1)) continue;
      const float tc = (SEMI != TILE_S_UNIT && Ttb) ? __ldg(Ttb + c * ts1) : 1.0f;
      const int cz = c * ks0 + zs;
      if constexpr (SEMI == TILE_S_UNIT) {
        nc += __popc(m0) + __popc(m1);
        continue;
      }
      while (m0) {  // v0: Δ(b,x,y) ⊗ OLD(c,y,z) ⊗ T(b,c,a)
        const int y = __ffs(m0) - 1;
        m0 &= m0 - 1;
        ++nc;
        const float t = tile_otimes<SEMI>(tile_otimes<SEMI>(Dt[bx + y * ks2], St[cz + y * ks1]), tc);
        if constexpr (SEMI == TILE_S_ADDMULT) {
          acc = __dadd_rn(acc, (double)t);
          aabs = __dadd_rn(aabs, fabs((double)t));
        } else {
          mx = (nc == 1 || t > mx) ? t : mx;
        }
      }
      while (m1) {  // v1: NEW(b,x,y) ⊗ Δ(c,y,z) ⊗ T(b,c,a)
        const int y = __ffs(m1) - 1;
        m1 &= m1 - 1;
        ++nc;
        const int sbxy = bx + y * ks2;
        const float dv = Dt[sbxy];
        const float nb = tbit(Sb, sbxy) ? (((d0 >> y) & 1u) ? oplus_state<SEMI>(St[sbxy], dv) : St[sbxy]) : dv;
        const float t = tile_otimes<SEMI>(tile_otimes<SEMI>(nb, Dt[cz + y * ks1]), tc);
        if constexpr (SEMI == TILE_S_ADDMULT) {
          acc = __dadd_rn(acc, (double)t);
          aabs = __dadd_rn(aabs, fabs((double)t));
        } else {
          mx = (nc == 1 || t > mx) ? t : mx;
        }
      }
    }
  }
  F.acc = acc;
  F.aabs = aabs;
  F.mx = mx;
  F.any = F.any || nc != F.ncand;
  F.ncand = nc;
}

// fp32 rounding certificate of an fp64 sum of n terms formed in some order
// whose canonical sequential sum must be reproduced: both lie within
// (n + k)·2^-53·Σ|t| of the exact sum (every term takes at most n + k
// roundings), so if every value in s ± d rounds to one fp32 value, that value
// is fl32(canonical sum).  Returns false when uncertified.
__device__ __forceinline__ bool certify32(double s, double ab, uint32_t n, int k, float& out) {
  const double d = (2.0 * (double)(n + k) + 4.0) * 0x1p-53 * ab * 1.01;
  const float lo = __double2float_rn(__dsub_rn(s, d)), hi = __double2float_rn(__dadd_rn(s, d));
  out = lo;
  return lo == hi;
}

// A round ends at its longest head item (C3: from round ~6 on, one item's
// walk IS the round).  The items of the heaviest pairs (all of them when
// they fit the partial buffer) are split into P parts by b
// (ranks ≡ part mod P), the parts run in parallel and their partial results
// are combined per head:
//   unit: any part;  max-min: the max (exact, order-free);
//   add-mult: the fp64 sum of the parts.  The sequential fp64 sum S_seq of
//   the oracle's canonical order and this S_par both lie within
//   (n + P)·2^-53·Σ|t| of the exact sum (n terms; every term takes at most
//   n + P roundings), so when every value in S_par ± d, d = (2(n + P) + 4)·
//   2^-53·Σ|t|·1.01, rounds to the same fp32 value, that value IS
//   fl32(S_seq) (rounding is monotone).  Otherwise (rare: S within d of an
//   fp32 rounding boundary) the head is recomputed sequentially in canonical
//   order.  Either way U is bit-identical to the sequential walk.
template <int SEMI>
__device__ __forceinline__ void compose_split(Frame& F, const TileRule& R, const TileRel& H, int items, uint8_t* pb,
                                           uint32_t* npairs, const uint16_t* pairs, const unsigned long long* AX,
                                           uint64_t& my_cand, uint32_t* tr) {
  const unsigned long long* SY = AX + 128;
  const unsigned long long* DY = AX + 192;
  const unsigned long long* BX = AX + 256;
  const int A = H.dom[0], Z = H.dom[2];
  pb = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pb) + 7) & ~uintptr_t(7));
  double* pacc = reinterpret_cast<double*>(pb);
  float* pabs = reinterpret_cast<float*>(pacc + TILE_CM_PARTS);  // Σ|t| rounded up
  uint32_t* pcnt = reinterpret_cast<uint32_t*>(pabs + TILE_CM_PARTS);
  uint32_t* Ub = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(F.sm) + H.sm_bits[2]);
  float* Ut = reinterpret_cast<float*>(const_cast<uint8_t*>(F.sm) + H.sm_tag[2]);
  // split every pair's items when at least two parts per item fit the
  // partial buffer (up to ~2 sub-items per thread), else the heaviest two
  // cost classes' items (C3: 4.53 -> 4.44 ms; with the canonical-order walk
  // the same split of the big rounds had measured slower, 6.42 vs 6.21 ms)
  const int npr = items / A;
  int ns = items * 2 <= TILE_CM_PARTS ? npr : min((int)(npairs[2] + npairs[3]), TILE_CM_PARTS / (2 * A));
  int P = 1;
  while (P < 8 && ns * A * P * 2 <= TILE_CM_PARTS && (ns * A * P < 2 * (int)blockDim.x || ns < npr)) P <<= 1;
  if (P == 1) ns = 0;
  const int nsub = ns * A * P, total = nsub + (npr - ns) * A;
  const int t = threadIdx.x, lane = t & 31;
  for (;;) {  // (pair, part, a): a fastest, so a warp's lanes share the b subset
    int base = 0;
    if (lane == 0) base = (int)atomicAdd(npairs + 1, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= total) break;
    const int i = base + lane;
    if (i >= total) continue;
    F.acc = 0.0;
    F.aabs = 0.0;
    F.mx = 0.0f;
    F.any = false;
    F.ncand = 0;
    const long long c0 = tr ? clock64() : 0;
    if (i >= nsub) {  // a whole item: U directly
      const int w = i - nsub + ns * A, pi = w / A, a = w - pi * A;
      const int p = pairs[pi], x = p / Z, z = p - x * Z;
      compose_bc32<SEMI>(F, R, a, x, z, (uint32_t)BX[x]);
      my_cand += F.ncand;
      if (tr) {
        atomicAdd(tr, F.ncand);
        atomicMax(tr + 2, (uint32_t)((clock64() - c0) >> 4));
      }
      if (F.any) {
        float u = F.mx;
        if constexpr (SEMI == TILE_S_ADDMULT) {
          if (!certify32(F.acc, F.aabs, F.ncand, 0, u) || F.Q->cm_nocert) {  // the canonical sequential walk
            F.acc = 0.0;
            F.ncand = 0;
            compose_core32<SEMI>(F, R, a, x, z, (uint32_t)SY[z], (uint32_t)DY[z], (uint32_t)BX[x]);
            u = (float)F.acc;
            if (tr) atomicAdd(tr + 1, 1u << 16);
          }
        }
        const int h = a * H.stride[0] + x * H.stride[1] + z * H.stride[2];
        atomicOr(Ub + (h >> 5), 1u << (h & 31));
        if constexpr (SEMI != TILE_S_UNIT) Ut[h] = u;
      }
      continue;
    }
    const int pi = i / (A * P), rem = i - pi * (A * P), part = rem / A, a = rem - part * A;
    const int p = pairs[pi], x = p / Z, z = p - x * Z;
    uint32_t bm = (uint32_t)BX[x], bs = 0;
    for (int r = 0; bm; ++r) {
      const uint32_t lo = bm & (0u - bm);
      bm ^= lo;
      if ((r & (P - 1)) == part) bs |= lo;
    }
    compose_bc32<SEMI>(F, R, a, x, z, bs);
    my_cand += F.ncand;
    if (tr) {
      atomicAdd(tr, F.ncand);
      atomicMax(tr + 2, (uint32_t)((clock64() - c0) >> 4));
    }
    const int j = (pi * A + a) * P + part;
    if (j >= TILE_CM_PARTS) __trap();  // bounds guard (compute-sanitizer is unavailable on the GPU pool)
    pacc[j] = SEMI == TILE_S_ADDMULT ? F.acc : (double)F.mx;
    pabs[j] = __double2float_ru(F.aabs);
    pcnt[j] = F.ncand;
  }
  if (!ns) return;
  __syncthreads();
  for (int it = t; it < ns * A; it += blockDim.x) {
    const int pi = it / A, a = it - pi * A;
    const int p = pairs[pi], x = p / Z, z = p - x * Z;
    double s = 0.0, ab = 0.0;
    float mx = 0.0f;
    uint32_t n = 0;
    for (int part = 0; part < P; ++part) {
      const int j = it * P + part;
      const uint32_t c = pcnt[j];
      if (!c) continue;
      if constexpr (SEMI == TILE_S_ADDMULT) {
        s = __dadd_rn(s, pacc[j]);
        ab = __dadd_rn(ab, (double)pabs[j]);
      } else if constexpr (SEMI == TILE_S_MAXMIN) {
        const float v = (float)pacc[j];
        mx = (n == 0 || v > mx) ? v : mx;
      }
      n += c;
    }
    if (!n) continue;
    float u = mx;
    if constexpr (SEMI == TILE_S_ADDMULT) {
      if (certify32(s, ab, n, P, u) && !F.Q->cm_nocert) {
      } else {  // uncertified: the canonical sequential walk
        F.acc = 0.0;
        F.aabs = 0.0;
        F.mx = 0.0f;
        F.any = false;
        F.ncand = 0;
        compose_core32<SEMI>(F, R, a, x, z, (uint32_t)SY[z], (uint32_t)DY[z], (uint32_t)BX[x]);
        u = (float)F.acc;
        if (tr) atomicAdd(tr + 1, 1u << 16);  // debug: fallbacks in the |Δ'| word's high half
      }
    }
    const int h = a * H.stride[0] + x * H.stride[1] + z * H.stride[2];
    atomicOr(Ub + (h >> 5), 1u << (h & 31));
    if constexpr (SEMI != TILE_S_UNIT) Ut[h] = u;
  }
}

// One recursive round of a stratum whose only recursive rule is the
// composition shape (TilePlan::cm_rule): U of every head slot, evaluating
// only the slots (a, x, z) whose pair (x, z) can receive a candidate:
//   (Δ(·, x, ·) ∩ OLD(·, ·, z)-sources) ∪ (NEW(·, x, ·) ∩ Δ(·, ·, z)-sources) ≠ ∅
// over y (a superset of the slots with candidates; the others get no U, as
// before).  Active pairs are listed in shared memory, heaviest first, and
// handed out with a fastest across lanes.  Per head the candidates are
// compose_bc32's (T-driven order, rounding certified, canonical fallback;
// compose_split) — U bit-identical to the canonical walk; with 64-bit masks
// (domains > 32) or LOBSTER_TILE_NO_SPLIT, compose_core's canonical walk.
template <int SEMI>
__device__ __forceinline__ void compose_rounds(Frame& F, const TilePlan& Q, uint8_t* sm, uint64_t& my_cand,
                                               uint32_t* tr) {
  const TileRule& R = TP(F).rule[Q.cm_rule];
  const TileRel& H = TP(F).rel[R.head];
  const int A = H.dom[0], X = H.dom[1], Z = H.dom[2];
  unsigned long long* AX = reinterpret_cast<unsigned long long*>(sm + Q.cm_off);  // y: Δ(b, x, y) for some b
  unsigned long long* NX = AX + 64;                                              // y: NEW(b, x, y)
  unsigned long long* SY = AX + 128;                                             // y: OLD(c, y, z) for some c
  unsigned long long* DY = AX + 192;                                             // y: Δ(c, y, z)
  unsigned long long* BX = AX + 256;                                             // b: NEW(b, x, ·) non-empty
  uint32_t* npairs = reinterpret_cast<uint32_t*>(AX + 320);
  // npairs: [0] active pairs, [1] work counter, [2..5] pairs per cost class, [6..9] class offsets
  uint32_t* slotof = npairs + 16;                                                // per pair: class << 16 | rank
  uint16_t* pairs = reinterpret_cast<uint16_t*>(slotof + X * Z);
  const unsigned long long* Sf2 = reinterpret_cast<const unsigned long long*>(sm + H.sm_fib[0][2]);
  const unsigned long long* Df2 = reinterpret_cast<const unsigned long long*>(sm + H.sm_fib[1][2]);
  const unsigned long long* Sf0 = reinterpret_cast<const unsigned long long*>(sm + H.sm_fib[0][0]);
  const unsigned long long* Df0 = reinterpret_cast<const unsigned long long*>(sm + H.sm_fib[1][0]);
  uint32_t* Ub = reinterpret_cast<uint32_t*>(sm + H.sm_bits[2]);
  float* Ut = reinterpret_cast<float*>(sm + H.sm_tag[2]);
  const int t = threadIdx.x;
  if (t < X) {
    unsigned long long ax = 0, nx = 0, bx = 0;
    for (int b = 0; b < A; ++b) {
      const int f = b * H.fstride[2][0] + t * H.fstride[2][1];
      const unsigned long long n = Sf2[f] | Df2[f];
      ax |= Df2[f];
      nx |= n;
      bx |= (unsigned long long)(n != 0ull) << b;
    }
    AX[t] = ax;
    NX[t] = nx;
    BX[t] = bx;
  } else if (t >= 64 && t < 64 + Z) {
    const int z = t - 64;
    unsigned long long sy = 0, dy = 0;
    for (int y = 0; y < H.dom[1]; ++y) {
      const int f = y * H.fstride[0][1] + z * H.fstride[0][2];
      sy |= (unsigned long long)(Sf0[f] != 0ull) << y;
      dy |= (unsigned long long)(Df0[f] != 0ull) << y;
    }
    SY[z] = sy;
    DY[z] = dy;
  } else if (t == 128) {
    for (int k = 0; k < 10; ++k) npairs[k] = 0;
  }
  const int nw = (H.D + 31) >> 5;
  for (int w = t; w < nw; w += blockDim.x) Ub[w] = 0u;
  __syncthreads();
  for (int p = t; p < X * Z; p += blockDim.x) {
    const int x = p / Z, z = p - x * Z;
    const unsigned long long ys = (AX[x] & SY[z]) | (NX[x] & DY[z]);
    if (!ys) continue;
    // longest first (a round ends at its slowest warp): class by the size of
    // the pair's (b, y) walk, heaviest class first
    const int cost = __popcll(BX[x]) * __popcll(ys);
    const int k = cost >= 96 ? 0 : cost >= 32 ? 1 : cost >= 8 ? 2 : 3;
    slotof[p] = ((uint32_t)k << 16) | atomicAdd(npairs + 2 + k, 1u);
  }
  __syncthreads();
  if (t == 0) {
    uint32_t o = 0;
    for (int k = 0; k < 4; ++k) {
      npairs[6 + k] = o;
      o += npairs[2 + k];
    }
    npairs[0] = o;
  }
  __syncthreads();
  for (int p = t; p < X * Z; p += blockDim.x) {
    const int x = p / Z, z = p - x * Z;
    if ((AX[x] & SY[z]) | (NX[x] & DY[z])) pairs[npairs[6 + (slotof[p] >> 16)] + (slotof[p] & 0xffffu)] = (uint16_t)p;
  }
  __syncthreads();
  const int items = (int)npairs[0] * A;
  const bool narrow = A <= 32 && H.dom[1] <= 32 && H.dom[2] <= 32;  // 32-bit masks (K == H)
  const int lane = t & 31;
  if (narrow && !F.Q->cm_nosplit) {
    compose_split<SEMI>(F, R, H, items, (uint8_t*)(pairs + X * Z), npairs, pairs, AX, my_cand, tr);
    return;
  }
  // warps claim 32 items at a time (items differ a lot in cost; a static
  // stride left warps waiting at the round's barrier)
  for (;;) {
    int base = 0;
    if (lane == 0) base = (int)atomicAdd(npairs + 1, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= items) break;
    const int i = base + lane;
    if (i >= items) continue;
    const int p = pairs[i / A], a = i - (i / A) * A;
    const int x = p / Z, z = p - x * Z;
    F.acc = 0.0;
    F.mx = 0.0f;
    F.any = false;
    F.ncand = 0;
    const long long c0 = tr ? clock64() : 0;
    if (narrow)
      compose_core32<SEMI>(F, R, a, x, z, (uint32_t)SY[z], (uint32_t)DY[z], (uint32_t)BX[x]);
    else
      compose_core<SEMI>(F, R, a, x, z, SY[z], DY[z], BX[x]);
    my_cand += F.ncand;
    if (tr) {  // debug (LOBSTER_TILE_TRACE): candidates, longest item (cycles / 16)
      atomicAdd(tr, F.ncand);
      atomicMax(tr + 2, (uint32_t)((clock64() - c0) >> 4));
    }
    if (F.any) {
      const int h = a * H.stride[0] + x * H.stride[1] + z * H.stride[2];
      atomicOr(Ub + (h >> 5), 1u << (h & 31));
      if constexpr (SEMI != TILE_S_UNIT) Ut[h] = SEMI == TILE_S_ADDMULT ? (float)F.acc : F.mx;
    }
  }
}

// U of head slot h of local relation `hr` (one round; seed = round 1)
template <int SEMI, int MAXL>
__device__ __forceinline__ void eval_head(Frame& F, int hr, int h, bool seed) {
  const TileRel& H = TP(F).rel[hr];
  TILE_UNROLL
  for (int ri = 0; ri < TP(F).nrule; ++ri) {
    const TileRule& R = TP(F).rule[ri];
    if (R.head != hr || (R.seed != 0) != seed) continue;
    bool ok = true;
    uint32_t bound = 0;
    F.vals = 0;
    int x = h;
    TILE_UNROLL
    for (int c = H.ncols - 1; c >= 0 && ok; --c) {  // head slot -> column coordinates -> variables
      const int co = x % H.dom[c];
      x /= H.dom[c];
      const int v = R.hvar[c];
      if (v < 0) {
        ok = R.hcst[c] == co;
      } else if ((bound >> v) & 1u) {
        ok = getv(F.vals, v) == co;  // repeated head variable
      } else {
        bound |= 1u << v;
        setv(F.vals, v, co);
      }
    }
    if (!ok || !cmps_ok(R, -1, F.vals)) continue;
    uint32_t alive = (1u << R.nvariant) - 1u;
    TILE_UNROLL
    for (int a = 0; a < R.natoms && alive; ++a) {
      if (R.atom[a].level >= 0) continue;
      TILE_UNROLL
      for (int j = 0; j < R.nvariant; ++j)
        if (((alive >> j) & 1u) && !present(F, R.atom[a], R.ver[j][a])) alive &= ~(1u << j);
    }
    if (R.shape == 1) {
      compose_head<SEMI>(F, R);
      continue;
    }
    if (alive) alive = prune(F, R, -1, alive);
    if (alive) enumerate<SEMI, MAXL>(F, R, alive);
  }
}

// The fixpoint of one stratum; Q: the launched plan, copied into shared
// memory by the caller (sm: the dynamic shared memory of the relations).
template <int SEMI, int MAXL = TILE_MAXLEV>
__device__ __forceinline__ void tile_body(const TilePlan& Q, uint8_t* sm, int* rounds_out, unsigned long long* ncand,
                                          int* cap_hit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  Frame F;
  F.P = &Q;
  F.Q = &Q;
  F.sm = sm;
  uint64_t my_cand = 0;
  for (int s = blockIdx.x; s < Q.nsamples; s += gridDim.x) {
    F.s = s;
    for (int i = threadIdx.x; i < TP(F).clear_words; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0u;
    __syncthreads();
    int round = 1;
    for (;;) {
      const bool seed = round == 1;
      // (i) + (iii): U per head slot (staged in shared memory; keeping the u
      // values in registers instead, with eval_head out of line, measured
      // 23.2 ms vs 17.5 ms on C3 — and 19.3 ms at 64 registers / 2 CTAs per SM)
      const long long ph0 = clock64();
      if (!seed && Q.cm_rule >= 0)
        compose_rounds<SEMI>(F, Q, sm, my_cand, Q.trace ? Q.trace + ((int64_t)s * 64 + min(round, 63)) * 4 : nullptr);
      else
      TILE_UNROLL
      for (int li = 0; li < TP(F).nlocal; ++li) {
        const int hr = TP(F).local_rel[li];
        const TileRel& H = TP(F).rel[hr];
        uint32_t* Ub = reinterpret_cast<uint32_t*>(sm + H.sm_bits[2]);
        float* Ut = reinterpret_cast<float*>(sm + H.sm_tag[2]);
        const int nw = (H.D + 31) >> 5;
        for (int w = warp; w < nw; w += nwarps) {
          const int h = (w << 5) + lane;
          F.acc = 0.0;
          F.mx = 0.0f;
          F.any = false;
          F.ncand = 0;
          if (h < H.D) eval_head<SEMI, MAXL>(F, hr, h, seed);
          my_cand += F.ncand;
          if (Q.trace && F.ncand) atomicAdd(Q.trace + ((int64_t)s * 64 + min(round, 63)) * 4, F.ncand);
          const uint32_t word = __ballot_sync(~0u, F.any);
          if (lane == 0) Ub[w] = word;
          if constexpr (SEMI != TILE_S_UNIT) {
            if (F.any) Ut[h] = SEMI == TILE_S_ADDMULT ? (float)F.acc : F.mx;
          }
        }
      }
      __syncthreads();
      if (Q.trace && threadIdx.x == 0)  // debug: the U phase (cycles / 16)
        atomicMax(Q.trace + ((int64_t)s * 64 + min(round, 63)) * 4 + 3, (uint32_t)((clock64() - ph0) >> 4));
      // (ii) S <- S ⊕ Δ; (iv) Δ' = changed or new U
      int grew = 0;
      TILE_UNROLL
      for (int li = 0; li < TP(F).nlocal; ++li) {
        const TileRel& H = TP(F).rel[TP(F).local_rel[li]];
        const TileRel& HQ = Q.rel[TP(F).local_rel[li]];
        uint32_t* Sb = reinterpret_cast<uint32_t*>(sm + H.sm_bits[0]);
        uint32_t* Db = reinterpret_cast<uint32_t*>(sm + H.sm_bits[1]);
        const uint32_t* Ub = reinterpret_cast<const uint32_t*>(sm + H.sm_bits[2]);
        const int nw = (H.D + 31) >> 5;
        for (int w = warp; w < nw; w += nwarps) {
          const int h = (w << 5) + lane;
          const uint32_t Sw = Sb[w], Dw = Db[w], Uw = Ub[w], bit = 1u << lane;
          const bool sp = Sw & bit, dp = Dw & bit, up = Uw & bit;
          bool nd;
          if constexpr (SEMI == TILE_S_UNIT) {
            nd = up && !(sp || dp);
          } else {
            float* St = reinterpret_cast<float*>(sm + H.sm_tag[0]);
            float* Dt = reinterpret_cast<float*>(sm + H.sm_tag[1]);
            const float* Ut = reinterpret_cast<const float*>(sm + H.sm_tag[2]);
            nd = false;
            if (h < H.D) {
              float sv = St[h];
              if (dp) sv = sp ? oplus_state<SEMI>(sv, Dt[h]) : Dt[h];
              if (dp) St[h] = sv;
              if (up) {
                const float u = Ut[h];
                nd = !(sp || dp) || __float_as_uint(oplus_state<SEMI>(sv, u)) != __float_as_uint(sv);
                if (nd) Dt[h] = u;
              }
            }
          }
          const uint32_t dword = __ballot_sync(~0u, nd);
          if (lane == 0) {
            Sb[w] = Sw | Dw;
            Db[w] = dword;
          }
          grew |= nd;
          if (Q.trace && nd) atomicAdd(Q.trace + ((int64_t)s * 64 + min(round, 63)) * 4 + 1, 1u);
        }
      }
      __syncthreads();
      // fibers of S and Δ from the bitmaps
      TILE_UNROLL
      for (int li = 0; li < TP(F).nlocal; ++li) {
        const TileRel& H = TP(F).rel[TP(F).local_rel[li]];
        const TileRel& HQ = Q.rel[TP(F).local_rel[li]];
        const uint32_t* Sb = reinterpret_cast<const uint32_t*>(sm + H.sm_bits[0]);
        const uint32_t* Db = reinterpret_cast<const uint32_t*>(sm + H.sm_bits[1]);
        TILE_UNROLL
        for (int c = 0; c < H.ncols; ++c) {
          if (!H.nfib[c]) continue;
          unsigned long long* Sf = reinterpret_cast<unsigned long long*>(sm + H.sm_fib[0][c]);
          unsigned long long* Df = reinterpret_cast<unsigned long long*>(sm + H.sm_fib[1][c]);
          for (int f = threadIdx.x; f < H.nfib[c]; f += blockDim.x) {
            int base = 0, x = f;  // decode the other columns (row-major, c skipped)
            for (int q = H.ncols - 1; q >= 0; --q) {
              if (q == c) continue;
              base += (x % H.dom[q]) * H.stride[q];
              x /= H.dom[q];
            }
            unsigned long long ws = 0, wd = 0;
            for (int k = 0; k < H.dom[c]; ++k) {
              const int slot = base + k * H.stride[c];
              ws |= (unsigned long long)tbit(Sb, slot) << k;
              wd |= (unsigned long long)tbit(Db, slot) << k;
            }
            Sf[f] = ws;
            Df[f] = wd;
          }
        }
      }
      if (!__syncthreads_or(grew)) break;
      if (round >= Q.max_iters) {
        if (threadIdx.x == 0) atomicExch(cap_hit, 1);
        break;
      }
      ++round;
    }
    if (threadIdx.x == 0) rounds_out[s] = round;
    // the final relation -> dense store of the packed layout (present slots only)
    TILE_UNROLL
      for (int li = 0; li < TP(F).nlocal; ++li) {
      const TileRel& H = TP(F).rel[TP(F).local_rel[li]];
        const TileRel& HQ = Q.rel[TP(F).local_rel[li]];
      const uint32_t* Sb = reinterpret_cast<const uint32_t*>(sm + H.sm_bits[0]);
      const uint32_t* Db = reinterpret_cast<const uint32_t*>(sm + H.sm_bits[1]);
      const float* St = reinterpret_cast<const float*>(sm + H.sm_tag[0]);
      uint32_t cnt = 0;
      for (int h = threadIdx.x; h < H.D; h += blockDim.x) {
        if (!tbit(Sb, h)) continue;  // Δ' was empty: S holds every tuple
        ++cnt;
        (void)Db;
        uint64_t pk = (uint64_t)s << H.psshift;
        int x = h;
        for (int c = H.ncols - 1; c >= 0; --c) {
          pk |= (uint64_t)(x % H.dom[c]) << H.pshift[c];
          x /= H.dom[c];
        }
        if constexpr (SEMI == TILE_S_UNIT) atomicOr(HQ.dfbits + (pk >> 5), 1u << (pk & 31u));
        else HQ.dfp[pk] = St[h];
      }
      cnt = __reduce_add_sync(~0u, cnt);
      if (lane == 0 && cnt) atomicAdd(Q.counts + li, (unsigned long long)cnt);
    }
    __syncthreads();
  }
  // candidates: one atomic per warp
  for (int o = 16; o; o >>= 1) my_cand += __shfl_down_sync(~0u, my_cand, o);
  if (lane == 0 && my_cand) atomicAdd(ncand, (unsigned long long)my_cand);
}

}  // namespace lob
