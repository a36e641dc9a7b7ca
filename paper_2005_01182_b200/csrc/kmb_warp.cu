// Warp engine: ONE WARP PER INSTANCE for batched small problems (BASELINE
// config 3: 4096 independent n = 128 solves).  Same algorithm as the grid
// engine (kmb_solver.cu) with a single column owner: lane l owns columns
// [CPL*l, CPL*l + CPL), so every per-column minimum stays in registers and the
// whole search is warp-synchronous — no block barrier, no shared atomics on
// the hot path, __reduce_min_sync (one REDUX) for the min-slack reduction.
//
// Reference path replaced: ot::solve_batched_km (hungarian.cpp:313-381) /
// ot::solve_km (:55-136) per instance.  Rounds restate hungarian.cpp:175-217
// (relax :164-172, absorb :186-199, delta + dual step :203-215, applied lazily);
// augmentation along the argmin-parent forest replaces TightPhase (:223-309);
// seed 1 = the reductions of :323-333.
//
// Arithmetic: costs in [0, 2^29) keep every dual, D and slack' inside int32
// (|u|, |v|, D <= maxC; slack' <= 3 maxC); the packed (value, row) key is 64-bit.
//
// Cost source: rows stream from global memory (L1/L2) with 128-bit loads, which
// leaves shared memory to per-instance state only, so a whole config-3 batch
// (4096 instances) is resident in one wave.  (Staging each matrix in shared
// memory by TMA fits 3 instances per SM: 9 waves, 3.2 ms; 16-bit row offsets
// halve the streamed bytes but cost an extra pass and unpacking: 1.117 vs
// 1.001 ms.  Both measured in round 1 and removed.)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kmb_common.cuh"
#include "kmb_internal.h"
#include "kmb_launch.h"

namespace kmb {

namespace {

// Build-time constants (A/B measured on config 3 in round 1, tools/ab_lib.py):
//   rows per relax batch: 72-register build 5 (4: 1.09, 5: 1.065, 6-8: 1.12 ms,
//   ptxas folds early rows of a longer batch before its later loads issue);
//   low-occupancy build 8 (2048 / 1536 batches .639 / .571 ms vs .664 / .598 at 5)
constexpr int kRB7 = 5, kRB4 = 8;
// rows per relax batch over the 16-bit resident copy (two registers a row)
#ifndef KMB_WARP_RB16_7
#define KMB_WARP_RB16_7 6
#endif
#ifndef KMB_WARP_RB16_4
#define KMB_WARP_RB16_4 8
#endif
constexpr int kRB16_7 = KMB_WARP_RB16_7, kRB16_4 = KMB_WARP_RB16_4;
// KMB_WARP_STAGE_CLOCKS (diagnostics): per-stage clock64 accounting
// (kmb_last_instance_stats columns 5-8); costs ~3%, off in production
#ifndef KMB_WARP_ROOMY8
#define KMB_WARP_ROOMY8 1
#endif
#ifndef KMB_WARP_STAGE_CLOCKS
#define KMB_WARP_STAGE_CLOCKS 0
#endif

// claim word for n <= 256: smaller is better; stamp decreases with the epoch
__device__ __forceinline__ uint32_t wclaim(int phase, int col) {
  return (static_cast<uint32_t>(0xFFFFFE - phase) << 8) | static_cast<uint32_t>(col);
}
__device__ __forceinline__ bool wclaimed_in(uint32_t c, int phase) {
  return (c >> 8) == static_cast<uint32_t>(0xFFFFFE - phase);
}

template <int CPL>
struct RowVec {
  int32_t x[CPL];
};

// Loads the lane's CPL columns of one row.  The pitch is padded to the warp
// width (32 * CPL), so every lane's vector load is in bounds; padding columns
// read whatever the pad holds and are masked as "reached".
template <int CPL>
__device__ __forceinline__ RowVec<CPL> load_row(const int32_t* p) {
  RowVec<CPL> r;
  if constexpr (CPL >= 4) {
#pragma unroll
    for (int h = 0; h < CPL / 4; ++h) {
      const int4 t = __ldg(reinterpret_cast<const int4*>(p) + h);
      r.x[4 * h + 0] = t.x; r.x[4 * h + 1] = t.y; r.x[4 * h + 2] = t.z; r.x[4 * h + 3] = t.w;
    }
  } else if constexpr (CPL == 2) {
    const int2 t = __ldg(reinterpret_cast<const int2*>(p));
    r.x[0] = t.x; r.x[1] = t.y;
  } else {
    r.x[0] = __ldg(p);
  }
  return r;
}

// 16-bit resident rows: CPL offsets from the row minimum (same warp-width
// pitch, 2 * CPL bytes a lane), returned already in key position (d << 8) -
// one PRMT each.  Plain (coherent) loads: the copy is written by this kernel.
template <int CPL>
struct RowVec16 {
  uint32_t x[CPL / 2];
};
template <int CPL>
__device__ __forceinline__ RowVec16<CPL> load_row16(const char* p) {
  static_assert(CPL == 4 || CPL == 8, "16-bit rows need 4 or 8 columns per lane");
  RowVec16<CPL> r;
  if constexpr (CPL == 8) {
    const uint4 t = *reinterpret_cast<const uint4*>(p);
    r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
  } else {
    const uint2 t = *reinterpret_cast<const uint2*>(p);
    r.x[0] = t.x; r.x[1] = t.y;
  }
  return r;
}
// Key-position offsets (d << 8) + tag of the two halves of a packed word: one
// PRMT each; the caller's fused add-min (VIADDMNMX) takes the tag.  Doing the unpack
// on the FMA pipe instead (mul.lo / mad.hi by powers of two; ptxas keeps a
// LEA.HI) was measured slower: 0.913 vs 0.899 ms on config 3.
__device__ __forceinline__ uint32_t lo16_key(uint32_t x) { return __byte_perm(x, 0u, 0x4104); }
__device__ __forceinline__ uint32_t hi16_key(uint32_t x) { return __byte_perm(x, 0u, 0x4324); }

}  // namespace

// Per-warp shared state (n <= 256), in 32-bit words: two row lists of (row,
// tag) pairs (4n; the free columns found in an epoch live in the idle list) +
// u, w, root_row, match_row, match_col, tree_par, claim (7n).  Kept small: what
// the CTAs per SM do not take of the unified cache is L1 for the streamed
// matrices.
// (+ n with the 16-bit resident copy: each row's minimum, bit 31 = the row does
// not fit 16 bits and is relaxed from the int32 matrix)
// The arrays are strided by the padded size 32 * CPL for n <= 128 (compile-time
// offsets from one base register instead of multiplies by n on every round's
// critical path), by n above (12 KB a warp would cost residency).
__host__ __device__ constexpr int warp_state_stride(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n; }
__host__ __device__ constexpr int warp_state_words(int n, bool u16) { return (u16 ? 12 : 11) * warp_state_stride(n); }

// Column keys.  Wide: ((c - w + 2^30) << 32) | row (any n, costs < 2^29).
// Narrow (n <= 256, costs < 2^21): ((c - w + 2^22) << 8) | row in 32 bits, so a
// relaxation is one shift-add and one unsigned min.  A row's tag is fixed when
// it is reached (w is constant while it stays reached): wide tag = 2^30 - w,
// narrow tag = ((2^22 - w) << 8) | row.  Both orders are (value, row): the
// same argmin and tie-breaking.
template <bool NARROW>
struct Keys;
template <>
struct Keys<false> {
  using K = uint64_t;
  static constexpr K INF = ~0ull;
  __device__ static uint32_t tag(int32_t w, int32_t) {
    return static_cast<uint32_t>(static_cast<int32_t>(KMB_BIAS) - w);
  }
  __device__ static K make(int32_t c, uint32_t tag, int32_t row) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(c) + tag) << 32) | static_cast<uint32_t>(row);
  }
  __device__ static int32_t val(K k) { return static_cast<int32_t>(static_cast<int64_t>(k >> 32) - KMB_BIAS); }
  static constexpr int32_t VOFF = 0;  // the search keeps v + VOFF per column
  __device__ static int32_t slack(K k, int32_t vq) { return val(k) - vq; }
  __device__ static int32_t row(K k) { return static_cast<int32_t>(static_cast<uint32_t>(k)); }
  __device__ static K kmin(K a, K b) { return a < b ? a : b; }
  __device__ static K from_wide(uint64_t k) { return k; }
  // row-list entry: (row, tag); the row's byte offset is row * pitch bytes
  __device__ static int2 ent(int32_t row, uint32_t tag, uint32_t) { return make_int2(row, static_cast<int32_t>(tag)); }
  __device__ static int32_t erow(int2 e) { return e.x; }
  __device__ static uint32_t eoff(int2 e, uint32_t pb) { return static_cast<uint32_t>(e.x) * pb; }
};
template <>
struct Keys<true> {
  using K = uint32_t;
  static constexpr K INF = 0xffffffffu;
  static constexpr int32_t NB = 1 << 22;
  __device__ static uint32_t tag(int32_t w, int32_t row) {
    return (static_cast<uint32_t>(NB - w) << 8) | static_cast<uint32_t>(row);
  }
  __device__ static K make(int32_t c, uint32_t tag, int32_t) {
    return (static_cast<uint32_t>(c) << 8) + tag;
  }
  __device__ static int32_t val(K k) { return static_cast<int32_t>(k >> 8) - NB; }
  static constexpr int32_t VOFF = NB;  // v is kept with the key bias added: slack' is one shift-subtract
  __device__ static int32_t slack(K k, int32_t vq) { return static_cast<int32_t>(k >> 8) - vq; }
  __device__ static int32_t row(K k) { return static_cast<int32_t>(k & 0xffu); }
  __device__ static K kmin(K a, K b) { return min(a, b); }
  // a wide key (c - w + 2^30, row) as a narrow one (c - w + 2^22, row)
  __device__ static K from_wide(uint64_t k) {
    if (k == Keys<false>::INF) return INF;
    return (static_cast<uint32_t>(Keys<false>::val(k) + NB) << 8) | static_cast<uint32_t>(k & 0xffu);
  }
  // row-list entry: (byte offset of the row, tag); the tag's low byte is the
  // row, so the relax adds the offset to the lane's base and nothing else
  // (5 address instructions per row -> 2, SASS)
  __device__ static int2 ent(int32_t row, uint32_t tag, uint32_t pb) {
    return make_int2(static_cast<int32_t>(static_cast<uint32_t>(row) * pb), static_cast<int32_t>(tag));
  }
  __device__ static int32_t erow(int2 e) { return e.y & 0xff; }
  __device__ static uint32_t eoff(int2 e, uint32_t) { return static_cast<uint32_t>(e.x); }
};

struct WarpSmem {
  int32_t *u, *w, *root_row, *match_row, *match_col, *tree_par;
  int32_t* ctr;  // [0] rows tail, [1] free columns found this epoch
  uint32_t* claim;
  int32_t* rminw;      // 16-bit mode only
  int2 *rows, *spare;  // (row, tag)
};

// One instance, whole warp.  Returns the status (0 ok, -2 internal).
// RB: rows per relax batch; CACHE: matched rows and their u in registers
// U16 (narrow keys only): relax from the 16-bit resident copy C16m
template <int CPL, bool NARROW, int RB, bool CACHE, bool U16 = false, int RB16 = 8>
__device__ __forceinline__ int solve_instance(const WarpArgs& a, const int32_t* Cm, int inst,
                                              const WarpSmem& S, int lane, const uint64_t (&k0)[CPL],
                                              const uint16_t* C16m = nullptr) {
  static_assert(!U16 || NARROW, "the 16-bit copy goes with narrow keys");
  using KO = Keys<NARROW>;
  using K = typename KO::K;
  constexpr uint32_t FULL = 0xffffffffu;
  const int n = a.n;
  constexpr uint32_t np = 32u * CPL;  // == a.pitch (launch_warp_batch checks it)
  constexpr uint32_t pb = 4u * np;    // row pitch in bytes
  const int c0 = CPL * lane;
  const char* const lb = reinterpret_cast<const char*>(Cm + c0);  // this lane's columns of row 0
  const char* const lb16 = reinterpret_cast<const char*>(C16m + c0);
  // Row-list entry of row i reached with w.  16-bit mode: the byte offset is
  // the row's in the 16-bit copy and the tag folds the row minimum in,
  // key = (d << 8) + tag' with d = C - rowmin; a row that does not fit 16 bits
  // keeps its int32 offset with bit 31 set and the plain tag.
  auto mk_ent = [&](int32_t i, int32_t wi) {
    if constexpr (U16) {
      const int32_t rm = S.rminw[i];
      const uint32_t t = KO::tag(wi, i);
      if (rm < 0) return make_int2(static_cast<int32_t>((static_cast<uint32_t>(i) * pb) | 0x80000000u), static_cast<int32_t>(t));
      return make_int2(static_cast<int32_t>(static_cast<uint32_t>(i) * (pb >> 1)),
                       static_cast<int32_t>(t + (static_cast<uint32_t>(rm) << 8)));
    } else {
      return KO::ent(i, KO::tag(wi, i), pb);
    }
  };
  int32_t* const u = S.u;
  int32_t* const w = S.w;
  int32_t* const root_row = S.root_row;
  int32_t* const match_row = S.match_row;
  int32_t* const match_col = S.match_col;
  int32_t* const tree_par = S.tree_par;
  uint32_t* const claim = S.claim;
  int2* rows = S.rows;
  int2* spare = S.spare;
  int32_t* found = reinterpret_cast<int32_t*>(spare);  // idle row list during an epoch

  for (int k = lane; k < n; k += 32) rows[k] = mk_ent(k, w[k]);
  if (lane == 0) {
    S.ctr[0] = n;
    S.ctr[1] = 0;
  }
  K key[CPL];
  int32_t v[CPL], dc[CPL];
  uint32_t pad = 0;
  // Narrow keys: a reached (or padding) column's v carries -RBIG while it is
  // reached, so its slack' = val - v sits near 2^29: never the minimum, never
  // equal to D (< 2^22) - the min and the tight test need no reached mask.
  // (Wide keys: slack' reaches 3 * 2^29, no headroom; they keep the mask.)
  constexpr int32_t RBIG = NARROW ? (1 << 29) : 0;
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    v[q] = KO::VOFF;
    dc[q] = 0;
    key[q] = KO::from_wide(k0[q]);  // every row relaxed once by the validation pass
    if (c0 + q >= n) {
      pad |= 1u << q;
      v[q] = KO::VOFF - RBIG;
    }
  }
  if (a.seed == 1) {  // column reduction, :328-333 (the keys already hold every row's u0-reduced costs)
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (!((pad >> q) & 1)) v[q] = KO::val(key[q]) + KO::VOFF;
  }
  uint32_t rch = pad;  // bit q: column c0+q reached (padding counts as reached)
  // CACHE (low-occupancy build): each column's matched row and its u in
  // registers between epoch ends (both change only there)
  int32_t mi2[CACHE ? CPL : 1], mu2[CACHE ? CPL : 1];
#pragma unroll
  for (int q = 0; q < (CACHE ? CPL : 1); ++q) {
    mi2[q] = -1;
    mu2[q] = 0;
  }
  int nrows = n, head = n, nfree = n;  // rows[0, nrows) reached; [head, nrows) to relax
  int32_t D = 0;
  int epochs = 0, dual_steps = 0, rows_scanned = n, rounds = 0;
  int status = 0;
  bool stuck = false;
  constexpr int round_cap = 4 * 256 * 256 + 64;  // n <= 256; an immediate (4 n^2 + 64 was recomputed every round)
  const long long t_start = clock64();
  long long cyc[4] = {0, 0, 0, 0};  // relax, min, absorb, epoch end
  long long tl = t_start;
#if KMB_WARP_STAGE_CLOCKS
#define KMB_WSTAGE(k)                 \
  do {                                \
    const long long t_ = clock64();   \
    cyc[k] += t_ - tl;                \
    tl = t_;                          \
  } while (0)
#else
#define KMB_WSTAGE(k) (void)tl
#endif
  __syncwarp();

  while (nfree > 0) {
    // a valid search ends in n epochs of <= 2n + 1 rounds and always has an
    // unreached column while a row is free
    if (++rounds > round_cap || stuck) {
      status = -2;
      break;
    }
    // ---- relax rows[head, nrows)  (hungarian.cpp:164-172) ----
    int r = head;
    if constexpr (U16) {
      // one row folded from the 16-bit copy (tag' in e.y) or, bit 31 of the
      // offset set, from the int32 matrix (plain tag)
      auto fold16 = [&](int2 e, const RowVec16<CPL>& cv) {
#pragma unroll
        for (int h = 0; h < CPL / 2; ++h) {
          // min((d << 8) + tag', key): the DPX add-min, one VIADDMNMX per column
          key[2 * h] = __viaddmin_u32(lo16_key(cv.x[h]), static_cast<uint32_t>(e.y), key[2 * h]);
          key[2 * h + 1] = __viaddmin_u32(hi16_key(cv.x[h]), static_cast<uint32_t>(e.y), key[2 * h + 1]);
        }
      };
      auto fold_any = [&](int2 e) {  // rare rows (warp-uniform branch)
        if (e.x < 0) {
          const RowVec<CPL> c32 = load_row<CPL>(reinterpret_cast<const int32_t*>(lb + (static_cast<uint32_t>(e.x) & 0x7fffffffu)));
#pragma unroll
          for (int q = 0; q < CPL; ++q) key[q] = KO::kmin(key[q], KO::make(c32.x[q], static_cast<uint32_t>(e.y), 0));
        } else {
          fold16(e, load_row16<CPL>(lb16 + static_cast<uint32_t>(e.x)));
        }
      };
      // RB16 rows in flight: entries, then all row loads, then the folds
      for (; r + RB16 <= nrows; r += RB16) {
        int2 e[RB16];
        int32_t anyw = 0;
#pragma unroll
        for (int k = 0; k < RB16; ++k) {
          e[k] = rows[r + k];
          anyw |= e[k].x;
        }
        if (anyw >= 0) {
          RowVec16<CPL> cv[RB16];
#pragma unroll
          for (int k = 0; k < RB16; ++k) cv[k] = load_row16<CPL>(lb16 + static_cast<uint32_t>(e[k].x));
#pragma unroll
          for (int k = 0; k < RB16; ++k) fold16(e[k], cv[k]);
        } else {
#pragma unroll
          for (int k = 0; k < RB16; ++k) fold_any(e[k]);
        }
      }
      if (nrows - r == 1) {
        fold_any(rows[r]);
      } else {
        // 2..RB16-1 rows: batches of TB with the last row repeated (the fold is idempotent)
        constexpr int TB = 4;
        for (; r < nrows; r += TB) {
          int2 e[TB];
          int32_t anyw = 0;
#pragma unroll
          for (int k = 0; k < TB; ++k) {
            e[k] = rows[min(r + k, nrows - 1)];
            anyw |= e[k].x;
          }
          if (anyw >= 0) {
            RowVec16<CPL> cv[TB];
#pragma unroll
            for (int k = 0; k < TB; ++k) cv[k] = load_row16<CPL>(lb16 + static_cast<uint32_t>(e[k].x));
#pragma unroll
            for (int k = 0; k < TB; ++k) fold16(e[k], cv[k]);
          } else {
#pragma unroll
            for (int k = 0; k < TB; ++k) fold_any(e[k]);
          }
        }
      }
    } else {
      // RB rows in flight: entries, then all row loads, then the folds
      for (; r + RB - 1 < nrows; r += RB) {
        int2 e[RB];
        RowVec<CPL> cv[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) e[k] = rows[r + k];
#pragma unroll
        for (int k = 0; k < RB; ++k) cv[k] = load_row<CPL>(reinterpret_cast<const int32_t*>(lb + KO::eoff(e[k], pb)));
#pragma unroll
        for (int k = 0; k < RB; ++k)
#pragma unroll
          for (int q = 0; q < CPL; ++q)
            key[q] = KO::kmin(key[q], KO::make(cv[k].x[q], static_cast<uint32_t>(e[k].y), KO::erow(e[k])));
      }
      if (nrows - r == 1) {
        const int2 e = rows[r];
        const RowVec<CPL> cv = load_row<CPL>(reinterpret_cast<const int32_t*>(lb + KO::eoff(e, pb)));
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          key[q] = KO::kmin(key[q], KO::make(cv.x[q], static_cast<uint32_t>(e.y), KO::erow(e)));
      } else if (r < nrows) {
        // 2..RB-1 rows: one batch with the last row repeated (the fold is
        // idempotent), so all loads are in flight together
        int2 e[RB];
        RowVec<CPL> cv[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) e[k] = rows[min(r + k, nrows - 1)];
#pragma unroll
        for (int k = 0; k < RB; ++k) cv[k] = load_row<CPL>(reinterpret_cast<const int32_t*>(lb + KO::eoff(e[k], pb)));
#pragma unroll
        for (int k = 0; k < RB; ++k)
#pragma unroll
          for (int q = 0; q < CPL; ++q)
            key[q] = KO::kmin(key[q], KO::make(cv[k].x[q], static_cast<uint32_t>(e[k].y), KO::erow(e[k])));
      }
    }
    r = nrows;
    rows_scanned += nrows - head;
    head = nrows;
    KMB_WSTAGE(0);
    // ---- min unreached slack' (hungarian.cpp:203-206) ----
    int32_t s[CPL];
    int32_t lm = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      s[q] = KO::slack(key[q], v[q]);
      if (NARROW || !((rch >> q) & 1)) lm = min(lm, s[q]);
    }
    const int32_t m = __reduce_min_sync(FULL, lm);
    // dual step (hungarian.cpp:207-215), applied lazily; no unreached column
    // left (an engine fault) ends the search at the next loop head
    stuck = NARROW ? m >= (RBIG >> 1) : m == 0x7fffffff;
    if (m > D && !stuck) {
      D = m;
      ++dual_steps;
    }
    KMB_WSTAGE(1);
    // ---- absorb zero-slack columns (hungarian.cpp:186-199) ----
    // Usually one column per round turns tight: only its lane branches in, and
    // appends go through warp-private shared counters (no per-column ballots).
    // (narrow keys: a lane holds a tight column exactly when its minimum is D)
    uint32_t tm = 0;
    if constexpr (!NARROW) {
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (!((rch >> q) & 1) && s[q] == D) tm |= 1u << q;
    }
    // (Numbering the slots in the single tight lane of the usual round and
    // broadcasting the totals - a ballot and two shuffles instead of the shared
    // atomics and the counter reads - was measured slower: 0.864 -> 0.910 ms.)
    if (NARROW ? lm == D : tm != 0) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        if (NARROW ? s[q] != D : !((tm >> q) & 1)) continue;
        rch |= 1u << q;
        const int col = c0 + q;
        dc[q] = D;
        v[q] -= RBIG;
        const int32_t par = KO::row(key[q]);
        tree_par[col] = par;
        const int32_t root = root_row[par];
        const int32_t i2 = CACHE ? mi2[CACHE ? q : 0] : match_col[col];
        if (i2 < 0) {
          atomicMin(claim + root, wclaim(epochs, col));
          found[atomicAdd(S.ctr + 1, 1)] = col;
        } else {
          const int32_t w2 = (CACHE ? mu2[CACHE ? q : 0] : u[i2]) - D;
          w[i2] = w2;
          root_row[i2] = root;
          rows[atomicAdd(S.ctr, 1)] = mk_ent(i2, w2);
        }
      }
    }
    __syncwarp();
    nrows = S.ctr[0];
    const int nfound = S.ctr[1];
    KMB_WSTAGE(2);
    if (nfound == 0) continue;

    // ---- epoch end: augment and dissolve the trees that reached a free column.
    // Columns (lane-owned): finalise dissolved ones; reset keys whose argmin row
    // leaves the search.
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      if ((pad >> q) & 1) continue;
      const int col = c0 + q;
      if ((rch >> q) & 1) {
        if (wclaimed_in(claim[root_row[tree_par[col]]], epochs)) {
          v[q] -= D - dc[q] - RBIG;
          rch &= ~(1u << q);
          key[q] = KO::INF;
        }
      } else if (key[q] != KO::INF && wclaimed_in(claim[root_row[KO::row(key[q])]], epochs)) {
        key[q] = KO::INF;
      }
    }
    // flip one parent-pointer path per claimed tree (its smallest free column)
    int won = 0;
    for (int fb = 0; fb < nfound; fb += 32) {
      const int f = fb + lane;
      bool winner = false;
      if (f < nfound) {
        int32_t j = found[f];
        if (claim[root_row[tree_par[j]]] == wclaim(epochs, j)) {
          winner = true;
          for (;;) {
            const int32_t i = tree_par[j];
            const int32_t nx = match_row[i];
            match_row[i] = j;
            match_col[j] = i;
            if (nx < 0) break;
            j = nx;
          }
        }
      }
      won += __popc(__ballot_sync(FULL, winner));
    }
    __syncwarp();  // found[] (the idle list) is read; the compaction overwrites it
    // rows: finalise dissolved ones (u = w + D), compact the survivors
    int ns = 0;
    for (int rb = 0; rb < nrows; rb += 32) {
      const int rr = rb + lane;
      bool keep = false;
      int2 e = make_int2(0, 0);
      if (rr < nrows) {
        e = rows[rr];
        const int32_t er = KO::erow(e);
        if (wclaimed_in(claim[root_row[er]], epochs)) u[er] = w[er] + D;
        else keep = true;
      }
      const uint32_t km = __ballot_sync(FULL, keep);
      if (keep) spare[ns + __popc(km & ((1u << lane) - 1))] = e;
      ns += __popc(km);
    }
    if (lane == 0) {
      S.ctr[0] = ns;
      S.ctr[1] = 0;
    }
    __syncwarp();
    nfree -= won;
    if constexpr (CACHE) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        mi2[q] = (pad >> q) & 1 ? -1 : match_col[c0 + q];
        mu2[q] = mi2[q] >= 0 ? u[mi2[q]] : 0;
      }
    }
    int2* t = rows;
    rows = spare;
    spare = t;
    found = reinterpret_cast<int32_t*>(spare);
    nrows = ns;
    head = 0;  // survivors relax once more for the reset columns
    ++epochs;
    KMB_WSTAGE(3);
  }
#undef KMB_WSTAGE
  const long long cycles = clock64() - t_start;
  // ---- outputs ----
  int64_t tot = 0;
  for (int k = lane; k < n; k += 32) {
    const int32_t mr = match_row[k];
    a.row_to_col[static_cast<int64_t>(inst) * n + k] = mr;
    a.u[static_cast<int64_t>(inst) * n + k] = u[k];
    if (mr >= 0) tot += __ldg(Cm + k * np + mr);
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q)
    if (c0 + q < n) a.v[static_cast<int64_t>(inst) * n + c0 + q] = v[q] - KO::VOFF + (((rch >> q) & 1) ? RBIG : 0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
  if (lane == 0) {
    a.total_cost[inst] = tot;
    if (a.stats) {
      int64_t* o = a.stats + KMB_ISTATS * static_cast<int64_t>(inst);
      o[0] = epochs;
      o[1] = dual_steps;
      o[2] = rows_scanned;
      o[3] = rounds;
      o[4] = cycles;
      for (int k = 0; k < 4; ++k) o[5 + k] = cyc[k];
    }
  }
  return status;
}

// MINB: resident CTAs per SM the build targets — 7 (72 registers: a 4096
// config-3 batch resident in one wave) or 4 (128 registers, deeper relax
// batches, matched rows cached in registers) for batches that need at most 16
// warps per SM
template <int CPL, int MINB = 7>
__global__ void __launch_bounds__(128, MINB) k_warp_batch(WarpArgs a) {
  // 8 columns a lane, 128-register build: 4 int32 rows / 8 16-bit rows per
  // batch (n = 256 x 4,096, 16-bit rows: 3.26 ms at 4, 2.89 at 8, 3.01 at 10,
  // 2.91 at 12; 6 int32 rows: n = 256 x 1,024 1.52 -> 1.62)
#ifndef KMB_WARP_RB8L
#define KMB_WARP_RB8L 4
#endif
#ifndef KMB_WARP_RB16_8L
#define KMB_WARP_RB16_8L 8
#endif
  constexpr int RB = CPL > 4 ? (MINB >= 7 ? 4 : KMB_WARP_RB8L) : (MINB >= 7 ? kRB7 : kRB4);
  constexpr int RB16 = CPL > 4 ? (MINB >= 7 ? 4 : KMB_WARP_RB16_8L) : (MINB >= 7 ? kRB16_7 : kRB16_4);
  constexpr bool CK = MINB < 7;
  // 16-bit resident copy (a.C16): written by the validation pass, read by every
  // later relax - half the bytes per row and half the L2 footprint of a batch
  // that does not fit the L2 as int32
  constexpr bool kU16able = CPL == 4 || CPL == 8;
  const bool use16 = kU16able && a.C16 != nullptr;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;  // warp in block
  const int wpb = blockDim.x >> 5;
  const int n = a.n;
  constexpr int np = 32 * CPL;  // == a.pitch (launch_warp_batch checks it)
  constexpr uint32_t FULL = 0xffffffffu;

  // carve this warp's slice: [2 counters | state]
  const size_t wbytes = static_cast<size_t>(warp_state_words(n, use16)) * 4 + 16;
  unsigned char* base = dyn + wib * ((wbytes + 15) & ~static_cast<size_t>(15));
  int32_t* ctr = reinterpret_cast<int32_t*>(base);
  int32_t* st = reinterpret_cast<int32_t*>(base + 16);
  WarpSmem S;
  const int sn = CPL <= 4 ? 32 * CPL : n;  // == warp_state_stride(n)
  S.rows = reinterpret_cast<int2*>(st);  // 8-byte aligned first
  S.spare = S.rows + sn;
  S.u = reinterpret_cast<int32_t*>(S.spare + sn);
  S.w = S.u + sn;
  S.root_row = S.w + sn;
  S.match_row = S.root_row + sn;
  S.match_col = S.match_row + sn;
  S.tree_par = S.match_col + sn;
  S.claim = reinterpret_cast<uint32_t*>(S.tree_par + sn);
  S.rminw = reinterpret_cast<int32_t*>(S.claim + sn);  // 16-bit mode only
  S.ctr = ctr;
  const int c0 = CPL * lane;

  for (int inst = blockIdx.x * wpb + wib; inst < a.batch; inst += gridDim.x * wpb) {
    const unsigned long long t_inst0 = globaltimer_ns();
#ifdef KMB_WARP_ALIAS  // diagnostics: instances share KMB_WARP_ALIAS matrices (L2 footprint probe; outputs of aliased instances repeat)
    const int32_t* Cm = a.C + static_cast<int64_t>(inst % KMB_WARP_ALIAS) * n * np;
#else
    const int32_t* Cm = a.C + static_cast<int64_t>(inst) * n * np;
#endif
    for (int k = lane; k < n; k += 32) {
      S.match_row[k] = -1;
      S.match_col[k] = -1;
      S.claim[k] = 0xFFFFFFFFu;
      S.root_row[k] = k;
    }
    __syncwarp();
    // validation (core.cpp:144-145 + device range) and row reductions
    // (hungarian.cpp:323-327): the warp walks the rows, lanes across columns,
    // IB rows in flight (loads first, then the per-row reductions)
    // The same pass is the search's first relax (every row reached at D = 0
    // with w = u0): the keys are folded here, in the wide (value, row) form
    // the key width is picked from afterwards, so the matrix is read once less.
    uint16_t* const C16m = use16 ? a.C16 + static_cast<int64_t>(inst) * n * np : nullptr;
    // per instance: packing stops (and the solve reads int32 rows) once more
    // than ~n/16 rows have a range beyond 16 bits - such rows are relaxed from
    // the int32 matrix anyway, one at a time
    bool pack = use16;
    int nwide = 0;
    int32_t lo_all = 0x7fffffff, hi_all = 0;
    uint64_t k0[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) k0[q] = Keys<false>::INF;
    constexpr int IB = CPL >= 8 ? 4 : 8;  // rows in flight (8 columns a lane: fewer, spills)
    for (int i0 = 0; i0 < n; i0 += IB) {
      RowVec<CPL> cv[IB];
#pragma unroll
      for (int k = 0; k < IB; ++k) cv[k] = load_row<CPL>(Cm + static_cast<int64_t>(min(i0 + k, n - 1)) * np + c0);
#pragma unroll
      for (int k = 0; k < IB; ++k) {
        const int i = i0 + k;
        if (i >= n) break;  // warp-uniform
        int32_t lo = 0x7fffffff, hi = 0;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (c0 + q < n) {
            lo = min(lo, cv[k].x[q]);
            hi = max(hi, cv[k].x[q]);
          }
        lo = __reduce_min_sync(FULL, lo);
        lo_all = min(lo_all, lo);
        hi_all = max(hi_all, hi);
        const int32_t u0 = a.seed == 1 ? lo : 0;
        const uint32_t tag = Keys<false>::tag(u0, i);
#pragma unroll
        for (int q = 0; q < CPL; ++q) k0[q] = Keys<false>::kmin(k0[q], Keys<false>::make(cv[k].x[q], tag, i));
        if (lane == (i & 31)) {
          S.u[i] = u0;
          S.w[i] = u0;
        }
        if constexpr (kU16able) {
          if (pack) {  // d = C - rowmin, saturated; a saturated valid column marks the row
            uint32_t d[CPL];
            bool sat = false;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
              const uint32_t x = static_cast<uint32_t>(cv[k].x[q]) - static_cast<uint32_t>(lo);
              d[q] = x >= 65535u ? 65535u : x;
              sat |= (c0 + q < n) && x >= 65535u;
            }
            sat = __any_sync(FULL, sat);
            uint16_t* out = C16m + static_cast<int64_t>(i) * np + c0;
            if constexpr (CPL == 8) {
              *reinterpret_cast<uint4*>(out) = make_uint4(d[0] | (d[1] << 16), d[2] | (d[3] << 16),
                                                          d[4] | (d[5] << 16), d[6] | (d[7] << 16));
            } else {
              *reinterpret_cast<uint2*>(out) = make_uint2(d[0] | (d[1] << 16), d[2] | (d[3] << 16));
            }
            if (lane == (i & 31)) S.rminw[i] = sat ? (lo | static_cast<int32_t>(0x80000000u)) : lo;
            nwide += sat;
          }
        }
      }
      if (nwide * 16 > n + 16) pack = false;
    }
    hi_all = __reduce_max_sync(FULL, hi_all);
    int status = lo_all < 0 ? 2 : (hi_all >= (1 << 29) ? 3 : 0);
    __syncwarp();
    if (status == 0) {
      if (hi_all >= (1 << 21)) {
        status = solve_instance<CPL, false, RB, CK>(a, Cm, inst, S, lane, k0);
      } else if (kU16able && pack) {
        if constexpr (kU16able) status = solve_instance<CPL, true, RB, CK, true, RB16>(a, Cm, inst, S, lane, k0, C16m);
      } else {
        status = solve_instance<CPL, true, RB, CK>(a, Cm, inst, S, lane, k0);
      }
    } else {
      for (int k = lane; k < n; k += 32) a.row_to_col[static_cast<int64_t>(inst) * n + k] = -1;
      if (lane == 0) a.total_cost[inst] = 0;
    }
    if (lane == 0) {
      a.status[inst] = status;
      if (a.stats) {
        a.stats[KMB_ISTATS * static_cast<int64_t>(inst) + 9] = static_cast<int64_t>(t_inst0);
        a.stats[KMB_ISTATS * static_cast<int64_t>(inst) + 10] = static_cast<int64_t>(globaltimer_ns());
      }
    }
    __syncwarp();
  }
}

int warp_max_n() { return 256; }

size_t warp_smem_per_warp(int n, bool u16) {
  return (static_cast<size_t>(warp_state_words(n, u16)) * 4 + 16 + 15) & ~static_cast<size_t>(15);
}

template <int CPL, int MINB = 7>
static cudaError_t launch_t(const WarpArgs& a, int sm_count, int wpb, int warps_per_sm,
                            cudaStream_t st, int* grid_out) {
  if constexpr (MINB == 7 && CPL >= 4) {
    // a batch that needs at most 4 CTAs (16 warps) per SM runs the 128-register
    // instance (config-3 shards of <= 2,368 instances); so does one whose
    // per-warp state leaves room for no more than 4 CTAs anyway (n > ~190: the
    // 72-register build of 8 columns a lane spills)
    const size_t smem4 = warp_smem_per_warp(a.n, (CPL == 4 || CPL == 8) && a.C16 != nullptr) * wpb + 1024;
    const bool few = (a.batch + wpb - 1) / wpb <= 4 * sm_count;
    const bool roomy = CPL == 8 && KMB_WARP_ROOMY8 && 5 * smem4 > 227 * 1024;
    if (warps_per_sm == 0 && (few || roomy))
      return launch_t<CPL, 4>(a, sm_count, wpb, warps_per_sm, st, grid_out);
  }
  auto kern = k_warp_batch<CPL, MINB>;
  const size_t smem = warp_smem_per_warp(a.n, (CPL == 4 || CPL == 8) && a.C16 != nullptr) * wpb;
  // Shared-memory carveout: just the state of the CTAs per SM this launch
  // needs (all instances resident in one wave, at most the register limit),
  // +1 KiB reserved per CTA; the rest of the unified cache is L1, which keeps
  // part of each streamed matrix close (config 3: 1.064 -> 1.004 ms with a
  // 196 KB carveout instead of the maximum; the longest instance alone 0.61 ->
  // 0.48 ms).  Registers per thread are read once per instantiation.
  static int regs_cached[2][4] = {};  // benign race: every thread computes the same value
  int& regs = regs_cached[MINB == 7 ? 0 : 1][CPL == 1 ? 0 : CPL == 2 ? 1 : CPL == 4 ? 2 : 3];
  if (!regs) {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return cudaGetLastError();
    regs = fa.numRegs > 0 ? fa.numRegs : 1;
  }
  const int per_cta_regs = ((regs + 7) / 8) * 8 * 32 * wpb;
  const int ctas = (a.batch + wpb - 1) / wpb;
  const int want = std::max(1, std::min(65536 / per_cta_regs, (ctas + sm_count - 1) / sm_count));
  const size_t need = static_cast<size_t>(want) * (smem + 1024);
  const int pct = static_cast<int>((need * 100 + 228 * 1024 - 1) / (228 * 1024));
  int occ = 0;
  cudaError_t e = prepare_launch(reinterpret_cast<const void*>(kern), 32 * wpb, smem,
                                 pct > 100 ? 100 : pct, &occ);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  if (warps_per_sm > 0 && warps_per_sm / wpb < occ) occ = warps_per_sm / wpb > 0 ? warps_per_sm / wpb : 1;
  int grid = sm_count * occ;
  if (grid > ctas) grid = ctas;
  if (grid_out) *grid_out = grid;
  kern<<<grid, 32 * wpb, smem, st>>>(a);
  return cudaGetLastError();
}

int warp_pitch(int n) {
  const int cpl = n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8;
  return 32 * cpl;
}

cudaError_t launch_warp_batch(const WarpArgs& a, int sm_count, int warps_per_sm, cudaStream_t st,
                              int* grid_out) {
  if (a.n < 1 || a.n > 256 || a.pitch != warp_pitch(a.n)) return cudaErrorInvalidValue;
  constexpr int wpb = 4;
  switch (a.pitch / 32) {
    case 1: return launch_t<1>(a, sm_count, wpb, warps_per_sm, st, grid_out);
    case 2: return launch_t<2>(a, sm_count, wpb, warps_per_sm, st, grid_out);
    case 4: return launch_t<4>(a, sm_count, wpb, warps_per_sm, st, grid_out);
    default: return launch_t<8>(a, sm_count, wpb, warps_per_sm, st, grid_out);
  }
}

}  // namespace kmb
