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
// Cost source (template SMEM_C):
//   true  — the instance's matrix is staged into shared memory with one TMA
//           bulk copy (cp.async.bulk + mbarrier) and re-read from SMEM;
//   false — rows stream from global memory (L1/L2) with 128-bit loads, which
//           leaves shared memory to per-instance state only, so far more
//           instances are resident per SM.
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

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Build-time switches (A/B measured on config 3, tools/ab_lib.py):
//   KMB_WARP_PREFETCH     TMA L2 prefetch of multi-batch relaxes: 1.17 -> 1.33 ms, off
//   KMB_WARP_CLAMP        short relaxes as one clamped batch: 1.142 -> 1.132 ms, on
//   KMB_WARP_STAGE_CLOCKS per-stage clock64 accounting (kmb_last_instance_stats
//                         columns 5-8): costs 2.7%, off unless diagnosing
#ifndef KMB_WARP_PREFETCH
#define KMB_WARP_PREFETCH 0
#endif
#ifndef KMB_WARP_CLAMP
#define KMB_WARP_CLAMP 1
#endif
#ifndef KMB_WARP_RB_FAT  // rows per relax batch in the low-occupancy instance
#define KMB_WARP_RB_FAT 8  // (2048 / 1536 batches: 72-reg build 0.671 / 0.600 ms; RB 5: .664 /
#endif                     // .598, 8: .639 / .571, 12: .637 / .568; + single-row preload .674 / .610)
#ifndef KMB_WARP_CACHE_ALL  // the register cache in the 72-register build too (A/B: spills, c3 0.997 -> 1.166 ms)
#define KMB_WARP_CACHE_ALL 0
#endif
#ifndef KMB_WARP_FAT_CACHE  // matched rows / u in registers in the low-occupancy build
// (A/B: 2048 0.639 -> 0.625 ms, 1536 0.571 -> 0.559)
#define KMB_WARP_FAT_CACHE 1
#endif
#ifndef KMB_WARP_FAT  // low-occupancy instance for batches of <= 16 warps per SM (A/B)
#define KMB_WARP_FAT 1
#endif
#ifndef KMB_WARP_RB4  // rows per relax batch for <= 4 columns per lane
#define KMB_WARP_RB4 5  // A/B on c3 (tools/ab_lib.py): 4: 1.09, 5: 1.065, 6-8: 1.12, 12: 1.19 ms
#endif
#ifndef KMB_WARP_STAGE_CLOCKS
#define KMB_WARP_STAGE_CLOCKS 0
#endif

// TMA bulk prefetch of `bytes` (multiple of 16) at a 16-byte aligned address into L2
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

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
template <int CPL, bool SMEM_C>
__device__ __forceinline__ RowVec<CPL> load_row(const int32_t* p) {
  RowVec<CPL> r;
  if constexpr (CPL >= 4) {
#pragma unroll
    for (int h = 0; h < CPL / 4; ++h) {
      const int4* q = reinterpret_cast<const int4*>(p) + h;
      const int4 t = SMEM_C ? *q : __ldg(q);
      r.x[4 * h + 0] = t.x; r.x[4 * h + 1] = t.y; r.x[4 * h + 2] = t.z; r.x[4 * h + 3] = t.w;
    }
  } else if constexpr (CPL == 2) {
    const int2* q = reinterpret_cast<const int2*>(p);
    const int2 t = SMEM_C ? *q : __ldg(q);
    r.x[0] = t.x; r.x[1] = t.y;
  } else {
    r.x[0] = SMEM_C ? *p : __ldg(p);
  }
  return r;
}

}  // namespace

// Per-warp shared state (n <= 256), in 32-bit words: two row lists of (row,
// tag) pairs (4n; the free columns found in an epoch live in the idle list) +
// u, w, root_row, match_row, match_col, tree_par, claim (7n) + the U16 row
// minima (n, U16 mode only).  Kept small: what the CTAs per SM do not take of
// the unified cache is L1 for the streamed matrices.
__host__ __device__ constexpr int warp_state_words(int n, bool u16) { return (u16 ? 12 : 11) * n; }

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
  __device__ static int32_t row(K k) { return static_cast<int32_t>(static_cast<uint32_t>(k)); }
  __device__ static K kmin(K a, K b) { return a < b ? a : b; }
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
  __device__ static int32_t row(K k) { return static_cast<int32_t>(k & 0xffu); }
  __device__ static K kmin(K a, K b) { return min(a, b); }
};

struct WarpSmem {
  int32_t *u, *w, *root_row, *match_row, *match_col, *tree_par;
  int32_t* rmin;  // U16 mode: row minimum | (wide row << 31)
  int32_t* ctr;  // [0] rows tail, [1] free columns found this epoch
  uint32_t* claim;
  int2 *rows, *spare;  // (row, tag)
};

// One instance, whole warp.  Returns the status (0 ok, -2 internal).
// U16 rows: 4 or 8 offsets from the row minimum (warp-width pitch, 8/16 B per
// lane), returned already shifted into key position (d << 8) — one PRMT each.
template <int CPL>
__device__ __forceinline__ RowVec<CPL> load_row16(const uint16_t* p) {
  RowVec<CPL> r;
  if constexpr (CPL == 8) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t wv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      r.x[2 * h] = static_cast<int32_t>(__byte_perm(wv[h], 0u, 0x4104));
      r.x[2 * h + 1] = static_cast<int32_t>(__byte_perm(wv[h], 0u, 0x4324));
    }
  } else {
    static_assert(CPL == 4, "U16 rows need 4 or 8 columns per lane");
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    r.x[0] = static_cast<int32_t>(__byte_perm(t.x, 0u, 0x4104));
    r.x[1] = static_cast<int32_t>(__byte_perm(t.x, 0u, 0x4324));
    r.x[2] = static_cast<int32_t>(__byte_perm(t.y, 0u, 0x4104));
    r.x[3] = static_cast<int32_t>(__byte_perm(t.y, 0u, 0x4324));
  }
  return r;
}

// U16 mode (narrow keys only): a row's tag folds its minimum in,
// key = (d << 8) + (tag + (rowmin << 8)) with d = C - rowmin; rows holding an
// offset >= 65535 ("wide") carry bit 31 and are relaxed from the int32 matrix.
template <bool NARROW, bool U16>
__device__ __forceinline__ uint32_t row_tag(int32_t w, int32_t row, const int32_t* rmin) {
  const uint32_t t = Keys<NARROW>::tag(w, row);
  if constexpr (U16) {
    const int32_t rm = rmin[row];
    return rm < 0 ? (t | 0x80000000u) : t + (static_cast<uint32_t>(rm) << 8);
  } else {
    return t;
  }
}

template <int CPL, bool SMEM_C, bool NARROW, bool U16 = false, int RB4 = KMB_WARP_RB4,
          bool CACHE = false>
__device__ __forceinline__ int solve_instance(const WarpArgs& a, const int32_t* Cm, int inst,
                                              const WarpSmem& S, int lane) {
  using KO = Keys<NARROW>;
  using K = typename KO::K;
  constexpr uint32_t FULL = 0xffffffffu;
  const int n = a.n;
  const uint32_t np = static_cast<uint32_t>(a.pitch);
  const int c0 = CPL * lane;
  const int32_t* const lb = Cm + c0;  // this lane's columns of row 0
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

  const uint16_t* const lb16 = U16 ? a.C16 + static_cast<int64_t>(inst) * n * np + c0 : nullptr;
  for (int k = lane; k < n; k += 32)
    rows[k] = make_int2(k, static_cast<int32_t>(row_tag<NARROW, U16>(w[k], k, S.rmin)));
  if (lane == 0) {
    S.ctr[0] = n;
    S.ctr[1] = 0;
  }
  K key[CPL];
  int32_t v[CPL], dc[CPL];
  uint32_t pad = 0;
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    v[q] = 0;
    dc[q] = 0;
    key[q] = KO::INF;
    if (c0 + q >= n) pad |= 1u << q;
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
  int nrows = n, head = 0, nfree = n;  // rows[0, nrows) reached; [head, nrows) to relax
  int32_t D = 0;
  int epochs = 0, dual_steps = 0, rows_scanned = 0, rounds = 0;
  int status = 0;
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
    ++rounds;
    // ---- relax rows[head, nrows)  (hungarian.cpp:164-172) ----
    int r = head;
    // RB rows in flight: entries, then all row loads, then the folds
    constexpr int RB = CPL <= 4 ? RB4 : 4;
    if constexpr (U16) {
      // offsets arrive pre-shifted: key = min(key, (d << 8) + tag'); the last
      // short batch repeats its last row (idempotent) instead of a serial tail
      auto fold16 = [&](int2 e, const RowVec<CPL>& cv) {
        if (e.y < 0) {  // wide row (rare, warp-uniform): exact int32 values
          const RowVec<CPL> c32 = load_row<CPL, false>(lb + static_cast<uint32_t>(e.x) * np);
          const uint32_t t = static_cast<uint32_t>(e.y) & 0x7fffffffu;
#pragma unroll
          for (int q = 0; q < CPL; ++q) key[q] = KO::kmin(key[q], KO::make(c32.x[q], t, e.x));
        } else {
#pragma unroll
          for (int q = 0; q < CPL; ++q)
            key[q] = KO::kmin(key[q], static_cast<uint32_t>(cv.x[q]) + static_cast<uint32_t>(e.y));
        }
      };
      for (; r + RB - 1 < nrows; r += RB) {
        int2 e[RB];
        RowVec<CPL> cv[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) e[k] = rows[r + k];
#pragma unroll
        for (int k = 0; k < RB; ++k) cv[k] = load_row16<CPL>(lb16 + static_cast<uint32_t>(e[k].x) * np);
        int any_wide = 0;
#pragma unroll
        for (int k = 0; k < RB; ++k) any_wide |= e[k].y;
        if (any_wide >= 0) {  // common case: no wide row in the batch, branch-free folds
#pragma unroll
          for (int k = 0; k < RB; ++k)
#pragma unroll
            for (int q = 0; q < CPL; ++q)
              key[q] = KO::kmin(key[q], static_cast<uint32_t>(cv[k].x[q]) + static_cast<uint32_t>(e[k].y));
        } else {
#pragma unroll
          for (int k = 0; k < RB; ++k) fold16(e[k], cv[k]);
        }
      }
      if (r < nrows) {
        int2 e[4];
        RowVec<CPL> cv[4];
        for (; r < nrows; r += 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) e[k] = rows[min(r + k, nrows - 1)];
#pragma unroll
          for (int k = 0; k < 4; ++k) cv[k] = load_row16<CPL>(lb16 + static_cast<uint32_t>(e[k].x) * np);
          if ((e[0].y | e[1].y | e[2].y | e[3].y) >= 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int q = 0; q < CPL; ++q)
                key[q] = KO::kmin(key[q], static_cast<uint32_t>(cv[k].x[q]) + static_cast<uint32_t>(e[k].y));
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) fold16(e[k], cv[k]);
          }
        }
        r = nrows;
      }
    }
    if (KMB_WARP_PREFETCH && !SMEM_C && !U16 && nrows - r > RB) {
      // more than one batch pending (first round, epoch starts): one lane per
      // row asks TMA to pull the rows into L2 so later batches hit there
      for (int k = r + RB + lane; k < nrows; k += 32)
        bulk_prefetch_l2(Cm + static_cast<uint32_t>(rows[k].x) * np, np * 4);
    }
    for (; r + RB - 1 < nrows; r += RB) {
      int2 e[RB];
      RowVec<CPL> cv[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) e[k] = rows[r + k];
#pragma unroll
      for (int k = 0; k < RB; ++k)
        cv[k] = load_row<CPL, SMEM_C>(lb + static_cast<uint32_t>(e[k].x) * np);
#pragma unroll
      for (int k = 0; k < RB; ++k)
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          key[q] = KO::kmin(key[q], KO::make(cv[k].x[q], static_cast<uint32_t>(e[k].y), e[k].x));
    }
    if (!KMB_WARP_CLAMP) {
      for (; r < nrows; ++r) {
        const int2 e = rows[r];
        const RowVec<CPL> cv = load_row<CPL, SMEM_C>(lb + static_cast<uint32_t>(e.x) * np);
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          key[q] = KO::kmin(key[q], KO::make(cv.x[q], static_cast<uint32_t>(e.y), e.x));
      }
    } else if (nrows - r == 1) {
      const int2 e = rows[r];
      const RowVec<CPL> cv = load_row<CPL, SMEM_C>(lb + static_cast<uint32_t>(e.x) * np);
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        key[q] = KO::kmin(key[q], KO::make(cv.x[q], static_cast<uint32_t>(e.y), e.x));
    } else if (r < nrows) {
      // 2..RB-1 rows: one batch with the last row repeated (the fold is
      // idempotent), so all loads are in flight together
      int2 e[RB];
      RowVec<CPL> cv[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) e[k] = rows[min(r + k, nrows - 1)];
#pragma unroll
      for (int k = 0; k < RB; ++k)
        cv[k] = load_row<CPL, SMEM_C>(lb + static_cast<uint32_t>(e[k].x) * np);
#pragma unroll
      for (int k = 0; k < RB; ++k)
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          key[q] = KO::kmin(key[q], KO::make(cv[k].x[q], static_cast<uint32_t>(e[k].y), e[k].x));
    }
    r = nrows;
    rows_scanned += nrows - head;
    head = nrows;
    KMB_WSTAGE(0);
    if (epochs == 0 && rounds == 1 && a.seed == 1) {  // column reduction, :328-333
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (!((pad >> q) & 1)) v[q] = KO::val(key[q]);
    }
    // ---- min unreached slack' (hungarian.cpp:203-206) ----
    int32_t s[CPL];
    int32_t lm = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      s[q] = KO::val(key[q]) - v[q];
      if (!((rch >> q) & 1)) lm = min(lm, s[q]);
    }
    const int32_t m = __reduce_min_sync(FULL, lm);
    if (m > D) {
      if (m == 0x7fffffff) {
        status = -2;
        break;
      }
      D = m;  // dual step (hungarian.cpp:207-215), applied lazily
      ++dual_steps;
    }
    KMB_WSTAGE(1);
    // ---- absorb zero-slack columns (hungarian.cpp:186-199) ----
    // Usually one column per round turns tight: only its lane branches in, and
    // appends go through warp-private shared counters (no per-column ballots).
    uint32_t tm = 0;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (!((rch >> q) & 1) && s[q] == D) tm |= 1u << q;
    if (tm) {
      rch |= tm;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        if (!((tm >> q) & 1)) continue;
        const int col = c0 + q;
        dc[q] = D;
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
          rows[atomicAdd(S.ctr, 1)] =
              make_int2(i2, static_cast<int32_t>(row_tag<NARROW, U16>(w2, i2, S.rmin)));
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
          v[q] -= D - dc[q];
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
        if (wclaimed_in(claim[root_row[e.x]], epochs)) u[e.x] = w[e.x] + D;
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
    if (mr >= 0) tot += SMEM_C ? Cm[k * np + mr] : __ldg(Cm + k * np + mr);
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q)
    if (c0 + q < n) a.v[static_cast<int64_t>(inst) * n + c0 + q] = v[q];
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
// batches) for batches that need at most 16 warps per SM
template <int CPL, bool SMEM_C, int MINB = 7>
__global__ void __launch_bounds__(128, MINB) k_warp_batch(WarpArgs a) {
  constexpr int RBK = MINB >= 7 ? KMB_WARP_RB4 : KMB_WARP_RB_FAT;
  constexpr bool CK = (MINB < 7 || KMB_WARP_CACHE_ALL) && KMB_WARP_FAT_CACHE;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;  // warp in block
  const int wpb = blockDim.x >> 5;
  const int n = a.n, np = a.pitch;
  constexpr uint32_t FULL = 0xffffffffu;

  // carve this warp's slice: [mbarrier | C (SMEM_C) | state]
  const size_t cbytes = SMEM_C ? static_cast<size_t>(n) * np * 4 : 0;
  constexpr bool kU16able = !SMEM_C && (CPL == 4 || CPL == 8);
  const bool use16 = kU16able && a.C16 != nullptr;
  const size_t wbytes = cbytes + static_cast<size_t>(warp_state_words(n, use16)) * 4 + 16;
  unsigned char* base = dyn + wib * ((wbytes + 15) & ~static_cast<size_t>(15));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base);
  int32_t* ctr = reinterpret_cast<int32_t*>(base + 8);  // 2 counters after the mbarrier
  int32_t* Cs = reinterpret_cast<int32_t*>(base + 16);
  int32_t* st = reinterpret_cast<int32_t*>(base + 16 + cbytes);
  WarpSmem S;
  S.rows = reinterpret_cast<int2*>(st);  // 8-byte aligned first
  S.spare = S.rows + n;
  S.u = reinterpret_cast<int32_t*>(S.spare + n);
  S.w = S.u + n;
  S.root_row = S.w + n;
  S.match_row = S.root_row + n;
  S.match_col = S.match_row + n;
  S.tree_par = S.match_col + n;
  S.claim = reinterpret_cast<uint32_t*>(S.tree_par + n);
  S.rmin = use16 ? reinterpret_cast<int32_t*>(S.claim + n) : nullptr;
  S.ctr = ctr;

  if (SMEM_C && lane == 0) mbar_init1(bar);
  __syncwarp();
  uint32_t parity = 0;
  const int c0 = CPL * lane;

  for (int inst = blockIdx.x * wpb + wib; inst < a.batch; inst += gridDim.x * wpb) {
    const unsigned long long t_inst0 = globaltimer_ns();
    const int32_t* Cg = a.C + static_cast<int64_t>(inst) * n * np;
    const int32_t* Cm = Cg;
    if constexpr (SMEM_C) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t total = static_cast<uint32_t>(n) * np * 4;
        mbar_expect(bar, total);
        for (uint32_t off = 0; off < total; off += 32768u) {
          const uint32_t b = total - off < 32768u ? total - off : 32768u;
          tma_bulk_g2s(reinterpret_cast<unsigned char*>(Cs) + off,
                       reinterpret_cast<const unsigned char*>(Cg) + off, b, bar);
        }
      }
      Cm = Cs;
    }
    for (int k = lane; k < n; k += 32) {
      S.match_row[k] = -1;
      S.match_col[k] = -1;
      S.claim[k] = 0xFFFFFFFFu;
      S.root_row[k] = k;
    }
    if constexpr (SMEM_C) {
      mbar_wait_parity(bar, parity);
      parity ^= 1;
    }
    __syncwarp();
    // validation (core.cpp:144-145 + device range) and row reductions
    // (hungarian.cpp:323-327): the warp walks the rows, lanes across columns —
    // or, in U16 mode, reads what the packing pass (k_pack16) computed
    int32_t lo_all = 0x7fffffff, hi_all = 0;
    if (use16) {
      for (int k = lane; k < n; k += 32) {
        const int32_t rm = __ldg(a.rmin + static_cast<int64_t>(inst) * n + k);
        S.rmin[k] = rm;
        const int32_t u0 = a.seed == 1 ? (rm & 0x7fffffff) : 0;
        S.u[k] = u0;
        S.w[k] = u0;
      }
      lo_all = __ldg(a.imin + inst);
      hi_all = __ldg(a.imax + inst);
    } else {
    // 8 rows in flight: loads first, then the per-row reductions
    for (int i0 = 0; i0 < n; i0 += 8) {
      RowVec<CPL> cv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        cv[k] = load_row<CPL, SMEM_C>(Cm + static_cast<int64_t>(min(i0 + k, n - 1)) * np + c0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
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
        if (lane == (i & 31)) {
          const int32_t u0 = a.seed == 1 ? lo : 0;
          S.u[i] = u0;
          S.w[i] = u0;
        }
      }
    }
    hi_all = __reduce_max_sync(FULL, hi_all);
    }
    int status = lo_all < 0 ? 2 : (hi_all >= (1 << 29) ? 3 : 0);
    __syncwarp();
    if (status == 0) {
      if constexpr (kU16able) {
        if (use16 && hi_all < (1 << 21))
          status = solve_instance<CPL, false, true, true>(a, Cm, inst, S, lane);
        else if (hi_all < (1 << 21))
          status = solve_instance<CPL, SMEM_C, true, false, RBK, CK>(a, Cm, inst, S, lane);
        else
          status = solve_instance<CPL, SMEM_C, false, false, RBK, CK>(a, Cm, inst, S, lane);
      } else {
        status = hi_all < (1 << 21) ? solve_instance<CPL, SMEM_C, true, false, RBK, CK>(a, Cm, inst, S, lane)
                                    : solve_instance<CPL, SMEM_C, false, false, RBK, CK>(a, Cm, inst, S, lane);
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

// U16 packing pass: per row, the minimum and the offsets d = C - min saturated
// at 65535 (16 bits, same warp-width pitch); a row with a saturated offset is
// flagged "wide" (bit 31 of its minimum) and relaxed from the int32 matrix.
// Also the per-instance min/max used for validation.  One warp per row.
template <int CPL>
__global__ void __launch_bounds__(256) k_pack16(WarpArgs a, uint16_t* C16, int32_t* rmin,
                                                int32_t* imin, int32_t* imax) {
  const int lane = threadIdx.x & 31;
  const int64_t nrows_all = static_cast<int64_t>(a.batch) * a.n;
  const int c0 = CPL * lane;
  for (int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < nrows_all;
       g += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const RowVec<CPL> cv = load_row<CPL, false>(a.C + g * a.pitch + c0);
    int32_t lo = 0x7fffffff, hi = 0;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (c0 + q < a.n) {
        lo = min(lo, cv.x[q]);
        hi = max(hi, cv.x[q]);
      }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    uint32_t d[CPL];
    bool wide = false;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int64_t x = static_cast<int64_t>(cv.x[q]) - lo;
      d[q] = x >= 65535 || x < 0 ? 65535u : static_cast<uint32_t>(x);
      wide |= (c0 + q < a.n) && x >= 65535;
    }
    wide = __any_sync(0xffffffffu, wide);
    uint16_t* out = C16 + g * a.pitch + c0;
    if constexpr (CPL == 8) {
      *reinterpret_cast<uint4*>(out) = make_uint4(d[0] | (d[1] << 16), d[2] | (d[3] << 16),
                                                  d[4] | (d[5] << 16), d[6] | (d[7] << 16));
    } else {
      *reinterpret_cast<uint2*>(out) = make_uint2(d[0] | (d[1] << 16), d[2] | (d[3] << 16));
    }
    if (lane == 0) {
      rmin[g] = wide ? (lo | static_cast<int32_t>(0x80000000u)) : lo;
      const int inst = static_cast<int>(g / a.n);
      atomicMin(imin + inst, lo);
      atomicMax(imax + inst, hi);
    }
  }
}

cudaError_t launch_pack16(const WarpArgs& a, int sm_count, uint16_t* C16, int32_t* rmin,
                          int32_t* imin, int32_t* imax, cudaStream_t st) {
  const int cpl = a.pitch / 32;
  if (cpl != 4 && cpl != 8) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(imin, 0x7f, static_cast<size_t>(a.batch) * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(imax, 0, static_cast<size_t>(a.batch) * 4, st);
  if (e != cudaSuccess) return e;
  const int blocks = sm_count * 8;
  if (cpl == 4) k_pack16<4><<<blocks, 256, 0, st>>>(a, C16, rmin, imin, imax);
  else k_pack16<8><<<blocks, 256, 0, st>>>(a, C16, rmin, imin, imax);
  return cudaGetLastError();
}

int warp_max_n() { return 256; }

size_t warp_smem_per_warp(int n, int pitch, bool smem_c, bool u16) {
  const size_t c = smem_c ? static_cast<size_t>(n) * pitch * 4 : 0;
  return (c + static_cast<size_t>(warp_state_words(n, u16)) * 4 + 16 + 15) & ~static_cast<size_t>(15);
}

template <int CPL, bool SMEM_C, int MINB = 7>
static cudaError_t launch_t(const WarpArgs& a, int sm_count, int wpb, int warps_per_sm,
                            cudaStream_t st, int* grid_out) {
  if constexpr (KMB_WARP_FAT && MINB == 7 && CPL == 4 && !SMEM_C) {
    // a batch that needs at most 4 CTAs (16 warps) per SM runs the 128-register
    // instance (config-3 shards of <= 2,368 instances)
    if (a.C16 == nullptr && warps_per_sm == 0 &&
        (a.batch + wpb - 1) / wpb <= 4 * sm_count)
      return launch_t<CPL, SMEM_C, 4>(a, sm_count, wpb, warps_per_sm, st, grid_out);
  }
  auto kern = k_warp_batch<CPL, SMEM_C, MINB>;
  const size_t smem = warp_smem_per_warp(a.n, a.pitch, SMEM_C, a.C16 != nullptr) * wpb;
  // Shared-memory carveout: just the state of the CTAs per SM this launch
  // needs (all instances resident in one wave, at most the register limit),
  // +1 KiB reserved per CTA; the rest of the unified cache is L1, which keeps
  // part of each streamed matrix close (config 3: 1.064 -> 1.004 ms with a
  // 196 KB carveout instead of the maximum; the longest instance alone 0.61 ->
  // 0.48 ms)
  int occ = 0;
  static int regs_cached[2][4] = {};  // per instantiation; benign race: every thread computes the same value
  int& regs = regs_cached[SMEM_C ? 1 : 0][CPL == 1 ? 0 : CPL == 2 ? 1 : CPL == 4 ? 2 : 3];
  if (!regs) {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return cudaGetLastError();
    regs = fa.numRegs > 0 ? fa.numRegs : 1;
  }
  int carve = cudaSharedmemCarveoutMaxShared;
  if (!SMEM_C) {
    const int per_cta_regs = ((regs + 7) / 8) * 8 * 32 * wpb;
    int want = 65536 / per_cta_regs;
    const int ctas = (a.batch + wpb - 1) / wpb;
    want = std::max(1, std::min(want, (ctas + sm_count - 1) / sm_count));
    const size_t need = static_cast<size_t>(want) * (smem + 1024);
    const int pct = static_cast<int>((need * 100 + 228 * 1024 - 1) / (228 * 1024));
    carve = pct > 100 ? 100 : pct;
  }
  cudaError_t e = prepare_launch(reinterpret_cast<const void*>(kern), 32 * wpb, smem, carve, &occ);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  static const bool debug_occ = getenv("KMB_DEBUG_OCC") != nullptr;
  if (debug_occ) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr, "k_warp_batch<%d,%d>: %d CTAs/SM x %d warps, dyn smem %zu B, regs %d, static smem %zu, local %zu, maxthr %d\n",
            CPL, SMEM_C ? 1 : 0, occ, wpb, smem, fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes, fa.maxThreadsPerBlock);
  }
  const int warps_needed = a.batch;
  if (warps_per_sm > 0 && warps_per_sm / wpb < occ) occ = warps_per_sm / wpb > 0 ? warps_per_sm / wpb : 1;
  int grid = sm_count * occ;
  const int grid_needed = (warps_needed + wpb - 1) / wpb;
  if (grid > grid_needed) grid = grid_needed;
  if (grid_out) *grid_out = grid;
  kern<<<grid, 32 * wpb, smem, st>>>(a);
  return cudaGetLastError();
}

int warp_pitch(int n) {
  const int cpl = n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8;
  return 32 * cpl;
}

cudaError_t launch_warp_batch(const WarpArgs& a, int sm_count, bool smem_c, int warps_per_sm,
                              cudaStream_t st, int* grid_out) {
  if (a.n < 1 || a.n > 256 || a.pitch != warp_pitch(a.n)) return cudaErrorInvalidValue;
  const int cpl = a.pitch / 32;
  if (smem_c && warp_smem_per_warp(a.n, a.pitch, true, false) > 227 * 1024) smem_c = false;
  const int wpb = smem_c ? 1 : 4;
#define KMB_L(C)                                                                          \
  return smem_c ? launch_t<C, true>(a, sm_count, wpb, warps_per_sm, st, grid_out)         \
                : launch_t<C, false>(a, sm_count, wpb, warps_per_sm, st, grid_out)
  switch (cpl) {
    case 1: KMB_L(1);
    case 2: KMB_L(2);
    case 4: KMB_L(4);
    default: KMB_L(8);
  }
#undef KMB_L
}

}  // namespace kmb
