// Single-instance exact KM / batched-KM engine for sm_100a: one persistent
// kernel, G column-slab CTAs, software grid barriers, all state on device.
//
// Reference path replaced: ot::solve_batched_km (hungarian.cpp:313-381) and,
// with seed 0, ot::solve_km (hungarian.cpp:55-136).  The engine keeps the three
// rules that make the reference's final duals canonical:
// same starting duals; a dual step only when the tight closure of the free rows
// holds no free column; the step over the full closure with delta = min slack.
// How it gets there differs from the reference:
//
//  * Lazy duals.  D is the dual shift accumulated by the search; row i reached
//    at shift Dr stores w_i = u_i - Dr, so a column's slack' = min_i (C_ij - w_i)
//    - v_j never changes under a dual step and column j is tight iff slack' == D.
//    A dual step is therefore D = min unreached slack' — no O(n) update — and
//    the duals are written back when a tree dissolves (u_i = w_i + D, v_j -= D - Dc_j).
//  * Relax = reduced-cost scan (hungarian.cpp:164-172).  CTA b owns columns
//    [b*W, b*W+W) of every row; each round it streams the W-wide slab of every
//    newly reached row with 128-bit no-allocate loads and folds them into
//    per-column packed (value, row) keys (kmb_common.cuh): min and argmin
//    parent in one unsigned min, reduced by warp shuffles then shared atomics.
//  * Min-slack (hungarian.cpp:203-206): block reduce -> one partial per CTA ->
//    every CTA reads all partials after the grid barrier (no second pass).
//  * Absorb (hungarian.cpp:186-199): zero-slack unreached columns of the slab
//    are reached; their matched rows are appended (warp-aggregated atomics) to
//    the phase's row list; free columns are recorded and claim their tree root.
//  * Augment: instead of the reference's per-phase full tight-graph rebuild
//    (TightPhase, hungarian.cpp:233-252, 55-80% of its CPU time) the search's
//    own argmin parents form an alternating forest of tight edges rooted at the
//    free rows; every tree that reached a free column flips the path of its
//    smallest such column.  Paths of distinct trees are vertex-disjoint.
//
// One round = relax + local absorb at D | barrier (+ dual step, absorb, barrier
// when nothing anywhere became tight).  An epoch ends after the round that
// absorbs a free column: claimed trees are dissolved and augmented, survivors
// stay reached (incremental epochs).  The barrier is a template:
// GridBarrier (software, any G <= #SMs, cooperative launch) or ClusterBarrier
// (one thread-block cluster of G <= 16 CTAs, hardware barrier.cluster).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "kmb_common.cuh"
#include "kmb_internal.h"

#ifndef KMB_SOLVER_FINE
#define KMB_SOLVER_FINE 0
#endif
#ifndef KMB_POLL_RELAXED  // grid barrier: relaxed polls + one acquire (1) or acquire polls (0)
#define KMB_POLL_RELAXED 0
#endif
#ifndef KMB_SOLVER_PREFETCH  // L2 bulk prefetch of rows appended by the absorb
#define KMB_SOLVER_PREFETCH 1
#endif
#if KMB_SOLVER_FINE
#include <cstdio>
#endif

namespace kmb {

// list_w entry: the dual shift D at which the row was reached (low 32 bits;
// 0 <= D <= max cost < 2^29) and the row's tree root (high 32 bits), so every
// CTA's relax learns the roots of the rows it scans from a word it loads anyway
// and keeps them in shared memory: the absorb then finds a parent's root
// without an L2 round trip (grid engine)
__device__ __forceinline__ int64_t lw_pack(int64_t D, int32_t root) {
  return static_cast<int64_t>((static_cast<uint64_t>(static_cast<uint32_t>(root)) << 32) |
                              static_cast<uint32_t>(D));
}
__device__ __forceinline__ int64_t lw_d(int64_t x) { return static_cast<int64_t>(static_cast<uint32_t>(x)); }
__device__ __forceinline__ int32_t lw_root(int64_t x) {
  return static_cast<int32_t>(static_cast<uint64_t>(x) >> 32);
}

constexpr int kThreads = 512;
#ifndef KMB_SOLVER_RB
#define KMB_SOLVER_RB 6  // A/B: 4: c5 111.5 c4 143.4 c2 23.9; 6: 109.6 142.2 24.2; 8: 109.0 149.4 25.1 ms
#endif
constexpr int kSolveBatch = KMB_SOLVER_RB;  // rows in flight per thread in the solve's relax
constexpr int kRelaxBatch = kSolveBatch;
#ifndef KMB_SCAN_RB
#define KMB_SCAN_RB 16  // A/B c5 full pass: 8: 5.53, 12: 6.08, 16: 6.12 TB/s
#endif
constexpr int kScanBatch = KMB_SCAN_RB;    // ... in the full-frontier scan (bandwidth-bound)

struct SlabSmem {
  int64_t part[kThreads / 32];
  int64_t m;
  int32_t append_base;
  int32_t ndseg;              // dirty segments after an epoch end
  int32_t abort;              // sharded ranks on GPUs: a barrier timed out
  int32_t my_rows, my_frees;  // this CTA's appends since the last barrier
  int32_t tot_rows, tot_frees;  // everyone's, delivered by the counting barrier
};

// ---- where the per-row / per-column search state lives -----------------------
// GMem: global memory (grid engine, any G).  DMem: the distributed shared memory
// of the one thread-block cluster (cluster engine, G a power of two): element i
// of every array lives in CTA (i mod G) at local index i / G, the append
// counters in CTA 0 and each CTA's min-slack partial in its own shared memory,
// so every dependent hop of a round is a DSMEM access instead of an L2 round
// trip.  The barriers order both (bar.sync + gpu-scope release/acquire, or
// barrier.cluster release/acquire).
struct GMem {
  const SolverArgs* a;
  __device__ int32_t* list_row(int p, int i) const { return a->list_row[p] + i; }
  __device__ int64_t* list_w(int p, int i) const { return a->list_w[p] + i; }
  __device__ int64_t* u(int i) const { return a->u + i; }
  __device__ int32_t* root_row(int i) const { return a->root_row + i; }
  __device__ int32_t* match_row(int i) const { return a->match_row + i; }
  __device__ int32_t* match_col(int i) const { return a->match_col + i; }
  __device__ int32_t* tree_par(int i) const { return a->tree_par + i; }
  __device__ uint64_t* claim(int i) const { return a->claim + i; }
  __device__ int32_t* found(int i) const { return a->found + i; }
  __device__ int* rcnt(int k) const { return &a->ctrl->rcnt[k]; }
  __device__ int* fcnt(int k) const { return &a->ctrl->fcnt[k]; }
  __device__ int64_t* partial(int b) const { return a->partial + b; }
  template <class T>
  __device__ static T ld(const T* p) { return ldcg(p); }
  // tree claims: 64-bit (epoch stamp, column) keys, smaller wins
  __device__ static uint64_t ckey(int ep, int col) { return claim_key(ep, col); }
  __device__ static bool claimed(uint64_t c, int ep) { return claimed_in(c, ep); }
  __device__ void claim_min(int root, uint64_t k) const {
    atomicMin(reinterpret_cast<unsigned long long*>(a->claim + root), static_cast<unsigned long long>(k));
  }
};

struct DMem {
  int64_t *lw[2], *u_;
  uint32_t* claim_;  // 32-bit claims: 64-bit atomicMin has no native DSMEM form
  int32_t *lrow[2], *root_, *mrow_, *mcol_, *tpar_, *found_;
  int* cnt;       // [0, 3) row appends, [3, 6) free-column appends: CTA 0's are live
  int64_t* part;  // this CTA's min-slack partial
  int shift, mask;
  template <class T>
  __device__ T* at(T* base, int i) const {
    return cooperative_groups::this_cluster().map_shared_rank(base + (i >> shift),
                                                              static_cast<unsigned>(i & mask));
  }
  __device__ int32_t* list_row(int p, int i) const { return at(lrow[p], i); }
  __device__ int64_t* list_w(int p, int i) const { return at(lw[p], i); }
  __device__ int64_t* u(int i) const { return at(u_, i); }
  __device__ int32_t* root_row(int i) const { return at(root_, i); }
  __device__ int32_t* match_row(int i) const { return at(mrow_, i); }
  __device__ int32_t* match_col(int i) const { return at(mcol_, i); }
  __device__ int32_t* tree_par(int i) const { return at(tpar_, i); }
  __device__ uint32_t* claim(int i) const { return at(claim_, i); }
  __device__ int32_t* found(int i) const { return at(found_, i); }
  // (stamp, column) in 32 bits: n <= 8192 columns (13 bits), stamp 0x7FFFF - (ep + 1)
  // decreasing with the epoch; the all-ones initial value matches no epoch
  __device__ static uint32_t ckey(int ep, int col) {
    return ((0x7FFFFu - static_cast<uint32_t>(ep + 1)) << 13) | static_cast<uint32_t>(col);
  }
  __device__ static bool claimed(uint32_t c, int ep) {
    return (c >> 13) == 0x7FFFFu - static_cast<uint32_t>(ep + 1);
  }
  __device__ void claim_min(int root, uint32_t k) const { atomicMin(claim(root), k); }
  __device__ int* rcnt(int k) const { return cooperative_groups::this_cluster().map_shared_rank(cnt + k, 0u); }
  __device__ int* fcnt(int k) const { return cooperative_groups::this_cluster().map_shared_rank(cnt + 3 + k, 0u); }
  __device__ int64_t* partial(int b) const {
    return cooperative_groups::this_cluster().map_shared_rank(part, static_cast<unsigned>(b));
  }
  template <class T>
  __device__ static T ld(const T* p) { return *reinterpret_cast<const volatile T*>(p); }
};

// RMem: the column-sharded engine's replicated row side (k_solve_sharded,
// DESIGN.md §5).  Rank r's CTAs own a slab of the columns and read rank r's
// replica of the row-side state; every write goes to every replica (P2P
// stores over NVLink when the ranks are GPUs, plain stores when they are CTA
// groups of one launch), so the barrier after it publishes it everywhere.
// Tree claims and the append counters live in the home block (rank 0) and are
// updated with atomics there.  Replica layout (shard_rep_bytes): int64 u[n],
// list_w[2][n], partial[G]; then int32 root_row, match_row, match_col,
// tree_par, list_row[2], found (n each).
template <class T>
struct RRef {
  unsigned char* const* bases;  // the R replica bases (shared memory)
  const unsigned char* mine;
  size_t off;
  int R;
  __device__ const RRef& operator*() const { return *this; }
  __device__ void operator=(T v) const {
    for (int r = 0; r < R; ++r) *reinterpret_cast<T*>(bases[r] + off) = v;
  }
  __device__ T load() const { return ldcg(reinterpret_cast<const T*>(mine + off)); }
  __device__ T* local() const { return reinterpret_cast<T*>(const_cast<unsigned char*>(mine) + off); }
};

__host__ __device__ inline size_t shard_rep_o32(int n, int G) {
  return (8ull * (3ull * n + G) + 15) & ~static_cast<size_t>(15);
}

struct RMem {
  unsigned char* const* bases;
  const unsigned char* mine;
  int R, n;
  size_t o32;
  Ctrl* ctrl;          // home
  uint64_t* claim_h;   // home
  template <class T>
  __device__ RRef<T> ref(size_t off) const { return RRef<T>{bases, mine, off, R}; }
  __device__ RRef<int64_t> u(int i) const { return ref<int64_t>(8ull * i); }
  __device__ RRef<int64_t> list_w(int p, int i) const { return ref<int64_t>(8ull * ((1ull + p) * n + i)); }
  __device__ RRef<int64_t> partial(int b) const { return ref<int64_t>(8ull * (3ull * n + b)); }
  __device__ RRef<int32_t> a32(int k, int i) const { return ref<int32_t>(o32 + 4ull * (static_cast<size_t>(k) * n + i)); }
  __device__ RRef<int32_t> root_row(int i) const { return a32(0, i); }
  __device__ RRef<int32_t> match_row(int i) const { return a32(1, i); }
  __device__ RRef<int32_t> match_col(int i) const { return a32(2, i); }
  __device__ RRef<int32_t> tree_par(int i) const { return a32(3, i); }
  __device__ RRef<int32_t> list_row(int p, int i) const { return a32(4 + p, i); }
  __device__ RRef<int32_t> found(int i) const { return a32(6, i); }
  __device__ uint64_t* claim(int i) const { return claim_h + i; }
  __device__ int* rcnt(int k) const { return &ctrl->rcnt[k]; }
  __device__ int* fcnt(int k) const { return &ctrl->fcnt[k]; }
  template <class T>
  __device__ static T ld(const RRef<T>& r) { return r.load(); }
  template <class T>
  __device__ static T ld(const T* p) { return ldcg(p); }
  __device__ static uint64_t ckey(int ep, int col) { return claim_key(ep, col); }
  __device__ static bool claimed(uint64_t c, int ep) { return claimed_in(c, ep); }
  __device__ void claim_min(int root, uint64_t k) const {
    atomicMin(reinterpret_cast<unsigned long long*>(claim_h + root), static_cast<unsigned long long>(k));
  }
};

// dynamic shared memory of the slab state (keys, v, Dc, reached, dirty segments)
__host__ __device__ inline size_t solver_smem_bytes_dev(int W) {
  return (static_cast<size_t>(W) * (8 + 8 + 8 + 1 + 1) + 16 + 15) & ~static_cast<size_t>(15);
}

// DSMEM bytes per CTA for n over G CTAs (L = ceil(n / G) elements of each array)
__host__ __device__ inline size_t dsm_bytes(int n, int G) {
  const size_t L = (static_cast<size_t>(n) + G - 1) / G;
  return L * (8 * 3 + 4 * 8) + 16 * 16;  // + per-array 16-byte alignment, counters
}

// ---- K1: row reductions + engine state init (hungarian.cpp:323-327) -------
// One warp per row, 128-bit loads; also seeds the phase-0 row list.
__global__ void __launch_bounds__(256) k_init_rows(SolverArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < a.n; i += nwarps) {
    // one pass per row: validation (core.cpp:144-145 + the device range) and,
    // for seed 1, the row minimum
    const int32_t* row = a.C + static_cast<int64_t>(i) * a.pitch;
    int32_t lo = 0x7fffffff, hi = 0;
    const int n4 = a.n >> 2;
    const int4* row4 = reinterpret_cast<const int4*>(row);
    for (int q = lane; q < n4; q += 32) {
      const int4 c = ld_stream(row4 + q);
      lo = min(lo, min(min(c.x, c.y), min(c.z, c.w)));
      hi = max(hi, max(max(c.x, c.y), max(c.z, c.w)));
    }
    for (int j = (n4 << 2) + lane; j < a.n; j += 32) {
      lo = min(lo, row[j]);
      hi = max(hi, row[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int64_t u0 = a.seed == 1 ? lo : 0;
    if (lane == 0) {
      if (lo < 0) atomicMax(&a.ctrl->status, 2);               // KMB_ENEGATIVE
      else if (hi >= (1 << 29)) atomicMax(&a.ctrl->status, 3);  // KMB_ERANGE
      a.u[i] = u0;
      a.list_row[0][i] = i;
      a.list_w[0][i] = static_cast<int64_t>(i) << 32;  // reached at D = 0, its own root
      a.root_row[i] = i;
      a.claim[i] = KMB_KEY_INF;
      a.match_row[i] = -1;
      a.match_col[i] = -1;
    }
  }
  // the rest of Ctrl was zeroed by the host (cudaMemsetAsync) before launch
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->tail[0] = a.n;
}

// ---- K3: reduced-cost scan of rows list[head, tail) over one column slab ----
// Thread (g, s): segment s = 4 consecutive columns, row group g.  When W = 4*S
// is a power of two, lanes sharing a segment differ only in their high lane
// bits (S < 32) and a xor-shuffle tree merges them before the shared atomics.
template <class Mem, int kRelaxBatch = kSolveBatch>
__device__ __forceinline__ void relax_slab(const int32_t* C, int64_t pitch, const Mem& M, int p,
                                           int head, int tail, int c0, int W, uint64_t* skey,
                                           int32_t* sroot = nullptr) {
  const int S = W >> 2;
  const int R = kThreads / S > 0 ? kThreads / S : 1;
  const int tid = threadIdx.x;
  const int Sreal = S < kThreads ? S : kThreads;
  const int lane = tid & 31;
  for (int sbase = 0; sbase < S; sbase += Sreal) {
    const int s = sbase + (tid % Sreal);
    const int g = tid / Sreal;
    uint64_t best0 = KMB_KEY_INF, best1 = KMB_KEY_INF, best2 = KMB_KEY_INF, best3 = KMB_KEY_INF;
    if (g < R) {
      const int32_t* base = C + c0 + 4 * s;
      int r = head + g;
      // kRelaxBatch rows in flight per thread: all list/tag loads, then all
      // 128-bit cost loads, then the folds
      for (; r + (kRelaxBatch - 1) * R < tail; r += kRelaxBatch * R) {
        int i[kRelaxBatch];
        uint32_t b[kRelaxBatch];
        int4 c[kRelaxBatch];
        int64_t dr[kRelaxBatch];
#pragma unroll
        for (int k = 0; k < kRelaxBatch; ++k) {
          i[k] = M.ld(M.list_row(p, r + k * R));
          dr[k] = M.ld(M.list_w(p, r + k * R));
        }
#pragma unroll
        for (int k = 0; k < kRelaxBatch; ++k) {
          c[k] = ld_stream(reinterpret_cast<const int4*>(base + static_cast<int64_t>(i[k]) * pitch));
          b[k] = row_bias(M.ld(M.u(i[k])) - lw_d(dr[k]));  // w = u - D at reach
        }
        if (sroot && s == 0)
#pragma unroll
          for (int k = 0; k < kRelaxBatch; ++k) sroot[i[k]] = lw_root(dr[k]);
#pragma unroll
        for (int k = 0; k < kRelaxBatch; ++k) {
          best0 = umin64(best0, pack_key(static_cast<uint32_t>(c[k].x) + b[k], i[k]));
          best1 = umin64(best1, pack_key(static_cast<uint32_t>(c[k].y) + b[k], i[k]));
          best2 = umin64(best2, pack_key(static_cast<uint32_t>(c[k].z) + b[k], i[k]));
          best3 = umin64(best3, pack_key(static_cast<uint32_t>(c[k].w) + b[k], i[k]));
        }
      }
      for (; r < tail; r += R) {
        const int i = M.ld(M.list_row(p, r));
        const int64_t drr = M.ld(M.list_w(p, r));
        const int4 c = ld_stream(reinterpret_cast<const int4*>(base + static_cast<int64_t>(i) * pitch));
        const uint32_t b = row_bias(M.ld(M.u(i)) - lw_d(drr));
        if (sroot && s == 0) sroot[i] = lw_root(drr);
        best0 = umin64(best0, pack_key(static_cast<uint32_t>(c.x) + b, i));
        best1 = umin64(best1, pack_key(static_cast<uint32_t>(c.y) + b, i));
        best2 = umin64(best2, pack_key(static_cast<uint32_t>(c.z) + b, i));
        best3 = umin64(best3, pack_key(static_cast<uint32_t>(c.w) + b, i));
      }
    }
    // merge lanes of the same segment inside the warp (power-of-two S only:
    // they then differ in their high lane bits; otherwise every thread's keys
    // go straight to the shared atomics)
    const bool merge = Sreal < 32 && (Sreal & (Sreal - 1)) == 0;
    if (merge) {
      for (int o = Sreal; o < 32; o <<= 1) {
        best0 = umin64(best0, __shfl_xor_sync(0xffffffffu, best0, o));
        best1 = umin64(best1, __shfl_xor_sync(0xffffffffu, best1, o));
        best2 = umin64(best2, __shfl_xor_sync(0xffffffffu, best2, o));
        best3 = umin64(best3, __shfl_xor_sync(0xffffffffu, best3, o));
      }
    }
    const bool writer = (g < R) && (!merge || lane < Sreal);
    if (writer && best0 != KMB_KEY_INF) {
      unsigned long long* k4 = reinterpret_cast<unsigned long long*>(skey + 4 * s);
      atomicMin(k4 + 0, best0);
      atomicMin(k4 + 1, best1);
      atomicMin(k4 + 2, best2);
      atomicMin(k4 + 3, best3);
    }
  }
}

// ---- K3': the epoch-start relax restricted to the slab's dirty segments -------
// After an epoch's trees are dissolved, only columns whose key was reset (their
// argmin row left, or they were reached inside a dissolved tree) can change when
// the surviving rows are relaxed again: every other unreached key is a minimum
// attained at a surviving row.  So the survivors are relaxed over
// the dirty 4-column segments only — the same keys as a full relax, at a few
// percent of the bytes (c5: ~94% of all relaxed rows are these re-relaxes).
// segs[0, nd) lists the dirty segments; thread (g, k) handles segs[k] for row
// group g, with k in [0, np2), np2 = nd rounded up to a power of two (lanes of
// the same k differ only in high lane bits, so a xor tree merges them).
template <class Mem>
__device__ __forceinline__ void relax_sel(const int32_t* C, int64_t pitch, const Mem& M, int p,
                                          int head, int tail, int c0, const int32_t* segs, int nd,
                                          uint64_t* skey) {
  int np2 = 1;
  while (np2 < nd) np2 <<= 1;
  const int R = kThreads / np2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int k = tid % np2, g = tid / np2;
  uint64_t best0 = KMB_KEY_INF, best1 = KMB_KEY_INF, best2 = KMB_KEY_INF, best3 = KMB_KEY_INF;
  const int sg = k < nd ? segs[k] : 0;
  if (k < nd) {
    const int32_t* base = C + c0 + 4 * sg;
    int r = head + g;
    for (; r + (kRelaxBatch - 1) * R < tail; r += kRelaxBatch * R) {
      int i[kRelaxBatch];
      uint32_t b[kRelaxBatch];
      int4 c[kRelaxBatch];
      int64_t dr[kRelaxBatch];
#pragma unroll
      for (int q = 0; q < kRelaxBatch; ++q) {
        i[q] = M.ld(M.list_row(p, r + q * R));
        dr[q] = M.ld(M.list_w(p, r + q * R));
      }
#pragma unroll
      for (int q = 0; q < kRelaxBatch; ++q) {
        c[q] = ld_stream(reinterpret_cast<const int4*>(base + static_cast<int64_t>(i[q]) * pitch));
        b[q] = row_bias(M.ld(M.u(i[q])) - lw_d(dr[q]));
      }
#pragma unroll
      for (int q = 0; q < kRelaxBatch; ++q) {
        best0 = umin64(best0, pack_key(static_cast<uint32_t>(c[q].x) + b[q], i[q]));
        best1 = umin64(best1, pack_key(static_cast<uint32_t>(c[q].y) + b[q], i[q]));
        best2 = umin64(best2, pack_key(static_cast<uint32_t>(c[q].z) + b[q], i[q]));
        best3 = umin64(best3, pack_key(static_cast<uint32_t>(c[q].w) + b[q], i[q]));
      }
    }
    for (; r < tail; r += R) {
      const int i = M.ld(M.list_row(p, r));
      const int64_t drr = M.ld(M.list_w(p, r));
      const int4 c = ld_stream(reinterpret_cast<const int4*>(base + static_cast<int64_t>(i) * pitch));
      const uint32_t b = row_bias(M.ld(M.u(i)) - lw_d(drr));
      best0 = umin64(best0, pack_key(static_cast<uint32_t>(c.x) + b, i));
      best1 = umin64(best1, pack_key(static_cast<uint32_t>(c.y) + b, i));
      best2 = umin64(best2, pack_key(static_cast<uint32_t>(c.z) + b, i));
      best3 = umin64(best3, pack_key(static_cast<uint32_t>(c.w) + b, i));
    }
  }
  if (np2 < 32) {
    for (int o = np2; o < 32; o <<= 1) {
      best0 = umin64(best0, __shfl_xor_sync(0xffffffffu, best0, o));
      best1 = umin64(best1, __shfl_xor_sync(0xffffffffu, best1, o));
      best2 = umin64(best2, __shfl_xor_sync(0xffffffffu, best2, o));
      best3 = umin64(best3, __shfl_xor_sync(0xffffffffu, best3, o));
    }
  }
  const bool writer = k < nd && (np2 >= 32 || lane < np2);
  if (writer && best0 != KMB_KEY_INF) {
    unsigned long long* k4 = reinterpret_cast<unsigned long long*>(skey + 4 * sg);
    atomicMin(k4 + 0, best0);
    atomicMin(k4 + 1, best1);
    atomicMin(k4 + 2, best2);
    atomicMin(k4 + 3, best3);
  }
}

// ---- the persistent engine ---------------------------------------------------
// Incremental epochs (CPU mirror kmm_solve_incr): the search is
// never restarted.  When a round absorbs free columns, the trees owning one are
// augmented and dissolved (their rows/columns finalised and un-reached), columns
// whose argmin row left are reset, the surviving rows are relaxed once more over
// the reset ("dirty") columns only — the rows appended in the epoch's last round
// having been relaxed over the whole slab first — and the search goes on at the
// same D.
template <class Barrier, int MK>  // MK: 0 GMem, 1 DMem, 2 RMem (column-sharded ranks)
__device__ __forceinline__ void solve_body(const SolverArgs& a, const ShardDevArgs* sh) {
  constexpr bool DSM = MK == 1, RS = MK == 2;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int W = a.W;
  uint64_t* skey = reinterpret_cast<uint64_t*>(dyn);
  int64_t* vloc = reinterpret_cast<int64_t*>(skey + W);
  int64_t* dcol = vloc + W;
  unsigned char* rch = reinterpret_cast<unsigned char*>(dcol + W);
  int32_t* dsegs = reinterpret_cast<int32_t*>(rch + W);  // dirty segments (W/4)
  // grid / sharded engines: the roots of the rows this CTA relaxed (n) and the
  // matches of its slab columns (W), so the absorb reads no global state
  const bool cache = !DSM && a.slab_cache;
  int32_t* sroot = cache ? dsegs + (W >> 2) : nullptr;
  int32_t* smatch = cache ? sroot + a.n : nullptr;
  __shared__ SlabSmem sm;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // column-sharded ranks (RS): this launch holds ranks rank_base, ... (gridDim.x /
  // Gr of them); gb is the CTA's index over all ranks' CTAs, G their count
  const int Gr = RS ? sh->Gr : 1;
  const int grank = RS ? sh->rank_base + static_cast<int>(blockIdx.x) / Gr : 0;
  const int lbr = RS ? static_cast<int>(blockIdx.x) % Gr : 0;
  const int gb = RS ? grank * Gr + lbr : static_cast<int>(blockIdx.x);
  const int G = RS ? sh->R * Gr : static_cast<int>(gridDim.x);
  const int c0 = gb * W;                     // the slab's first column
  const int cl0 = RS ? lbr * W : c0;         // ... in the cost block this rank holds
  const int32_t* const Cb = RS ? sh->slab[grank] : a.C;
  const int64_t pitch = RS ? sh->slab_pitch : a.pitch;
  const bool leader = (gb == 0 && tid == 0);
  Barrier bar = Barrier::make(&a.ctrl->bar_counter, static_cast<unsigned>(G));
  Ctrl* ctrl = a.ctrl;
  const int gtid = gb * kThreads + tid;
  const int gthreads = G * kThreads;

  using Mem = std::conditional_t<DSM, DMem, std::conditional_t<RS, RMem, GMem>>;
  Mem M;
  if constexpr (DSM) {  // carve the distributed arrays, copy k_init_rows' state in
    const int L = (a.n + G - 1) / G;
    unsigned char* q = dyn + solver_smem_bytes_dev(W);
    auto take = [&](size_t bytes) {
      unsigned char* r = q;
      q += (bytes + 15) & ~static_cast<size_t>(15);
      return r;
    };
    M.lw[0] = reinterpret_cast<int64_t*>(take(8ull * L));
    M.lw[1] = reinterpret_cast<int64_t*>(take(8ull * L));
    M.u_ = reinterpret_cast<int64_t*>(take(8ull * L));
    M.claim_ = reinterpret_cast<uint32_t*>(take(4ull * L));
    M.lrow[0] = reinterpret_cast<int32_t*>(take(4ull * L));
    M.lrow[1] = reinterpret_cast<int32_t*>(take(4ull * L));
    M.root_ = reinterpret_cast<int32_t*>(take(4ull * L));
    M.mrow_ = reinterpret_cast<int32_t*>(take(4ull * L));
    M.mcol_ = reinterpret_cast<int32_t*>(take(4ull * L));
    M.tpar_ = reinterpret_cast<int32_t*>(take(4ull * L));
    M.found_ = reinterpret_cast<int32_t*>(take(4ull * L));
    M.cnt = reinterpret_cast<int*>(take(8 * 4));
    M.part = reinterpret_cast<int64_t*>(take(8));
    M.shift = __ffs(G) - 1;
    M.mask = G - 1;
    for (int k = tid; k < L; k += kThreads) {
      const int i = k * G + static_cast<int>(blockIdx.x);
      if (i >= a.n) break;
      M.u_[k] = ldcg(a.u + i);
      M.claim_[k] = 0xFFFFFFFFu;  // unclaimed (k_init_rows' all-ones)
      M.lrow[0][k] = ldcg(a.list_row[0] + i);
      M.lw[0][k] = ldcg(a.list_w[0] + i);
      M.root_[k] = ldcg(a.root_row + i);
      M.mrow_[k] = ldcg(a.match_row + i);
      M.mcol_[k] = ldcg(a.match_col + i);
    }
    if (tid < 6) M.cnt[tid] = 0;
    bar.sync();  // every CTA's copy in place before any remote access
  } else if constexpr (RS) {
    __shared__ unsigned char* rbases[KMB_MAX_RANKS];
    if (tid < sh->R) rbases[tid] = sh->rep[tid];
    __syncthreads();
    M.bases = rbases;
    M.mine = rbases[grank];
    M.R = sh->R;
    M.n = a.n;
    M.o32 = shard_rep_o32(a.n, G);
    M.ctrl = ctrl;
    M.claim_h = a.claim;
  } else {
    M.a = &a;
  }

  if constexpr (RS) {
    // K1 over the rank's slab (k_init_rows for one rank): validation and the
    // row minima of this rank's columns, combined over the ranks through the
    // home block; each rank initialises its own replica
    const int wl = lbr * (kThreads / 32) + wid, nwl = Gr * (kThreads / 32);
    const int ncl = min(Gr * W, a.n - grank * Gr * W);  // this rank's real columns
    for (int i = wl; i < a.n; i += nwl) {
      int32_t lo = 0x7fffffff, hi = 0;
      const int32_t* row = Cb + static_cast<int64_t>(i) * pitch;
      for (int j = lane; j < ncl; j += 32) {
        const int32_t x = __ldg(row + j);
        lo = min(lo, x);
        hi = max(hi, x);
      }
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      if (lane == 0) {
        if (lo < 0) atomicMax(&ctrl->status, 2);               // KMB_ENEGATIVE
        else if (hi >= (1 << 29)) atomicMax(&ctrl->status, 3);  // KMB_ERANGE
        sh->rowmin[static_cast<int64_t>(grank) * a.n + i] = lo;
        *M.list_row(0, i).local() = i;
        *M.list_w(0, i).local() = static_cast<int64_t>(i) << 32;
        *M.root_row(i).local() = i;
        *M.match_row(i).local() = -1;
        *M.match_col(i).local() = -1;
        if (grank == 0) a.claim[i] = KMB_KEY_INF;
      }
    }
  }
  if (tid == 0) {
    sm.my_rows = sm.my_frees = 0;
    sm.tot_rows = sm.tot_frees = 0;
  }
  // Shared append counters are triple-buffered by barrier index: appends made
  // between barriers k-1 and k go to cnt[k % 3], every CTA reads it right after
  // barrier k, and the leader clears cnt[(k+2) % 3] after barrier k (last read
  // after barrier k-1, next used after barrier k+1), so a fast CTA's appends
  // never race a slow CTA's read.
  int kb = 0;
  // Grid engine: the barrier word also carries the append totals (each CTA
  // adds 1 | rows << 16 | frees << 40), so nobody re-reads the counters after
  // it — one L2 round trip less per barrier.  Other engines read the counters.
  // The sharded engine's ranks may be GPUs: system-scope release / acquire.
  constexpr bool kCounted = std::is_same_v<Barrier, GridBarrier> && !DSM;
  if (tid == 0) sm.abort = 0;
  // returns false when the sharded ranks' barrier timed out (then every CTA
  // that waited leaves the solve; the host reports the status)
  auto gsync = [&]() -> bool {
    if constexpr (kCounted) {
      __syncthreads();
      if (tid == 0) {
        unsigned long long* w = &ctrl->cbar[(kb + 1) % 3];
        const unsigned long long add = 1ull | (static_cast<unsigned long long>(sm.my_rows) << 16) |
                                       (static_cast<unsigned long long>(sm.my_frees) << 40);
        // KMB_POLL_RELAXED: poll relaxed, then one acquire load of the
        // completed word (it reads the last arrival's add, so it synchronises
        // with every arrival's release; the word cannot be cleared in between:
        // that happens after the next barrier).  Otherwise every poll is an
        // acquire (an L1 invalidation each, but no extra round trip at the end).
        unsigned long long v;
        if (RS && sh->sys) {  // ranks on several GPUs: system scope
          // a rank whose kernel never started (or died) must not leave the
          // others spinning: after 20 s without the barrier completing every
          // waiting CTA gives up and the solve reports an error
          asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(w), "l"(add) : "memory");
          const unsigned long long t_wait = globaltimer_ns();
          do {
            v = KMB_POLL_RELAXED ? ld_relaxed_sys_u64(w) : ld_acquire_sys_u64(w);
            if ((v & 0xFFFFull) < static_cast<unsigned long long>(G) &&
                globaltimer_ns() - t_wait > 20000000000ull) {
              sm.abort = 1;
              break;
            }
          } while ((v & 0xFFFFull) < static_cast<unsigned long long>(G));
          if (KMB_POLL_RELAXED) v = ld_acquire_sys_u64(w);
        } else {
          asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(w), "l"(add) : "memory");
          do {
            v = KMB_POLL_RELAXED ? ld_relaxed_u64(w) : ld_acquire_u64(w);
          } while ((v & 0xFFFFull) < static_cast<unsigned long long>(G));
          if (KMB_POLL_RELAXED) v = ld_acquire_u64(w);
        }
        sm.tot_rows = static_cast<int32_t>((v >> 16) & 0xFFFFFFull);
        sm.tot_frees = static_cast<int32_t>(v >> 40);
        sm.my_rows = sm.my_frees = 0;
      }
      __syncthreads();
    } else {
      bar.sync();
    }
    ++kb;
    if (leader) {
      *M.rcnt((kb + 2) % 3) = 0;
      *M.fcnt((kb + 2) % 3) = 0;
      if constexpr (kCounted) ctrl->cbar[(kb + 2) % 3] = 0;
    }
    if (RS && sm.abort) {
      if (tid == 0) atomicExch(&ctrl->status, -3);
      return false;
    }
    return true;
  };
  if constexpr (RS) {
    if (!gsync()) return;  // every rank's row minima and replica in place
    const int lt = lbr * kThreads + tid, nlt = Gr * kThreads;
    for (int i = lt; i < a.n; i += nlt) {
      int32_t lo = 0x7fffffff;
      for (int r = 0; r < sh->R; ++r) lo = min(lo, ldcg(sh->rowmin + static_cast<int64_t>(r) * a.n + i));
      *M.u(i).local() = a.seed == 1 ? lo : 0;  // hungarian.cpp:323-327
    }
    if (!gsync()) return;
  }
  if (ldcg(&ctrl->status) != 0) return;  // invalid input (k_init_rows), all CTAs agree
  for (int c = tid; c < W; c += kThreads) {
    vloc[c] = 0;  // seed 0: v = 0
    skey[c] = KMB_KEY_INF;
    rch[c] = (c0 + c < a.n) ? 0 : 1;  // padding columns never count
    if (cache) smatch[c] = -1;
  }
  __syncthreads();
  int64_t dual_steps = 0, rows_scanned = 0, seg_rows = 0;
  // stage clock (leader only): 0 relax + absorb + local min, 1 B1, 2 dual-step absorb,
  // 3 B2 (dual steps only), 4 epoch end, 5 B3
  long long prof[6] = {0, 0, 0, 0, 0, 0};
  long long rounds_total = 0;
  unsigned long long tprev = leader ? globaltimer_ns() : 0ull;
#define KMB_STAGE(k)                                   \
  do {                                                 \
    if (leader) {                                      \
      const unsigned long long t_ = globaltimer_ns();  \
      prof[k] += static_cast<long long>(t_ - tprev);   \
      tprev = t_;                                      \
    }                                                  \
  } while (0)
  unsigned long long deadline = a.deadline_ns;
  if (deadline >> 63) deadline = globaltimer_ns() + (deadline & ~(1ull << 63));  // relative budget

  auto got_rows = [&]() { return kCounted ? sm.tot_rows : M.ld(M.rcnt(kb % 3)); };
  auto got_frees = [&]() { return kCounted ? sm.tot_frees : M.ld(M.fcnt(kb % 3)); };
  int64_t D = 0;
  int p = 0, epoch = 0, head = 0, tail = a.n;  // rows list[p][0, tail) are reached
  int nfound = 0;                              // free columns absorbed this epoch
  bool fatal = false, stopped = false;
  bool dirty_round = false;  // this round re-relaxes survivors over dirty segments only
  if (tid == 0) sm.ndseg = 0;
#if KMB_SOLVER_FINE
  long long fine[4] = {0, 0, 0, 0};  // leader: relax issue->done, sync, absorb, min
  long long fl = clock64();
#define KMB_FINE(k)                    \
  do {                                 \
    if (leader) {                      \
      const long long t_ = clock64();  \
      fine[k] += t_ - fl;              \
      fl = t_;                         \
    }                                  \
  } while (0)
#else
#define KMB_FINE(k) (void)0
#endif
  for (;;) {
    KMB_FINE(3);
    if (dirty_round) {
      dirty_round = false;
      if (sm.ndseg > 0) relax_sel(Cb, pitch, M, p, head, tail, cl0, dsegs, sm.ndseg, skey);
      seg_rows += static_cast<int64_t>(tail - head) * sm.ndseg;
    } else {
      relax_slab(Cb, pitch, M, p, head, tail, cl0, W, skey, sroot);
      rows_scanned += tail - head;
    }
    KMB_FINE(0);
    __syncthreads();
    KMB_FINE(1);
    // a valid search ends within n epochs of at most 2n + 1 rounds each; every
    // CTA counts the same rounds, so all of them stop together if it does not
    if (rounds_total > 4ll * a.n * a.n + 64) {
      if (leader) ctrl->status = -2;
      fatal = true;
      break;
    }
    if (rounds_total == 0 && a.seed == 1)  // column reduction, hungarian.cpp:328-333
      for (int c = tid; c < W; c += kThreads)
        if (c0 + c < a.n) vloc[c] = key_val(skey[c]);
    ++rounds_total;
    // absorb the slab's tight columns at the current D (hungarian.cpp:186-199):
    // tightness is a per-column test, no global information needed
    auto absorb_at = [&](int64_t Dn) {
      int* rc = M.rcnt((kb + 1) % 3);
      int* fc = M.fcnt((kb + 1) % 3);
      for (int cb = 0; cb < W; cb += kThreads) {
        const int c = cb + tid;
        bool newrow = false, newfree = false;
        int32_t i2 = -1, col = c0 + c, root = 0;
        if (c < W && !rch[c] && key_val(skey[c]) - vloc[c] == Dn) {
          rch[c] = 1;
          dcol[c] = Dn;
          const int32_t par = key_row(skey[c]);
          *M.tree_par(col) = par;
          root = cache ? sroot[par] : M.ld(M.root_row(par));
          i2 = cache ? smatch[c] : M.ld(M.match_col(col));
          if (i2 < 0) {
            newfree = true;
            M.claim_min(root, M.ckey(epoch, col));
          } else {
            newrow = true;  // the list keeps D at reach; w = u - Dn is formed by the relax
            *M.root_row(i2) = root;
#if KMB_SOLVER_PREFETCH
            // every CTA scans this row next round: start pulling it into L2 now,
            // so the barrier and the list reads hide the DRAM latency
            // (sharded: this rank's slab row; a rank cannot prefetch into a
            // peer GPU's L2)
            if (a.prefetch_rows)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                               (RS ? sh->slab[grank] : a.C) + static_cast<int64_t>(i2) * pitch),
                           "r"(static_cast<uint32_t>((RS ? static_cast<int64_t>(Gr) * W : pitch) * 4))
                           : "memory");
#endif
          }
        }
        // warp-aggregated appends
        const unsigned rowmask = __ballot_sync(0xffffffffu, newrow);
        if (rowmask) {
          int base = 0;
          if (lane == 0) {
            base = atomicAdd(rc, __popc(rowmask));
            if (kCounted) atomicAdd(&sm.my_rows, __popc(rowmask));
          }
          base = __shfl_sync(0xffffffffu, base, 0);
          if (newrow) {
            const int pos = tail + base + __popc(rowmask & ((1u << lane) - 1));
            *M.list_row(p, pos) = i2;
            *M.list_w(p, pos) = lw_pack(Dn, root);
          }
        }
        const unsigned fmask = __ballot_sync(0xffffffffu, newfree);
        if (fmask) {
          int base = 0;
          if (lane == 0) {
            base = atomicAdd(fc, __popc(fmask));
            if (kCounted) atomicAdd(&sm.my_frees, __popc(fmask));
          }
          base = __shfl_sync(0xffffffffu, base, 0);
          if (newfree) *M.found(nfound + base + __popc(fmask & ((1u << lane) - 1))) = col;
        }
      }
    };
    absorb_at(D);
    __syncthreads();
    KMB_FINE(2);
    // min slack' of the columns still unreached: only used if no CTA progressed
    int64_t lm = KMB_I64_INF;
    for (int c = tid; c < W; c += kThreads)
      if (!rch[c]) {
        const int64_t s = key_val(skey[c]) - vloc[c];
        lm = s < lm ? s : lm;
      }
    lm = warp_min_i64(lm);
    if (lane == 0) sm.part[wid] = lm;
    __syncthreads();
    if (wid == 0) {
      int64_t x = lane < kThreads / 32 ? sm.part[lane] : KMB_I64_INF;
      x = warp_min_i64(x);
      if (lane == 0) *M.partial(gb) = x;
    }
    KMB_STAGE(0);
    if (!gsync()) {  // ---------------------------------------------- B1
      fatal = true;
      break;
    }
    KMB_STAGE(1);
    int added = got_rows();
    int fadded = got_frees();
    if (added == 0 && fadded == 0) {
      // no tight column anywhere and no pending row: dual step (:201-215)
      if (wid == 0) {
        int64_t x = KMB_I64_INF;
        for (int b = lane; b < G; b += 32) {
          const int64_t y = M.ld(M.partial(b));
          x = y < x ? y : x;
        }
        x = warp_min_i64(x);
        if (lane == 0) sm.m = x;
      }
      __syncthreads();
      const int64_t m = sm.m;
      if (m == KMB_I64_INF) {  // no unreached column: cannot happen on valid input
        if (leader) ctrl->status = -2;
        fatal = true;
        break;
      }
      D = m;
      ++dual_steps;
      absorb_at(D);
      KMB_STAGE(2);
      if (!gsync()) {  // ------------------------------------------ B2 (dual steps only)
        fatal = true;
        break;
      }
      KMB_STAGE(3);
      added = got_rows();
      fadded = got_frees();
    }
    head = tail;
    tail += added;
    nfound += fadded;
    if (nfound == 0) continue;

    // ---- epoch end: augment and dissolve the trees that reached a free column ----
    // First relax the rows appended this round over the whole slab (the next
    // round re-relaxes survivors over dirty segments only, so every survivor
    // must already be in the keys); a key whose argmin is one of them that gets
    // dissolved is reset below like any other.
    relax_slab(Cb, pitch, M, p, head, tail, cl0, W, skey, sroot);
    rows_scanned += tail - head;
    __syncthreads();
    // columns of the slab: finalise dissolved ones, reset keys whose argmin row leaves
    for (int c = tid; c < W; c += kThreads) {
      const int col = c0 + c;
      if (col >= a.n) continue;
      if (rch[c]) {
        const int32_t root = M.ld(M.root_row(M.ld(M.tree_par(col))));
        if (M.claimed(M.ld(M.claim(root)), epoch)) {
          vloc[c] -= D - dcol[c];
          rch[c] = 0;
          skey[c] = KMB_KEY_INF;
        }
      } else if (skey[c] != KMB_KEY_INF) {
        const int32_t root = M.ld(M.root_row(key_row(skey[c])));
        if (M.claimed(M.ld(M.claim(root)), epoch)) skey[c] = KMB_KEY_INF;
      }
    }
    // dirty segments: 4-column groups holding an unreached column whose key
    // was just reset (only those change when the survivors are relaxed again)
    __syncthreads();
    if (tid == 0) sm.ndseg = 0;
    __syncthreads();
    for (int sgi = tid; sgi < (W >> 2); sgi += kThreads) {
      bool d = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = 4 * sgi + q;
        d |= !rch[c] && skey[c] == KMB_KEY_INF;
      }
      if (d) dsegs[atomicAdd(&sm.ndseg, 1)] = sgi;
    }
    // rows: finalise dissolved ones (u = w + D), carry the survivors over
    int* sc = M.rcnt((kb + 1) % 3);
    for (int r = gtid; r < tail; r += gthreads) {
      const int32_t i = M.ld(M.list_row(p, r));
      const int64_t dr = M.ld(M.list_w(p, r));
      if (M.claimed(M.ld(M.claim(M.ld(M.root_row(i)))), epoch)) {
        // u = w + D.  (Another CTA's epoch-end relax of this row, if it was
        // appended this round, may read u before or after this write: either
        // way every key it could set has this dissolved row as argmin and is
        // reset by that CTA's column pass.)
        *M.u(i) = M.ld(M.u(i)) - lw_d(dr) + D;
      } else {
        const int pos = atomicAdd(sc, 1);
        if (kCounted) atomicAdd(&sm.my_rows, 1);
        *M.list_row(p ^ 1, pos) = i;
        *M.list_w(p ^ 1, pos) = dr;
      }
    }
    // flip one parent-pointer path per claimed tree (its smallest free column)
    int won = 0;
    for (int f = gtid; f < nfound; f += gthreads) {
      int32_t j = M.ld(M.found(f));
      const int32_t root = M.ld(M.root_row(M.ld(M.tree_par(j))));
      if (M.ld(M.claim(root)) != M.ckey(epoch, j)) continue;
      ++won;
      for (;;) {
        const int32_t i = M.ld(M.tree_par(j));
        const int32_t nxt = M.ld(M.match_row(i));
        *M.match_row(i) = j;
        *M.match_col(j) = i;
        if (nxt < 0) break;
        j = nxt;
      }
    }
    won = __reduce_add_sync(0xffffffffu, won);
    if (lane == 0 && won) atomicAdd(&ctrl->matched, won);
    if (leader) {
      ctrl->phases = epoch + 1;
      if (deadline && globaltimer_ns() > deadline) ctrl->stop = 1;
    }
    KMB_STAGE(4);
    if (!gsync()) {  // ---------------------------------------------- B3
      fatal = true;
      break;
    }
    KMB_STAGE(5);
    p ^= 1;
    ++epoch;
    head = 0;
    tail = got_rows();  // survivors
    if (cache)  // the augmenting paths just flipped some of this slab's matches
      for (int c = tid; c < W; c += kThreads) smatch[c] = c0 + c < a.n ? M.ld(M.match_col(c0 + c)) : -1;
    dirty_round = true;
    nfound = 0;
    if (ldcg(&ctrl->matched) == a.n) break;
    if (ldcg(&ctrl->stop) != 0) {
      stopped = true;
      break;
    }
  }
  if (stopped) {  // time budget: write back the surviving trees' lazy duals
    for (int r = gtid; r < tail; r += gthreads) {
      const int32_t i = M.ld(M.list_row(p, r));
      *M.u(i) = M.ld(M.u(i)) - lw_d(M.ld(M.list_w(p, r))) + D;
    }
    for (int c = tid; c < W; c += kThreads)
      if (rch[c] && c0 + c < a.n) vloc[c] -= D - dcol[c];
  }
  if constexpr (DSM) {  // results back to global (u, matching); no remote access after
    bar.sync();
    const int L = (a.n + G - 1) / G;
    for (int k = tid; k < L; k += kThreads) {
      const int i = k * G + static_cast<int>(blockIdx.x);
      if (i >= a.n) break;
      a.u[i] = M.u_[k];
      a.match_row[i] = M.mrow_[k];
      a.match_col[i] = M.mcol_[k];
    }
  }
  (void)fatal;
  int64_t* const vo = RS ? sh->vout[grank] + cl0 : a.v + c0;
  for (int c = tid; c < W; c += kThreads)
    if (c0 + c < a.n) vo[c] = vloc[c];
  if constexpr (RS) {  // K10 over the slab: sum of C[match_col[j]][j] (core.cpp:76-90)
    long long o = 0;
    for (int c = tid; c < W; c += kThreads)
      if (c0 + c < a.n) {
        const int32_t i = M.ld(M.match_col(c0 + c));
        if (i >= 0) o += Cb[static_cast<int64_t>(i) * pitch + cl0 + c];
      }
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) o += __shfl_xor_sync(0xffffffffu, o, q);
    if (lane == 0 && o) atomicAdd(&ctrl->obj, static_cast<unsigned long long>(o));
  }
#if KMB_SOLVER_FINE
  if (leader)
    printf("k_solve leader fine (cycles/round over %lld rounds): relax %lld, sync %lld, absorb %lld, other %lld\n",
           rounds_total, fine[0] / rounds_total, fine[1] / rounds_total, fine[2] / rounds_total,
           fine[3] / rounds_total);
#endif
  if (tid == 0 && seg_rows)
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctrl->seg_rows),
              static_cast<unsigned long long>(seg_rows));
  if (leader) {
    ctrl->free_rows = a.n - ldcg(&ctrl->matched);
    ctrl->dual_steps = dual_steps;
    ctrl->rows_scanned = rows_scanned;
    ctrl->rounds = rounds_total;
    for (int k = 0; k < 6; ++k) ctrl->stage_ns[k] = prof[k];
  }
}

template <class Barrier, bool DSM>
__global__ void __launch_bounds__(kThreads, 1) k_solve(SolverArgs a) {
  solve_body<Barrier, DSM ? 1 : 0>(a, nullptr);
}

// column-sharded ranks with a replicated row side (RMem); `sh` in device memory
__global__ void __launch_bounds__(kThreads, 1) k_solve_sharded(SolverArgs a, const ShardDevArgs* sh) {
  solve_body<GridBarrier, 2>(a, sh);
}

// ---- full-frontier scan microbenchmark ------------------------------------------
// The engine's reduced-cost scan (relax_slab) with every row in the frontier:
// one pass over the whole n x n matrix per launch, keys written out so the pass
// cannot be elided.  Measures what K3 sustains from HBM when it is not waiting
// on barriers ("full-matrix pass").
__global__ void __launch_bounds__(kThreads, 1) k_scan_all(SolverArgs a, uint64_t* keys_out) {
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* skey = reinterpret_cast<uint64_t*>(dyn);
  const int W = a.W, c0 = blockIdx.x * W;
  for (int c = threadIdx.x; c < W; c += kThreads) skey[c] = KMB_KEY_INF;
  __syncthreads();
  relax_slab<GMem, kScanBatch>(a.C, a.pitch, GMem{&a}, 0, 0, a.n, c0, W, skey);
  __syncthreads();
  for (int c = threadIdx.x; c < W; c += kThreads)
    if (c0 + c < a.n) keys_out[c0 + c] = skey[c];
}

cudaError_t launch_scan_all(const SolverArgs& a, int G, uint64_t* keys_out, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(a.W) * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_scan_all, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  k_scan_all<<<G, kThreads, smem, st>>>(a, keys_out);
  return cudaGetLastError();
}

// ---- K10: objective  sum_i C[i][match_row[i]] (core.cpp:76-90, int64) -------
__global__ void k_objective(const int32_t* C, int64_t pitch, int n, const int32_t* match_row,
                            unsigned long long* out) {
  int64_t s = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = match_row[i];
    if (j >= 0) s += C[static_cast<int64_t>(i) * pitch + j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(s));
}

size_t solver_smem_bytes(int W) { return solver_smem_bytes_dev(W); }

cudaError_t launch_solver_init(const SolverArgs& a, cudaStream_t st) {
  k_init_rows<<<256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_solver(const SolverArgs& a, int G, bool cluster, cudaStream_t st) {
  cudaError_t e = launch_solver_init(a, st);
  if (e != cudaSuccess) return e;
  const size_t smem = solver_smem_bytes(a.W) + (a.slab_cache ? 4ull * (a.n + a.W) : 0);
  if (!cluster) {
    auto kern = k_solve<GridBarrier, false>;
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    void* params[] = {const_cast<SolverArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(G), dim3(kThreads), params,
                                       smem, st);
  }
  // one thread-block cluster of G <= 16 CTAs: hardware cluster barriers; the
  // search state in the cluster's distributed shared memory when G is a power
  // of two (element i -> CTA i mod G) and it fits
  static const bool no_dsm = getenv("KMB_NO_DSM") != nullptr;  // A/B switch
  // (the DSMEM claim words hold the column in 13 bits: n <= 8192)
  const bool dsm = !no_dsm && a.n <= 8192 && (G & (G - 1)) == 0 && smem + dsm_bytes(a.n, G) <= 200 * 1024;
  auto kern = dsm ? k_solve<ClusterBarrier, true> : k_solve<ClusterBarrier, false>;
  const size_t csmem = smem + (dsm ? dsm_bytes(a.n, G) : 0);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  if (csmem > 48 * 1024) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(csmem));
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = csmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_objective(const int32_t* C, int64_t pitch, int n, const int32_t* match_row,
                             unsigned long long* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  const int blocks = (n + 255) / 256 < 148 ? (n + 255) / 256 : 148;
  k_objective<<<blocks, 256, 0, st>>>(C, pitch, n, match_row, out);
  return cudaGetLastError();
}

int solver_threads() { return kThreads; }

size_t shard_rep_bytes(int n, int G) { return shard_rep_o32(n, G) + 4ull * 7 * n; }

cudaError_t launch_solver_sharded(const SolverArgs& a, const ShardDevArgs* sh_dev, int grid, cudaStream_t st) {
  const size_t smem = solver_smem_bytes(a.W) + (a.slab_cache ? 4ull * (a.n + a.W) : 0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_solve_sharded, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  void* params[] = {const_cast<SolverArgs*>(&a), const_cast<ShardDevArgs**>(&sh_dev)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_solve_sharded), dim3(grid), dim3(kThreads),
                                     params, smem, st);
}

}  // namespace kmb
