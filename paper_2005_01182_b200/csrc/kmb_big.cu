// Single-CTA engine ("big CTA", KMB_OPT_ENGINE 8): one 512-thread CTA solves
// one instance with 256 < n <= 4096 — configs 2 and 4 — entirely inside one SM.
//
// Why: those instances are latency-bound (c2: 6,709 rounds relaxing ~2 rows
// each; c4: 33,909 rounds of ~3), so the multi-CTA engines pay a cluster or
// grid barrier and DSMEM/L2 hops every round for almost no bandwidth.  Here a
// round's synchronisation is two __syncthreads and every piece of search state
// lives in this SM's shared memory; only the cost rows come from L2.
//
// The algorithm is the engines': lazy duals, packed
// (value, row) column keys, argmin-parent forest augmentation, incremental
// epochs, and the dirty-column epoch start — after the claimed trees dissolve,
// only the reset columns can change when the survivors are relaxed again, so
// they are recomputed cooperatively (threads split the survivor rows of each
// dirty column) instead of streaming every survivor row through one SM.
//
// Layout: thread t owns CPT columns in groups of V contiguous ones, group g at
// columns V·(t + g·T) .. V·(t + g·T) + V - 1, so a row is read with one V-wide
// load per group (V = 2 at two columns per thread, see launch_nt); per-column
// key / v / Dc in registers; per-row state, the row lists,
// parents, matching, 32-bit tree claims and the dirty-column list in shared
// memory (14n words: 224 KB at n = 4096).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <type_traits>

#include "kmb_common.cuh"
#include "kmb_internal.h"
#include "kmb_launch.h"

// survivor rows in flight per thread in the dirty-column recompute.  More does
// not help (c4: 8: 156, 16: 168, 32: 191 ms): the gathers are 4-byte loads
// from scattered sectors, bound by the SM's L1 request rate, not latency.
#ifndef KMB_BIG_GB
#define KMB_BIG_GB 8
#endif
#ifndef KMB_BIG_CLOCKS  // diagnostics: thread 0's stage cycles, printed per instance
#define KMB_BIG_CLOCKS 0
#endif
#if KMB_BIG_CLOCKS
#include <cstdio>
#define BIG_CLK(k)                  \
  do {                              \
    const long long t_ = clock64(); \
    clk[k] += t_ - clk_last;        \
    clk_last = t_;                  \
  } while (0)
#else
#define BIG_CLK(k) (void)0
#endif

namespace kmb {
namespace {

constexpr uint32_t FULL = 0xffffffffu;

// packed key: ((c - w + 2^30) << 32) | row — min = smallest reduced cost, ties
// to the smallest row (kmb_common.cuh)
struct BK {
  __device__ static uint32_t tag(int32_t w) { return static_cast<uint32_t>(static_cast<int32_t>(KMB_BIAS) - w); }
  __device__ static uint64_t make(int32_t c, uint32_t tag, int32_t row) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(c) + tag) << 32) | static_cast<uint32_t>(row);
  }
  __device__ static int32_t val(uint64_t k) {
    return static_cast<int32_t>(static_cast<int64_t>(k >> 32) - KMB_BIAS);
  }
  __device__ static int32_t row(uint64_t k) { return static_cast<int32_t>(static_cast<uint32_t>(k)); }
};

// tree claims: (epoch stamp, column) in 32 bits, smaller wins; columns < 4096
__device__ __forceinline__ uint32_t bclaim(int ep, int col) {
  return ((0xFFFFEu - static_cast<uint32_t>(ep)) << 12) | static_cast<uint32_t>(col);
}
__device__ __forceinline__ bool bclaimed(uint32_t c, int ep) {
  return (c >> 12) == 0xFFFFEu - static_cast<uint32_t>(ep);
}

struct BigShared {
  int32_t red[32];
  int32_t nrows, nfound, ns, won, nd;
  int32_t lo_all, hi_all, stop;
  unsigned long long tot;
};

// V contiguous int32 of a row (16·V-bit vector load of immutable costs)
template <int V>
__device__ __forceinline__ void load_vec(const int32_t* p, int32_t* out) {
  if constexpr (V == 4) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(p));
    out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
  } else if constexpr (V == 2) {
    const int2 x = __ldg(reinterpret_cast<const int2*>(p));
    out[0] = x.x; out[1] = x.y;
  } else {
    out[0] = __ldg(p);
  }
}

template <int CPT, int kT, int V>
__global__ void __launch_bounds__(kT, 1) k_big(BigArgs a) {
  static_assert(CPT % V == 0, "columns per thread must be whole vector groups");
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BigShared sm;
  const int n = a.n;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  // column of this thread's q-th slot
  auto colof = [&](int q) { return V * (t + (q / V) * kT) + (q % V); };
  int2* rows = reinterpret_cast<int2*>(dyn);
  int2* spare = rows + n;  // also the dirty-column keys in the round after an epoch end
  int32_t* u = reinterpret_cast<int32_t*>(spare + n);
  int32_t* w = u + n;
  int32_t* root_row = w + n;
  int32_t* match_row = root_row + n;
  int32_t* match_col = match_row + n;
  int32_t* tree_par = match_col + n;
  int32_t* found = tree_par + n;
  int32_t* dlist = found + n;  // dirty columns
  int32_t* dpos = dlist + n;   // column -> index in dlist (valid for dirty ones)
  uint32_t* claim = reinterpret_cast<uint32_t*>(dpos + n);

  for (int inst = blockIdx.x; inst < a.batch; inst += gridDim.x) {
    const int32_t* Cm = a.C + static_cast<int64_t>(inst) * a.inst_stride;
    const int64_t ld = a.ld;
    const unsigned long long t0 = globaltimer_ns();
    if (t == 0) {
      sm.lo_all = INT_MAX;
      sm.hi_all = 0;
      sm.nrows = n;
      sm.nfound = 0;
      sm.stop = 0;
      sm.tot = 0;
    }
    __syncthreads();
    // validation (core.cpp:144-145 + device range) and row reductions
    // (hungarian.cpp:323-327): one warp per row
    {
      int32_t lo_all = INT_MAX, hi_all = 0;
      for (int i = wid; i < n; i += kT / 32) {
        int32_t lo = INT_MAX, hi = 0;
        for (int k = lane; k < n; k += 32) {
          const int32_t x = __ldg(Cm + i * ld + k);
          lo = min(lo, x);
          hi = max(hi, x);
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        lo_all = min(lo_all, lo);
        hi_all = max(hi_all, hi);
        if (lane == 0) {
          const int32_t u0 = a.seed == 1 ? lo : 0;
          u[i] = u0;
          w[i] = u0;
        }
      }
      if (lane == 0) {
        atomicMin(&sm.lo_all, lo_all);
        atomicMax(&sm.hi_all, hi_all);
      }
    }
    for (int k = t; k < n; k += kT) {
      match_row[k] = -1;
      match_col[k] = -1;
      claim[k] = 0xFFFFFFFFu;
      root_row[k] = k;
    }
    __syncthreads();
    const int status0 = sm.lo_all < 0 ? 2 : (sm.hi_all >= (1 << 29) ? 3 : 0);
    if (status0) {  // invalid instance: no stale totals or stats for async callers
      if (t == 0) {
        a.status[inst] = status0;
        a.total_cost[inst] = 0;
        if (a.converged) a.converged[inst] = 0;
      }
      if (a.stats && t < KMB_ISTATS) a.stats[KMB_ISTATS * static_cast<int64_t>(inst) + t] = 0;
      for (int k = t; k < n; k += kT) a.row_to_col[static_cast<int64_t>(inst) * n + k] = -1;
      __syncthreads();
      continue;
    }
    for (int k = t; k < n; k += kT) rows[k] = make_int2(k, static_cast<int32_t>(BK::tag(w[k])));

    uint64_t key[CPT];
    int32_t v[CPT], dc[CPT];
    uint32_t rch = 0;  // bit q: column t + q*T reached (padding counts as reached)
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      key[q] = ~0ull;
      v[q] = 0;
      dc[q] = 0;
      if (colof(q) >= n) rch |= 1u << q;
    }
    int nrows = n, head = 0, nfree = n, nfound = 0;
    int32_t D = 0;
    int epochs = 0, dual_steps = 0, rounds = 0;
    int64_t rows_scanned = 0, dirty_elems = 0;
    bool dirty_round = false, stopped = false;
    int status = 0;
    __syncthreads();

    // relax rows[from, to) over all of this thread's columns.  The row count is
    // uniform across the CTA, so batches of exactly K rows (K = RB, then 2, 1)
    // issue no predicated-off work: a lone SM is issue-bound here (ncu: 67%
    // issue active, long-scoreboard stalls 9%).  Offsets are 32-bit (n <= 4096).
    const int ld32 = static_cast<int>(a.ld);
    auto relax_k = [&](int r, auto kc) {
      constexpr int K = decltype(kc)::value;
      int2 e[K];
      int32_t c[K][CPT];
#pragma unroll
      for (int k = 0; k < K; ++k) e[k] = rows[r + k];
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int g = 0; g < CPT / V; ++g) {
          const int col = V * (t + g * kT);  // the pitch is padded to V: a group is in or out
          if (col < n) load_vec<V>(Cm + (e[k].x * ld32 + col), &c[k][g * V]);
          else
#pragma unroll
            for (int h = 0; h < V; ++h) c[k][g * V + h] = 0;
        }
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const uint64_t kk = BK::make(c[k][q], static_cast<uint32_t>(e[k].y), e[k].x);
          key[q] = kk < key[q] ? kk : key[q];
        }
    };
    auto relax_full = [&](int from, int to) {
      constexpr int RB = CPT >= 4 ? 2 : (CPT == 2 ? 4 : 6);
      int r = from;
      for (; r + RB <= to; r += RB) relax_k(r, std::integral_constant<int, RB>{});
      if constexpr (RB > 2)
        for (; r + 2 <= to; r += 2) relax_k(r, std::integral_constant<int, 2>{});
      if (r < to) relax_k(r, std::integral_constant<int, 1>{});
    };

#if KMB_BIG_CLOCKS
    long long clk[6] = {0, 0, 0, 0, 0, 0}, clk_last = clock64();  // relax, dirty, min, absorb, epoch, sync
#endif
    while (nfree > 0) {
      if (rounds > 4 * n * n + 64) {  // a valid search ends in n epochs of <= 2n + 1 rounds
        status = -2;
        break;
      }
      ++rounds;
      // ---- relax (hungarian.cpp:164-172) ----
      if (!dirty_round) {
        relax_full(head, nrows);
        rows_scanned += nrows - head;
        BIG_CLK(0);
      } else {
        // epoch start: only the dirty (reset) columns change; threads split the
        // survivor rows of each dirty column, then the owners take the minima
        dirty_round = false;
        const int nd = sm.nd;
        // the old row list (spare after the swap) is dead: its 8n bytes hold the keys
        uint64_t* dkey = reinterpret_cast<uint64_t*>(spare);
        for (int k = t; k < nd; k += kT) dkey[k] = ~0ull;
        __syncthreads();
        if (nd > 0) {
          const int groups = max(1, kT / nd);  // row groups per dirty column
          for (int item = t; item < nd * groups; item += kT) {
            const int k = item % nd, g = item / nd;
            const int col = dlist[k];
            uint64_t best = ~0ull;
            constexpr int GB = KMB_BIG_GB;
            for (int r = g; r < nrows; r += groups * GB) {
              int2 e[GB];
              int32_t c[GB];
#pragma unroll
              for (int b = 0; b < GB; ++b) {
                const int rr = r + b * groups;
                e[b] = rr < nrows ? rows[rr] : make_int2(-1, 0);
              }
#pragma unroll
              for (int b = 0; b < GB; ++b) c[b] = e[b].x >= 0 ? __ldcg(Cm + e[b].x * ld + col) : 0;
#pragma unroll
              for (int b = 0; b < GB; ++b) {
                const uint64_t kk = e[b].x >= 0 ? BK::make(c[b], static_cast<uint32_t>(e[b].y), e[b].x) : ~0ull;
                best = kk < best ? kk : best;
              }
            }
            atomicMin(reinterpret_cast<unsigned long long*>(dkey + k), static_cast<unsigned long long>(best));
          }
          dirty_elems += static_cast<int64_t>(nd) * nrows;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int col = colof(q);
          if (col < n && !((rch >> q) & 1) && key[q] == ~0ull)
            key[q] = reinterpret_cast<const uint64_t*>(spare)[dpos[col]];
        }
        BIG_CLK(1);
      }
      head = nrows;
      if (epochs == 0 && rounds == 1 && a.seed == 1) {  // column reduction, :328-333
#pragma unroll
        for (int q = 0; q < CPT; ++q)
          if (!((rch >> q) & 1)) v[q] = BK::val(key[q]);
      }
      // ---- min unreached slack' (hungarian.cpp:203-206) ----
      int32_t s[CPT];
      int32_t lm = INT_MAX;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        s[q] = BK::val(key[q]) - v[q];
        if (!((rch >> q) & 1)) lm = min(lm, s[q]);
      }
      lm = __reduce_min_sync(FULL, lm);
      if (lane == 0) sm.red[wid] = lm;
      BIG_CLK(2);
      __syncthreads();
      BIG_CLK(5);
      const int32_t m = __reduce_min_sync(FULL, lane < kT / 32 ? sm.red[lane] : INT_MAX);
      if (m > D) {
        if (m == INT_MAX) {
          status = -2;
          break;
        }
        D = m;  // dual step (hungarian.cpp:207-215), applied lazily
        ++dual_steps;
      }
      // ---- absorb zero-slack columns (hungarian.cpp:186-199) ----
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        if (((rch >> q) & 1) || s[q] != D) continue;
        const int col = colof(q);
        rch |= 1u << q;
        dc[q] = D;
        const int32_t par = BK::row(key[q]);
        tree_par[col] = par;
        const int32_t root = root_row[par];
        const int32_t i2 = match_col[col];
        if (i2 < 0) {
          atomicMin(claim + root, bclaim(epochs, col));
          found[atomicAdd(&sm.nfound, 1)] = col;
        } else {
          const int32_t w2 = u[i2] - D;
          w[i2] = w2;
          root_row[i2] = root;
          rows[atomicAdd(&sm.nrows, 1)] = make_int2(i2, static_cast<int32_t>(BK::tag(w2)));
        }
      }
      BIG_CLK(3);
      __syncthreads();
      BIG_CLK(5);
      nrows = sm.nrows;
      nfound = sm.nfound;
      if (nfound == 0) continue;

      // ---- epoch end: augment and dissolve the trees that reached a free column.
      // The rows appended this round are relaxed over all columns first (the
      // dirty-column epoch start relies on every survivor being in the keys).
      relax_full(head, nrows);
      rows_scanned += nrows - head;
      if (t == 0) {
        sm.ns = 0;
        sm.won = 0;
        sm.nd = 0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int col = colof(q);
        if (col >= n) continue;
        if ((rch >> q) & 1) {
          if (bclaimed(claim[root_row[tree_par[col]]], epochs)) {
            v[q] -= D - dc[q];
            rch &= ~(1u << q);
            key[q] = ~0ull;
          }
        } else if (key[q] != ~0ull && bclaimed(claim[root_row[BK::row(key[q])]], epochs)) {
          key[q] = ~0ull;
        }
        if (!((rch >> q) & 1) && key[q] == ~0ull) {  // dirty: recomputed next round
          const int k = atomicAdd(&sm.nd, 1);
          dlist[k] = col;
          dpos[col] = k;
        }
      }
      for (int r = t; r < nrows; r += kT) {
        const int2 e = rows[r];
        if (bclaimed(claim[root_row[e.x]], epochs)) u[e.x] = w[e.x] + D;
        else spare[atomicAdd(&sm.ns, 1)] = e;
      }
      int won = 0;
      for (int f = t; f < nfound; f += kT) {
        int32_t j = found[f];
        if (claim[root_row[tree_par[j]]] != bclaim(epochs, j)) continue;
        ++won;
        for (;;) {  // flip the parent-pointer path
          const int32_t i = tree_par[j];
          const int32_t nx = match_row[i];
          match_row[i] = j;
          match_col[j] = i;
          if (nx < 0) break;
          j = nx;
        }
      }
      won = __reduce_add_sync(FULL, won);
      if (lane == 0 && won) atomicAdd(&sm.won, won);
      if (t == 0 && a.deadline_ns > 0 && globaltimer_ns() - t0 > static_cast<unsigned long long>(a.deadline_ns))
        sm.stop = 1;
      __syncthreads();
      nfree -= sm.won;
      nrows = sm.ns;
      int2* tmp = rows;
      rows = spare;
      spare = tmp;
      head = 0;
      nfound = 0;
      ++epochs;
      dirty_round = true;
      const int stop = sm.stop;
      __syncthreads();
      if (t == 0) {
        sm.nrows = nrows;
        sm.nfound = 0;
      }
      __syncthreads();
      BIG_CLK(4);
      if (stop && nfree > 0) {
        stopped = true;
        break;
      }
    }
#if KMB_BIG_CLOCKS
    if (t == 0 && inst == 0)
      printf("k_big n %d rounds %d epochs %d: relax %lld dirty %lld min %lld absorb %lld epoch %lld sync %lld (cycles/round; dirty and epoch per epoch: %lld %lld)\n",
             n, rounds, epochs, clk[0] / rounds, clk[1] / rounds, clk[2] / rounds, clk[3] / rounds,
             clk[4] / rounds, clk[5] / rounds, clk[1] / (epochs ? epochs : 1), clk[4] / (epochs ? epochs : 1));
#endif
    if (stopped) {  // time budget: write back the surviving trees' lazy duals
      for (int r = t; r < nrows; r += kT) {
        const int2 e = rows[r];
        u[e.x] = w[e.x] + D;
      }
#pragma unroll
      for (int q = 0; q < CPT; ++q)
        if (((rch >> q) & 1) && colof(q) < n) v[q] -= D - dc[q];
    }
    __syncthreads();
    // ---- outputs ----
    long long tot = 0;
    for (int k = t; k < n; k += kT) {
      const int32_t mr = match_row[k];
      a.row_to_col[static_cast<int64_t>(inst) * n + k] = mr;
      a.u[static_cast<int64_t>(inst) * n + k] = u[k];
      if (mr >= 0) tot += __ldg(Cm + k * ld + mr);
    }
#pragma unroll
    for (int q = 0; q < CPT; ++q)
      if (colof(q) < n) a.v[static_cast<int64_t>(inst) * n + colof(q)] = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) atomicAdd(&sm.tot, static_cast<unsigned long long>(tot));
    __syncthreads();
    if (t == 0) {
      a.total_cost[inst] = static_cast<int64_t>(sm.tot);
      a.status[inst] = (stopped && status == 0) ? 4 : status;  // 4: budget expired (host: converged = 0)
      if (a.converged) a.converged[inst] = (!stopped && status == 0) ? 1 : 0;
      if (a.stats) {
        int64_t* o = a.stats + KMB_ISTATS * static_cast<int64_t>(inst);
        o[0] = epochs;
        o[1] = dual_steps;
        o[2] = rows_scanned;
        o[3] = rounds;
        o[4] = static_cast<int64_t>(globaltimer_ns() - t0);
        o[5] = dirty_elems;
        o[6] = o[7] = o[8] = 0;
        o[9] = static_cast<int64_t>(t0);
        o[10] = static_cast<int64_t>(globaltimer_ns());
      }
    }
    __syncthreads();
  }
}

}  // namespace

size_t big_smem_bytes(int n) { return static_cast<size_t>(n) * (8 + 8 + 4 * 10); }

int big_max_n() { return 4096; }

#ifndef KMB_BIG_CARVE
#define KMB_BIG_CARVE 1
#endif

// Row-load width: LDG.E.64 at two columns per thread (n <= 1024: c2 8.60 ->
// 8.45 ms, n = 700 2.62 -> 2.53); scalar above, where a thread's V-wide groups
// put stride-V bank conflicts on every per-column shared array of the absorb
// and the epoch end (c4 on this engine: V = 4 171 ms, V = 2 150, V = 1 140;
// n = 3072: 36.7 / 34.9 / 33.7 ms; tools/ab_raw.py, round 2)
template <int CPT, int NT, int V = (CPT == 2 ? 2 : 1)>
static cudaError_t launch_nt(const BigArgs& a, int sm_count, size_t smem, cudaStream_t st) {
  const void* k = reinterpret_cast<const void*>(k_big<CPT, NT, V>);
  // carveout: the shared memory of the CTAs per SM this batch needs (+1 KiB
  // each, one CTA per SM for a single instance); the rest of the unified cache
  // is L1 for the cost rows
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>(227 * 1024 / (smem + 1024),
                                                              (std::max(a.batch, a.carve_batch) + sm_count - 1) / sm_count));
  const int carve = static_cast<int>(std::min<int64_t>(
      100, (want * static_cast<int64_t>(smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
  int occ = 0;
  cudaError_t e = prepare_launch(k, NT, smem, KMB_BIG_CARVE ? carve : 100, &occ);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int grid = static_cast<int>(std::min<int64_t>(a.batch, static_cast<int64_t>(occ) * sm_count));
  k_big<CPT, NT, V><<<grid, NT, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_big(const BigArgs& a, int sm_count, cudaStream_t st) {
  if (a.n < 1 || a.n > big_max_n()) return cudaErrorInvalidValue;
  const size_t smem = big_smem_bytes(a.n);
  // 512 threads per CTA: a lone SM is issue-bound, so columns per thread trade
  // per-warp overhead against per-thread work.  Measured in round 1 (c2 / c4 /
  // uniform n=2048 / geometric n=3072, ms): 1024 threads 8.88 / 158 / 16.2 /
  // 107, 512: 8.85 / 157 / 14.1 / 103, 256: 10.9 / 214 / 17.2 / 135.
  const int cpt = (a.n + 511) / 512;
  if (cpt <= 1) return launch_nt<1, 512>(a, sm_count, smem, st);
  if (cpt <= 2) return launch_nt<2, 512>(a, sm_count, smem, st);
  if (cpt <= 4) return launch_nt<4, 512>(a, sm_count, smem, st);
  return launch_nt<8, 512>(a, sm_count, smem, st);
}

}  // namespace kmb
