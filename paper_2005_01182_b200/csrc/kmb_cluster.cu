// Replicated cluster engine (KMB_OPT_ENGINE 11): one thread-block cluster of
// G <= 16 CTAs solves one instance; CTA b owns a slab of the columns with its
// per-column keys, v and Dc in registers (the single-CTA engine's layout,
// kmb_big.cu, spread over G SMs) and holds a REPLICA of the row side — the
// reached-row lists, u, w, roots and the matching — in its own shared memory.
//
// Why: the cluster engine (engine 5, kmb_solver.cu) keeps that state in ONE
// place (global or distributed shared memory), so each round of c4 chains
// several 200-cycle DSMEM hops (list -> u -> cost row; parent -> root) and costs
// ~3.9 us.  Here every read of row-side state is a local shared-memory read and
// the cost row comes from L2; what a round publishes — its min-slack partial
// and the rows it appends — is written into every replica with DSMEM stores,
// and two hardware cluster barriers (barrier.cluster, release/acquire) per round
// order it.  Tree claims, the append counters and the found-column list live in
// CTA 0 ("home", DSMEM atomics, 32-bit claim words: (epoch stamp, column)).
//
// The search is the engines' (hungarian.cpp:175-217 with lazy
// duals; argmin-parent forest augmentation; incremental epochs; dirty-column
// epoch starts): every replica applies the same updates, so all replicas hold
// the same row SETS (list order may differ per CTA; the packed (value, row)
// keys make the result independent of it) and the same values.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <type_traits>

#include "kmb_common.cuh"
#include "kmb_internal.h"
#include "kmb_launch.h"

#ifndef KMB_CL_DEBUG  // bounds checks with printf (debug builds only)
#define KMB_CL_DEBUG 0
#endif
#ifndef KMB_CL_CLOCKS  // diagnostics: CTA 0 thread 0's cycles per stage, printed
#define KMB_CL_CLOCKS 0
#endif
#if KMB_CL_CLOCKS
#include <cstdio>
#define CLK(k)                      \
  do {                              \
    const long long t_ = clock64(); \
    clk[k] += t_ - clk_last;        \
    clk_last = t_;                  \
  } while (0)
#else
#define CLK(k) (void)0
#endif
#if KMB_CL_DEBUG
#include <cstdio>
#define CLCHK(cond, what, x)                                                                   \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("CLCHK %s b=%d t=%d x=%d round=%d epoch=%d\n", what, b, t, (int)(x), rounds, epochs); \
      asm volatile("exit;");                                                                   \
    }                                                                                          \
  } while (0)
#else
#define CLCHK(cond, what, x) (void)0
#endif

namespace kmb {
namespace {

namespace cg = cooperative_groups;
constexpr uint32_t FULL = 0xffffffffu;
constexpr int kMaxG = 16;

// packed key ((c - w + 2^30) << 32) | row, as the single-CTA engine's
struct CK {
  __device__ static uint32_t tag(int32_t w) { return static_cast<uint32_t>(static_cast<int32_t>(KMB_BIAS) - w); }
  __device__ static uint64_t make(int32_t c, uint32_t tag, int32_t row) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(c) + tag) << 32) | static_cast<uint32_t>(row);
  }
  __device__ static int32_t val(uint64_t k) { return static_cast<int32_t>(static_cast<int64_t>(k >> 32) - KMB_BIAS); }
  __device__ static int32_t row(uint64_t k) { return static_cast<int32_t>(static_cast<uint32_t>(k)); }
};

// home tree claims: (epoch stamp, column) in 32 bits, smaller wins (stamps
// decrease with the epoch: stale claims never block); columns < 2^14
__device__ __forceinline__ uint32_t cclaim(int ep, int col) {
  return ((0x3FFFEu - static_cast<uint32_t>(ep)) << 14) | static_cast<uint32_t>(col);
}
__device__ __forceinline__ bool cclaimed(uint32_t c, int ep) {
  return (c >> 14) == 0x3FFFEu - static_cast<uint32_t>(ep);
}

struct ClShared {
  long long part[2][kMaxG];   // every CTA's min-slack partial (broadcast; by round parity)
  int32_t red[32];            // per-warp partial minima
  int32_t cnt[3], fcnt[3];    // home: row / free-column appends of a BFS round (round % 3)
  int32_t cnt2[2], fcnt2[2];  // home: ... of a dual-step absorb (by dual-step parity)
  int32_t won, stop;          // home: trees augmented this epoch; time budget expired
  int32_t ns, nd;             // local: survivors, dirty columns
  int32_t lo_all, hi_all;     // validation of this CTA's rows
  unsigned long long tot;     // home: objective
};

template <int CPT, int kT>
__global__ void __launch_bounds__(kT, 1) k_cluster(BigArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ ClShared sm;
  cg::cluster_group cl = cg::this_cluster();
  const int G = static_cast<int>(cl.num_blocks());
  const int b = static_cast<int>(cl.block_rank());
  const int n = a.n;
  const int Wc = CPT * kT;                 // columns per CTA
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int c0 = b * Wc;                   // this CTA's first column
  // replicated row side
  int2* rows = reinterpret_cast<int2*>(dyn);
  int2* spare = rows + n;  // also the dirty-column keys in the round after an epoch end
  int32_t* u = reinterpret_cast<int32_t*>(spare + n);
  int32_t* w = u + n;
  int32_t* root_row = w + n;
  int32_t* match_row = root_row + n;
  uint32_t* claim = reinterpret_cast<uint32_t*>(match_row + n);  // home in CTA 0, an epoch-end copy elsewhere
  int32_t* found = reinterpret_cast<int32_t*>(claim + n);        // used in CTA 0
  // this CTA's columns
  int32_t* tpar = found + n;
  int32_t* mcol = tpar + Wc;
  int32_t* dlist = mcol + Wc;
  int32_t* dpos = dlist + Wc;
  // home (CTA 0) and peer views
  uint32_t* h_claim = cl.map_shared_rank(claim, 0u);
  int32_t* h_found = cl.map_shared_rank(found, 0u);
  ClShared* h_sm = cl.map_shared_rank(&sm, 0u);
  auto colof = [&](int q) { return c0 + t + q * kT; };
  auto owner = [&](int col) { return col / Wc; };

  const int nclusters = static_cast<int>(gridDim.x) / G;
  const int cid = static_cast<int>(blockIdx.x) / G;
  for (int inst = cid; inst < a.batch; inst += nclusters) {
    const int32_t* Cm = a.C + static_cast<int64_t>(inst) * a.inst_stride;
    const int ld32 = static_cast<int>(a.ld);
    const unsigned long long t0 = globaltimer_ns();
    if (t == 0) {
      sm.lo_all = INT_MAX;
      sm.hi_all = 0;
      for (int k = 0; k < 3; ++k) sm.cnt[k] = sm.fcnt[k] = 0;
      sm.cnt2[0] = sm.cnt2[1] = sm.fcnt2[0] = sm.fcnt2[1] = 0;
      sm.won = 0;
      sm.stop = 0;
      sm.ns = 0;
      sm.nd = 0;
      sm.tot = 0;
    }
    for (int k = t; k < n; k += kT) {
      match_row[k] = -1;
      root_row[k] = k;
      claim[k] = 0xFFFFFFFFu;
    }
    for (int k = t; k < Wc; k += kT) mcol[k] = -1;
    cl.sync();  // home counters initialised before any CTA's atomics reach them
    // validation (core.cpp:144-145 + device range) and the row reductions
    // (hungarian.cpp:323-327): CTA b takes rows i = b (mod G), one warp per
    // row, and stores u0 = w0 into every replica
    {
      int32_t lo_all = INT_MAX, hi_all = 0;
      for (int i = b + G * wid; i < n; i += G * (kT / 32)) {
        int32_t lo = INT_MAX, hi = 0;
        for (int k = lane; k < n; k += 32) {
          const int32_t x = __ldg(Cm + static_cast<int64_t>(i) * a.ld + k);
          lo = min(lo, x);
          hi = max(hi, x);
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        lo_all = min(lo_all, lo);
        hi_all = max(hi_all, hi);
        const int32_t u0 = a.seed == 1 ? lo : 0;
        if (lane < G) {  // lane r writes replica r
          cl.map_shared_rank(u, static_cast<unsigned>(lane))[i] = u0;
          cl.map_shared_rank(w, static_cast<unsigned>(lane))[i] = u0;
        }
      }
      if (lane == 0) {
        atomicMin(&h_sm->lo_all, lo_all);
        atomicMax(&h_sm->hi_all, hi_all);
      }
    }
    cl.sync();  // u0 everywhere, home validation complete
    const int status0 = h_sm->lo_all < 0 ? 2 : (h_sm->hi_all >= (1 << 29) ? 3 : 0);
    if (status0) {
      if (b == 0 && t == 0) {
        a.status[inst] = status0;
        a.total_cost[inst] = 0;
        if (a.converged) a.converged[inst] = 0;
      }
      if (b == 0 && a.stats && t < KMB_ISTATS) a.stats[KMB_ISTATS * static_cast<int64_t>(inst) + t] = 0;
      for (int k = b * kT + t; k < n; k += G * kT) a.row_to_col[static_cast<int64_t>(inst) * n + k] = -1;
      cl.sync();  // nobody reinitialises home state while a peer still reads it
      continue;
    }
    for (int k = t; k < n; k += kT) rows[k] = make_int2(k, static_cast<int32_t>(CK::tag(w[k])));

    uint64_t key[CPT];
    int32_t v[CPT], dc[CPT];
    uint32_t rch = 0;  // bit q: column colof(q) reached (columns past n count as reached)
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      key[q] = ~0ull;
      v[q] = 0;
      dc[q] = 0;
      if (colof(q) >= n || t + q * kT >= Wc) rch |= 1u << q;
    }
    int nrows = n, head = 0, nfree = n;
    int32_t D = 0;
    int epochs = 0, dual_steps = 0, rounds = 0;
    int64_t rows_scanned = 0;
    bool dirty_round = false, stopped = false;
    int status = 0;
    __syncthreads();

    // relax rows[from, to) over this thread's columns; exact-size batches
    // (a batch past `to` repeats its last row: the fold is idempotent, and a
    // short relax then costs one L2 latency instead of one per partial batch)
    auto relax_k = [&](int r, int to, auto kc) {
      constexpr int K = decltype(kc)::value;
      int2 e[K];
      int32_t c[K][CPT];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        e[k] = rows[min(r + k, to - 1)];
        CLCHK(e[k].x >= 0 && e[k].x < n, "relax row", e[k].x);
      }
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int col = colof(q);
          c[k][q] = col < n ? __ldg(Cm + (e[k].x * ld32 + col)) : 0;
        }
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const uint64_t kk = CK::make(c[k][q], static_cast<uint32_t>(e[k].y), e[k].x);
          key[q] = kk < key[q] ? kk : key[q];
        }
    };
    auto relax_full = [&](int from, int to) {
      constexpr int RB = CPT >= 4 ? 2 : (CPT == 2 ? 4 : 6);
      for (int r = from; r < to; r += RB) relax_k(r, to, std::integral_constant<int, RB>{});
    };

#if KMB_CL_CLOCKS
    long long clk[8] = {0, 0, 0, 0, 0, 0, 0, 0}, clk_last = clock64();
#endif
    while (nfree > 0) {
      CLK(7);
      if (rounds > 4 * n * n + 64) {  // a valid search ends in n epochs of <= 2n + 1 rounds
        status = -2;
        break;
      }
      ++rounds;
      // ---- relax (hungarian.cpp:164-172) ----
      if (!dirty_round) {
        relax_full(head, nrows);
        rows_scanned += nrows - head;
      } else {
        // epoch start: only this CTA's dirty (reset) columns change; threads
        // split the survivor rows of each, then the owners take the minima
        dirty_round = false;
        const int nd = sm.nd;
        CLCHK(nd >= 0 && nd <= n && nd <= Wc, "nd", nd);
        uint64_t* dkey = reinterpret_cast<uint64_t*>(spare);  // the old list is dead
        for (int k = t; k < nd; k += kT) dkey[k] = ~0ull;
        __syncthreads();
        if (nd > 0) {
          const int groups = max(1, kT / nd);
          for (int item = t; item < nd * groups; item += kT) {
            const int k = item % nd, g = item / nd;
            const int col = c0 + dlist[k];
            CLCHK(col >= c0 && col < n, "dlist col", col);
            uint64_t best = ~0ull;
            constexpr int GB = 8;
            for (int r = g; r < nrows; r += groups * GB) {
              int2 e[GB];
              int32_t c[GB];
#pragma unroll
              for (int q = 0; q < GB; ++q) {
                const int rr = r + q * groups;
                e[q] = rr < nrows ? rows[rr] : make_int2(-1, 0);
              }
#pragma unroll
              for (int q = 0; q < GB; ++q) c[q] = e[q].x >= 0 ? __ldcg(Cm + e[q].x * a.ld + col) : 0;
#pragma unroll
              for (int q = 0; q < GB; ++q) {
                const uint64_t kk = e[q].x >= 0 ? CK::make(c[q], static_cast<uint32_t>(e[q].y), e[q].x) : ~0ull;
                best = kk < best ? kk : best;
              }
            }
            atomicMin(reinterpret_cast<unsigned long long*>(dkey + k), static_cast<unsigned long long>(best));
          }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int lc = t + q * kT;
          if (!((rch >> q) & 1) && key[q] == ~0ull) {
            CLCHK(dpos[lc] >= 0 && dpos[lc] < nd, "dpos", dpos[lc]);
            key[q] = dkey[dpos[lc]];
          }
        }
        if (t == 0) sm.nd = 0;
      }
      head = nrows;
      CLK(0);
      if (epochs == 0 && rounds == 1 && a.seed == 1) {  // column reduction, :328-333
#pragma unroll
        for (int q = 0; q < CPT; ++q)
          if (!((rch >> q) & 1)) v[q] = CK::val(key[q]);
      }
      // ---- absorb zero-slack columns (hungarian.cpp:186-199) at the current D
      // first — a column tight at D is absorbed in any case — and publish the
      // minimum over the columns that stay unreached: a BFS round needs ONE
      // cluster barrier, a dual-step round (hungarian.cpp:201-215) two.  The
      // appends of a warp are counted with one home atomic and broadcast to the
      // replicas by the warp's lanes (lane r stores into CTA r).
      int32_t s[CPT];
#pragma unroll
      for (int q = 0; q < CPT; ++q) s[q] = CK::val(key[q]) - v[q];
      auto absorb = [&](int32_t Dn, int* hcnt, int* hfcnt) {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const bool tight = !((rch >> q) & 1) && s[q] == Dn;
          const int lc = t + q * kT, col = c0 + lc;
          int32_t i2 = -1, root = 0, w2 = 0;
          if (tight) {
            rch |= 1u << q;
            dc[q] = Dn;
            const int32_t pr = CK::row(key[q]);
            CLCHK(pr >= 0 && pr < n, "absorb parent", pr);
            tpar[lc] = pr;
            root = root_row[pr];
            i2 = mcol[lc];
            CLCHK(i2 >= -1 && i2 < n, "absorb match", i2);
            if (i2 < 0) atomicMin(h_claim + root, cclaim(epochs, col));
            else w2 = u[i2] - Dn;
          }
          const unsigned rowmask = __ballot_sync(FULL, tight && i2 >= 0);
          const unsigned fmask = __ballot_sync(FULL, tight && i2 < 0);
          if (rowmask) {
            int base = 0;
            if (lane == 0) base = atomicAdd(hcnt, __popc(rowmask));
            base = __shfl_sync(FULL, base, 0);
            const int pos = nrows + base + __popc(rowmask & ((1u << lane) - 1));
            unsigned mk = rowmask;
            while (mk) {
              const int src = __ffs(mk) - 1;
              mk &= mk - 1;
              const int p = __shfl_sync(FULL, pos, src);
              const int32_t ii = __shfl_sync(FULL, i2, src);
              const int32_t ww = __shfl_sync(FULL, w2, src);
              const int32_t rt = __shfl_sync(FULL, root, src);
              CLCHK(p < n, "append pos", p);
              if (lane < G) {
                const unsigned r = static_cast<unsigned>(lane);
                cl.map_shared_rank(rows, r)[p] = make_int2(ii, static_cast<int32_t>(CK::tag(ww)));
                cl.map_shared_rank(w, r)[ii] = ww;
                cl.map_shared_rank(root_row, r)[ii] = rt;
              }
            }
          }
          if (fmask) {
            int base = 0;
            if (lane == 0) base = atomicAdd(hfcnt, __popc(fmask));
            base = __shfl_sync(FULL, base, 0);
            if (tight && i2 < 0) h_found[base + __popc(fmask & ((1u << lane) - 1))] = col;
          }
        }
      };
      const int kb = rounds % 3;  // this round's counter slot (home, triple-buffered)
      absorb(D, &h_sm->cnt[kb], &h_sm->fcnt[kb]);
      CLK(1);
      int32_t lm = INT_MAX;
#pragma unroll
      for (int q = 0; q < CPT; ++q)
        if (!((rch >> q) & 1)) lm = min(lm, s[q]);
      lm = __reduce_min_sync(FULL, lm);
      if (lane == 0) sm.red[wid] = lm;
      __syncthreads();
      if (wid == 0) {
        const int32_t x = __reduce_min_sync(FULL, lane < kT / 32 ? sm.red[lane] : INT_MAX);
        if (lane < G) cl.map_shared_rank(sm.part[kb & 1], static_cast<unsigned>(lane))[b] = x;
      }
      CLK(2);
      cl.sync();  // ------------------------------------------------------- C1
      CLK(3);
      // slot kb - 1 was last read after the previous C1 (everyone is past it);
      // it is written again two rounds on, after the next C1
      if (b == 0 && t == 0) {
        const int kc = kb == 0 ? 2 : kb - 1;
        sm.cnt[kc] = 0;
        sm.fcnt[kc] = 0;
      }
      int added = h_sm->cnt[kb], nfound = h_sm->fcnt[kb];
      CLK(4);
      if (added == 0 && nfound == 0) {
        // nothing tight anywhere: dual step D = min slack' over the cluster
        int32_t m = INT_MAX;
        for (int r = 0; r < G; ++r) m = min(m, static_cast<int32_t>(sm.part[kb & 1][r]));
        if (m == INT_MAX) {  // no unreached column: cannot happen on valid input
          status = -2;
          break;
        }
        D = m;  // applied lazily
        ++dual_steps;
        const int db = dual_steps & 1;
        absorb(D, &h_sm->cnt2[db], &h_sm->fcnt2[db]);
        cl.sync();  // ----------------------------------------------------- C2
        added = h_sm->cnt2[db];
        nfound = h_sm->fcnt2[db];
        // the other parity was last read after the previous dual step's C2
        if (b == 0 && t == 0) {
          sm.cnt2[db ^ 1] = 0;
          sm.fcnt2[db ^ 1] = 0;
        }
        CLK(5);
      }
      nrows += added;
      if (nfound == 0) continue;

      // ---- epoch end: augment and dissolve the trees that reached a free column.
      // The rows appended this round are relaxed over all columns first (the
      // dirty-column epoch start relies on every survivor being in the keys).
      relax_full(head, nrows);
      rows_scanned += nrows - head;
      // the epoch's claims, read n times below: one bulk copy from home (16-byte
      // DSMEM loads) instead of a 200-cycle DSMEM read per row and column
      if (b != 0) {
        const int4* src = reinterpret_cast<const int4*>(h_claim);
        int4* dst = reinterpret_cast<int4*>(claim);
        for (int k = t; k < (n >> 2); k += kT) dst[k] = src[k];
        for (int k = (n & ~3) + t; k < n; k += kT) claim[k] = h_claim[k];
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int lc = t + q * kT;
        if (colof(q) >= n || lc >= Wc) continue;
        if ((rch >> q) & 1) {
          CLCHK(tpar[lc] >= 0 && tpar[lc] < n, "reached parent", tpar[lc]);
          if (cclaimed(claim[root_row[tpar[lc]]], epochs)) {
            v[q] -= D - dc[q];
            rch &= ~(1u << q);
            key[q] = ~0ull;
          }
        } else if (key[q] != ~0ull && cclaimed(claim[root_row[CK::row(key[q])]], epochs)) {
          key[q] = ~0ull;
        }
        if (!((rch >> q) & 1) && key[q] == ~0ull) {  // dirty: recomputed next round
          const int k = atomicAdd(&sm.nd, 1);
          CLCHK(k >= 0 && k < Wc, "dirty pos", k);
          dlist[k] = lc;
          dpos[lc] = k;
        }
      }
      CLCHK(nrows <= n, "nrows", nrows);
      for (int r = t; r < nrows; r += kT) {
        const int2 e = rows[r];
        CLCHK(e.x >= 0 && e.x < n, "list row", e.x);
        if (cclaimed(claim[root_row[e.x]], epochs)) u[e.x] = w[e.x] + D;
        else {
          const int sp = atomicAdd(&sm.ns, 1);
          CLCHK(sp >= 0 && sp < n, "survivor pos", sp);
          spare[sp] = e;
        }
      }
      // flip one path per claimed tree (its smallest free column); the found
      // columns are split over the cluster's threads
      int won = 0;
      for (int f = b * kT + t; f < nfound; f += G * kT) {
        int32_t j = h_found[f];
        CLCHK(j >= 0 && j < n, "found col", j);
        int32_t i = cl.map_shared_rank(tpar, static_cast<unsigned>(owner(j)))[j % Wc];
        CLCHK(i >= 0 && i < n, "found parent", i);
        if (claim[root_row[i]] != cclaim(epochs, j)) continue;
        ++won;
        for (;;) {
          CLCHK(j >= 0 && j < n, "path col", j);
          i = cl.map_shared_rank(tpar, static_cast<unsigned>(owner(j)))[j % Wc];
          CLCHK(i >= 0 && i < n, "path row", i);
          const int32_t nx = match_row[i];
          CLCHK(nx >= -1 && nx < n, "path next", nx);
          for (int r = 0; r < G; ++r) cl.map_shared_rank(match_row, static_cast<unsigned>(r))[i] = j;
          cl.map_shared_rank(mcol, static_cast<unsigned>(owner(j)))[j % Wc] = i;
          if (nx < 0) break;
          j = nx;
        }
      }
      won = __reduce_add_sync(FULL, won);
      if (lane == 0 && won) atomicAdd(&h_sm->won, won);
      if (b == 0 && t == 0 && a.deadline_ns > 0 &&
          globaltimer_ns() - t0 > static_cast<unsigned long long>(a.deadline_ns))
        sm.stop = 1;
      cl.sync();  // ------------------------------------------------------- C3
      nfree -= h_sm->won;
      const int stop = h_sm->stop;
      nrows = sm.ns;
      int2* tmp = rows;
      rows = spare;
      spare = tmp;
      head = nrows;  // survivors are folded in; the dirty columns are recomputed
      dirty_round = true;
      ++epochs;
      cl.sync();  // everyone read won / ns before they are reset
      if (t == 0) {
        sm.ns = 0;
        if (b == 0) sm.won = 0;
      }
      __syncthreads();
      CLK(6);
      if (stop && nfree > 0) {
        stopped = true;
        break;
      }
    }
#if KMB_CL_CLOCKS
    if (b == 0 && t == 0)
      printf("k_cluster n %d G %d rounds %d epochs %d dual %d: cycles/round relax %lld absorb %lld reduce %lld C1 %lld counters %lld dual %lld epoch %lld loop %lld\n",
             n, G, rounds, epochs, dual_steps, clk[0] / rounds, clk[1] / rounds, clk[2] / rounds, clk[3] / rounds,
             clk[4] / rounds, clk[5] / rounds, clk[6] / rounds, clk[7] / rounds);
#endif
    // a failing CTA broke out alone only where every CTA takes the same branch
    // (the cluster-wide m, the round cap), so the cluster stays in step
    if (stopped) {  // time budget: write back the surviving trees' lazy duals
      for (int r = t; r < nrows; r += kT) {
        const int2 e = rows[r];
        u[e.x] = w[e.x] + D;
      }
#pragma unroll
      for (int q = 0; q < CPT; ++q)
        if (((rch >> q) & 1) && colof(q) < n && t + q * kT < Wc) v[q] -= D - dc[q];
    }
    // ---- outputs: u and the matching from replica 0, v and the objective per slab
    long long tot = 0;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int lc = t + q * kT, col = colof(q);
      if (col >= n || lc >= Wc) continue;
      a.v[static_cast<int64_t>(inst) * n + col] = v[q];
      const int32_t i = mcol[lc];
      if (i >= 0) tot += __ldg(Cm + static_cast<int64_t>(i) * a.ld + col);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0 && tot) atomicAdd(&h_sm->tot, static_cast<unsigned long long>(tot));
    if (b == 0)
      for (int k = t; k < n; k += kT) {
        a.row_to_col[static_cast<int64_t>(inst) * n + k] = match_row[k];
        a.u[static_cast<int64_t>(inst) * n + k] = u[k];
      }
    cl.sync();  // the objective is summed; nobody starts the next instance early
    if (b == 0 && t == 0) {
      a.total_cost[inst] = static_cast<int64_t>(sm.tot);
      a.status[inst] = (stopped && status == 0) ? 4 : status;
      if (a.converged) a.converged[inst] = (!stopped && status == 0) ? 1 : 0;
      if (a.stats) {
        int64_t* o = a.stats + KMB_ISTATS * static_cast<int64_t>(inst);
        o[0] = epochs;
        o[1] = dual_steps;
        o[2] = rows_scanned;
        o[3] = rounds;
        o[4] = static_cast<int64_t>(globaltimer_ns() - t0);
        o[5] = o[6] = o[7] = o[8] = 0;
        o[9] = static_cast<int64_t>(t0);
        o[10] = static_cast<int64_t>(globaltimer_ns());
      }
    }
    cl.sync();
  }
}

constexpr int kClT = 256;

template <int CPT>
cudaError_t launch_cpt(const BigArgs& a, int G, int clusters, size_t smem, cudaStream_t st) {
  auto kern = k_cluster<CPT, kClT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G * clusters);
  cfg.blockDim = dim3(kClT);
  cfg.dynamicSmemBytes = smem;
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

}  // namespace

// columns per thread of the instantiation that serves n over G CTAs (1, 2 or 4)
static int cluster_cpt(int n, int G) {
  const int cpt = ((n + G - 1) / G + kClT - 1) / kClT;
  return cpt <= 1 ? 1 : (cpt <= 2 ? 2 : 4);
}

// shared memory of one CTA: the replicated row side (40 B per row) and this
// CTA's column arrays (16 B per column of the instantiation's slab width)
size_t cluster_smem_bytes(int n, int G) {
  const int Wc = cluster_cpt(n, G) * kClT;
  return static_cast<size_t>(n) * 40 + static_cast<size_t>(Wc) * 16;
}

int cluster_max_n() { return 5120; }

cudaError_t launch_cluster(const BigArgs& a, int G, int sm_count, cudaStream_t st) {
  if (a.n < 1 || a.n > cluster_max_n() || G < 1 || G > kMaxG) return cudaErrorInvalidValue;
  // at most 4 columns per thread: widen the cluster for large n
  G = std::min(kMaxG, std::max(G, (a.n + 4 * kClT - 1) / (4 * kClT)));
  const size_t smem = cluster_smem_bytes(a.n, G);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const int clusters = std::max(1, std::min(a.batch, sm_count / G));
  switch (cluster_cpt(a.n, G)) {
    case 1: return launch_cpt<1>(a, G, clusters, smem, st);
    case 2: return launch_cpt<2>(a, G, clusters, smem, st);
    default: return launch_cpt<4>(a, G, clusters, smem, st);
  }
}

}  // namespace kmb
