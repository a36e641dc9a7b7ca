// Gauss-Seidel auction on the GPU, bit-identical to
// the reference's ot::solve_auction / ot::solve_auction_scaled
// (auction.cpp:14-229): same bidder order, same double prices, same bid count.
//
// The reference's bids are sequential by construction (each bid reads the
// prices the previous one wrote), so the parallelism is inside a bid and
// across instances:
//  * one bid = one row scan: value_j = -C[i][j] - p[j], the best value (first
//    index on ties), the multiset second best (auction.cpp:44-74).  A thread
//    group scans the row coalesced, keeps (best, j, second) per thread in
//    column order, and reduces on order-preserving 64-bit keys with REDUX:
//      best = max; j = the smallest index holding it;
//      second = max over threads of (holds the winner ? its second : its best)
//    — exactly the sequential scan's (best, best_j, second), since max is
//    exact in floating point;
//  * the bidder: the reference pops the smallest row of a min-heap that
//    always holds exactly the unassigned rows (auction.cpp:22-23, 145-150),
//    i.e. the smallest unassigned row — found here with ballots over a bitmask
//    of unassigned rows (and likewise for unowned columns in try_complete);
//  * groups: one warp per instance for n <= 256 (a 32-thread CTA, up to 32
//    per SM — the whole config-3 batch is resident at once), 256 threads for
//    n <= 4096, 1024 threads above; prices, owners and the two bitmasks live
//    in shared memory (12n + n/4 bytes: n <= 18,000).
//
// Every price operation is the reference's, in its order, with explicitly
// rounded double ops: p[j] += (best - second) + eps; value = (-c) - p[j];
// eps <- max(eps / theta, eps_final); edge_ok = value >= (best - eps) - 1e-9.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <algorithm>
#include <cstdint>

#include "kmb_common.cuh"
#include "kmb_internal.h"
#include "kmb_launch.h"

#ifndef KMB_AUCTION_CLOCKS  // diagnostics: per-stage SM cycles of block 0, printed
#define KMB_AUCTION_CLOCKS 0
#endif
#if KMB_AUCTION_CLOCKS
#include <cstdio>
__device__ long long g_auc_clk[4];
#define AUC_CLK(k)                      \
  do {                                  \
    const long long t_ = clock64();     \
    g_auc_clk[k] += t_ - auc_tl;        \
    auc_tl = t_;                        \
  } while (0)
#else
#define AUC_CLK(k) (void)0
#endif

namespace kmb {
namespace {

constexpr uint32_t FULL = 0xffffffffu;

struct Bid {
  double best, second;
  int32_t j;
};

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

// Order-preserving 64-bit key of a double (no NaN here; -0.0 < +0.0, and the
// values -c - p are never +0.0), so the warp reductions run on REDUX.
__device__ __forceinline__ uint64_t okey(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? (static_cast<uint64_t>(b) | 0x8000000000000000ull) : ~static_cast<uint64_t>(b);
}
__device__ __forceinline__ double from_okey(uint64_t k) {
  return __longlong_as_double(static_cast<long long>(
      (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k) {
  const uint32_t hi = __reduce_max_sync(FULL, static_cast<uint32_t>(k >> 32));
  const uint32_t lo =
      __reduce_max_sync(FULL, static_cast<uint32_t>(k >> 32) == hi ? static_cast<uint32_t>(k) : 0u);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// (best, j, second) of a warp's 32 partial triples: best = the largest value,
// j = the smallest index holding it, second = the largest value of every
// other element — each lane offers its own second if it holds the winner,
// else its best.  Exactly the sequential scan's result (auction.cpp:47-58).
__device__ __forceinline__ void warp_bid(uint64_t& kb, uint64_t& ks, int32_t& j) {
  const uint64_t best = warp_max_u64(kb);
  const int32_t jw = static_cast<int32_t>(
      __reduce_min_sync(FULL, kb == best ? static_cast<uint32_t>(j) : 0x7FFFFFFFu));
  ks = warp_max_u64(j == jw ? ks : kb);
  kb = best;
  j = jw;
}

__device__ __forceinline__ double value_of(int32_t c, double p) {  // auction.cpp:34-36
  return __dsub_rn(-static_cast<double>(c), p);
}

template <int NT>
struct AucShared {
  uint64_t wb[NT / 32], ws[NT / 32];  // per-warp (best, second) keys
  int32_t wj[NT / 32];
  int32_t bidder;       // smallest unassigned row
  int32_t unmatched;
  int32_t flag;         // try_complete accepted
  int32_t expired;      // time budget expired
  int32_t rows[2], cols[2], nr, nc;
  unsigned long long t0, tot;
};

// Block-wide scan of row i: every thread of warp 0 ends with the block's
// (best, j, second); with NT > 32 the warps meet in shared memory (one barrier).
template <int NT>
__device__ __forceinline__ Bid scan_row(const int32_t* __restrict__ row, const double* p, int n,
                                        AucShared<NT>& S) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double best = -INFINITY, second = -INFINITY;
  int32_t j = 0x7FFFFFFF;
  constexpr int U = 8;
  for (int c0 = tid; c0 < n; c0 += NT * U) {
    int32_t cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * NT;
      cv[u] = c < n ? __ldg(row + c) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * NT;
      if (c < n) {  // columns in increasing order: first index on ties
        const double v = value_of(cv[u], p[c]);
        if (v > best) {
          second = best;
          best = v;
          j = c;
        } else if (v > second) {
          second = v;
        }
      }
    }
  }
#if KMB_AUCTION_CLOCKS
  long long auc_tl = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) { auc_tl = clock64(); g_auc_clk[3] += auc_tl; }
#endif
  uint64_t kb = okey(best), ks = okey(second);
  warp_bid(kb, ks, j);
  if constexpr (NT > 32) {
    if (lane == 0) {
      S.wb[wid] = kb;
      S.ws[wid] = ks;
      S.wj[wid] = j;
    }
    __syncthreads();
    if (wid == 0) {
      kb = lane < NT / 32 ? S.wb[lane] : 0ull;
      ks = lane < NT / 32 ? S.ws[lane] : 0ull;
      j = lane < NT / 32 ? S.wj[lane] : 0x7FFFFFFF;
      warp_bid(kb, ks, j);
    }
  }
  return Bid{from_okey(kb), from_okey(ks), j};
}

// Warp 0: the first `want` set bits of `mask` (words [0, words)) at or after
// bit `from`, in increasing order; returns how many were found.
__device__ __forceinline__ int first_bits(const uint32_t* mask, int words, int from, int want,
                                          int32_t* out) {
  const int lane = threadIdx.x & 31;
  int got = 0;
  for (int w0 = from >> 5; w0 < words && got < want; w0 += 32) {
    const int w = w0 + lane;
    uint32_t m = w < words ? mask[w] : 0u;
    if (w == (from >> 5)) m &= ~0u << (from & 31);
    uint32_t nz = __ballot_sync(FULL, m != 0u);
    while (nz && got < want) {
      const int l = __ffs(nz) - 1;
      uint32_t mw = __shfl_sync(FULL, m, l);
      while (mw && got < want) {
        const int b = __ffs(mw) - 1;
        out[got++] = ((w0 + l) << 5) + b;
        mw &= mw - 1;
      }
      nz &= nz - 1;
    }
  }
  return got;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_auction(AuctionArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ AucShared<NT> S;
  const int n = a.n;
  const int words = (n + 31) >> 5;
  double* p = reinterpret_cast<double*>(dyn);
  int32_t* owner = reinterpret_cast<int32_t*>(p + n);
  uint32_t* ua = reinterpret_cast<uint32_t*>(owner + n);  // unassigned rows
  uint32_t* uc = ua + words;                              // unowned columns
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  for (int inst = blockIdx.x; inst < a.batch; inst += gridDim.x) {
    const int32_t* Cm = a.C + static_cast<int64_t>(inst) * a.inst_stride;
    // validation (core.cpp:30-55: nonnegative costs) and max_cost
    // (core.cpp:10-13) come from k_auction_minmax
    if (tid == 0) {
      S.t0 = globaltimer_ns();
      S.tot = 0;
    }
    for (int j = tid; j < n; j += NT) p[j] = 0.0;
    __syncthreads();
    if (a.cmin[inst] < 0) {
      if (tid == 0) a.status[inst] = KMB_ENEGATIVE;
      continue;
    }
    // ---- epsilon schedule (auction.cpp:189-190, 207-216)
    double eps = a.eps0, ef = a.eps_final;
    if (a.scaled) {
      ef = a.eps_final > 0.0 ? a.eps_final : 1.0 / static_cast<double>(n + 1);
      eps = a.eps0 > 0.0 ? a.eps0 : dmax(static_cast<double>(a.cmax[inst]) / 2.0, ef);
      eps = dmax(eps, ef);
    }
    int64_t total_bids = 0;
    bool complete = false;
    for (;;) {  // one AuctionCore per epsilon round (auction.cpp:220-228)
      for (int j = tid; j < n; j += NT) owner[j] = -1;
      for (int w = tid; w < words; w += NT) {
        const uint32_t m = (w == words - 1 && (n & 31)) ? (1u << (n & 31)) - 1u : FULL;
        ua[w] = m;
        uc[w] = m;
      }
      if (tid == 0) {
        S.unmatched = n;
        S.bidder = 0;
      }
      __syncthreads();
      const int64_t budget = a.max_bids - total_bids;
      int64_t bids = 0;
      complete = true;
      // AuctionCore::run (auction.cpp:133-158)
      while (S.unmatched > 0) {
        if (S.unmatched <= 2) {
          // ---- try_complete (auction.cpp:79-120)
          if (wid == 0) {
            int32_t r[2], c[2];
            const int nr = first_bits(ua, words, 0, 2, r);
            const int nc = first_bits(uc, words, 0, 2, c);
            if (lane == 0) {
              S.nr = nr;
              S.nc = nc;
              S.rows[0] = r[0];
              S.rows[1] = nr > 1 ? r[1] : r[0];
              S.cols[0] = c[0];
              S.cols[1] = nc > 1 ? c[1] : c[0];
            }
          }
          __syncthreads();
          const int nr = S.nr;
          const int32_t r0 = S.rows[0], r1 = S.rows[1];
          const Bid b0 = scan_row<NT>(Cm + static_cast<int64_t>(r0) * a.ld, p, n, S);
          double bv1 = 0.0;
          if (nr > 1) {
            __syncthreads();
            bv1 = scan_row<NT>(Cm + static_cast<int64_t>(r1) * a.ld, p, n, S).best;
          }
          if (tid == 0) {
            const double bv0 = b0.best;
            auto C = [&](int32_t i, int32_t j) { return Cm[static_cast<int64_t>(i) * a.ld + j]; };
            auto edge_ok = [&](int32_t i, int32_t j, double bv) {
              return value_of(C(i, j), p[j]) >= __dsub_rn(__dsub_rn(bv, eps), 1e-9);
            };
            auto commit = [&](int32_t i, int32_t j) {
              owner[j] = i;
              ua[i >> 5] &= ~(1u << (i & 31));
              uc[j >> 5] &= ~(1u << (j & 31));
              --S.unmatched;
            };
            int ok = 0;
            const int32_t c0 = S.cols[0], c1 = S.cols[1];
            if (nr == 1) {
              if (edge_ok(r0, c0, bv0)) {
                commit(r0, c0);
                ok = 1;
              }
            } else {
              const int64_t straight = static_cast<int64_t>(C(r0, c0)) + C(r1, c1);
              const int64_t crossed = static_cast<int64_t>(C(r0, c1)) + C(r1, c0);
              const bool straight_first = straight <= crossed;
              for (int pass = 0; pass < 2 && !ok; ++pass) {
                const bool take_straight = (pass == 0) == straight_first;
                const int32_t j0 = take_straight ? c0 : c1;
                const int32_t j1 = take_straight ? c1 : c0;
                if (edge_ok(r0, j0, bv0) && edge_ok(r1, j1, bv1)) {
                  commit(r0, j0);
                  commit(r1, j1);
                  ok = 1;
                }
              }
            }
            S.flag = ok;
          }
          __syncthreads();
          if (S.flag) break;
        }
        if (bids >= budget) {
          complete = false;
          break;
        }
        if (a.budget_ns > 0 && (bids & 0x3FF) == 0) {  // auction.cpp:140-144
          if (tid == 0) S.expired = (globaltimer_ns() - S.t0) > static_cast<unsigned long long>(a.budget_ns);
          __syncthreads();
          const int expired = S.expired;
          __syncthreads();
          if (expired) {
            complete = false;
            break;
          }
        }
        // ---- bid (auction.cpp:44-74)
#if KMB_AUCTION_CLOCKS
        long long auc_tl = clock64();
        const bool clk = blockIdx.x == 0 && tid == 0;
        if (clk) g_auc_clk[3] -= auc_tl;  // [3] += (local scan end - bid start)
#endif
        const int32_t i = S.bidder;
        Bid b = scan_row<NT>(Cm + static_cast<int64_t>(i) * a.ld, p, n, S);
#if KMB_AUCTION_CLOCKS
        if (clk) AUC_CLK(0);  // whole scan incl. reduce
#endif
        if (wid == 0) {
          if (n == 1) b.second = b.best;
          int32_t displaced = 0;
          if (lane == 0) {
            const int32_t j = b.j;
            p[j] = __dadd_rn(p[j], __dadd_rn(__dsub_rn(b.best, b.second), eps));
            displaced = owner[j];
            owner[j] = i;
            ua[i >> 5] &= ~(1u << (i & 31));
            if (displaced >= 0)
              ua[displaced >> 5] |= 1u << (displaced & 31);
            else {
              uc[j >> 5] &= ~(1u << (j & 31));
              --S.unmatched;
            }
          }
          displaced = __shfl_sync(FULL, displaced, 0);
          __syncwarp();
          // next bidder: the displaced row if it is below i, else the first
          // unassigned row after i (every row below i is assigned)
          int32_t nx = -1;
          if (displaced >= 0 && displaced < i) {
            nx = displaced;
          } else {
            int32_t f[1] = {-1};
            if (first_bits(ua, words, i + 1, 1, f) == 0) f[0] = -1;
            nx = f[0];
          }
          if (lane == 0) S.bidder = nx;
        }
#if KMB_AUCTION_CLOCKS
        if (clk) AUC_CLK(1);  // commit + next bidder
#endif
        ++bids;
        __syncthreads();
#if KMB_AUCTION_CLOCKS
        if (clk) AUC_CLK(2);  // barrier + loop top
#endif
      }
      total_bids += bids;
      if (!a.scaled || !complete || eps <= ef) break;
      eps = dmax(__ddiv_rn(eps, a.theta), ef);  // auction.cpp:226
      __syncthreads();
    }
    // ---- outputs (finish, auction.cpp:161-179)
    __syncthreads();
#if KMB_AUCTION_CLOCKS
    if (blockIdx.x == 0 && tid == 0)
      printf("auction blk0 inst %d bids %lld: scan %lld (local part %lld) commit %lld loop %lld cycles/bid\n",
             inst, (long long)total_bids, g_auc_clk[0] / total_bids, g_auc_clk[3] / total_bids,
             g_auc_clk[1] / total_bids, g_auc_clk[2] / total_bids);
#endif
    if (a.prices)
      for (int j = tid; j < n; j += NT) a.prices[static_cast<int64_t>(inst) * n + j] = p[j];
    if (a.row_to_col) {
      for (int r = tid; r < n; r += NT) a.row_to_col[static_cast<int64_t>(inst) * n + r] = -1;
      __syncthreads();
      for (int j = tid; j < n; j += NT)
        if (owner[j] >= 0) a.row_to_col[static_cast<int64_t>(inst) * n + owner[j]] = j;
    }
    long long tot = 0;
    for (int j = tid; j < n; j += NT)
      if (owner[j] >= 0) tot += __ldg(Cm + static_cast<int64_t>(owner[j]) * a.ld + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) atomicAdd(&S.tot, static_cast<unsigned long long>(tot));
    __syncthreads();
    if (tid == 0) {
      if (a.total_cost) a.total_cost[inst] = static_cast<int64_t>(S.tot);
      if (a.bids) a.bids[inst] = total_bids;
      if (a.complete) a.complete[inst] = complete ? 1 : 0;
      if (a.eps_last) a.eps_last[inst] = eps;
      a.status[inst] = 0;
    }
    __syncthreads();
  }
}

// ---- warp engine (n <= 32 * CPL <= 256): one warp per instance, all state in
// registers — lane l holds columns l + 32q (price, owner) and word l of the
// unassigned-row and unowned-column bitmasks — so a bid is loads, a handful of
// FP64 ops and five REDUX, with no shared memory and no barrier.
template <int CPL>
struct WarpAuction {
  double p[CPL];
  int32_t own[CPL];
  uint32_t ua, uc;  // this lane's bitmask words
  int unmatched;

  __device__ __forceinline__ double price_of(int32_t j) const {  // p[j], warp-uniform
    // one shuffle per slot, then a value select (a select of p[q] would be
    // folded into a dynamically indexed load and push p[] to local memory)
    const uint32_t sel = 1u << (j >> 5);
    double r = __shfl_sync(FULL, p[0], j & 31);
#pragma unroll
    for (int q = 1; q < CPL; ++q) {
      const double t = __shfl_sync(FULL, p[q], j & 31);
      r = ((sel >> q) & 1u) ? t : r;
    }
    return r;
  }
  // (best, j, second) of row i at the current prices (auction.cpp:44-58)
  __device__ __forceinline__ void scan(const int32_t* __restrict__ row, int n, double& best,
                                      double& second, int32_t& j) const {
    const int lane = threadIdx.x & 31;
    int32_t cv[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      cv[q] = c < n ? __ldg(row + c) : 0;
    }
    double b = -INFINITY, s = -INFINITY;
    int32_t bj = 0x7FFFFFFF;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      if (c < n) {
        const double v = value_of(cv[q], p[q]);
        if (v > b) {
          s = b;
          b = v;
          bj = c;
        } else if (v > s) {
          s = v;
        }
      }
    }
    uint64_t kb = okey(b), ks = okey(s);
    warp_bid(kb, ks, bj);
    best = from_okey(kb);
    second = from_okey(ks);
    j = bj;
  }
  // edge_ok (auction.cpp:90-92) with the row's best value bv precomputed
  __device__ __forceinline__ bool edge_ok(const int32_t* Cm, int64_t ld, int32_t i, int32_t j,
                                          double bv, double eps) const {
    const double v = value_of(__ldg(Cm + static_cast<int64_t>(i) * ld + j), price_of(j));
    return v >= __dsub_rn(__dsub_rn(bv, eps), 1e-9);
  }
  __device__ __forceinline__ void commit(int32_t i, int32_t j) {
    const int lane = threadIdx.x & 31;
    const uint32_t sel = lane == (j & 31) ? 1u << (j >> 5) : 0u;
#pragma unroll
    for (int q = 0; q < CPL; ++q) own[q] = ((sel >> q) & 1u) ? i : own[q];
    if (lane == (i >> 5)) ua &= ~(1u << (i & 31));
    if (lane == (j >> 5)) uc &= ~(1u << (j & 31));
    --unmatched;
  }
};

// the first two set bits of a warp-distributed bitmask (lane l = word l)
__device__ __forceinline__ int first_two(uint32_t word, int32_t& b0, int32_t& b1) {
  uint32_t bal = __ballot_sync(FULL, word != 0u);
  if (!bal) return 0;
  const int l0 = __ffs(bal) - 1;
  uint32_t w = __shfl_sync(FULL, word, l0);
  b0 = (l0 << 5) + __ffs(w) - 1;
  w &= w - 1;
  if (w) {
    b1 = (l0 << 5) + __ffs(w) - 1;
    return 2;
  }
  bal &= bal - 1;
  if (!bal) return 1;
  const int l1 = __ffs(bal) - 1;
  b1 = (l1 << 5) + __ffs(__shfl_sync(FULL, word, l1)) - 1;
  return 2;
}

template <int CPL>
__global__ void __launch_bounds__(32, CPL <= 4 ? 28 : 16) k_auction_warp(AuctionArgs a) {
  const int lane = threadIdx.x;
  const int n = a.n;
  const int words = (n + 31) >> 5;
  const uint32_t wmask =
      lane < words ? ((lane == words - 1 && (n & 31)) ? (1u << (n & 31)) - 1u : FULL) : 0u;
  for (int inst = blockIdx.x; inst < a.batch; inst += gridDim.x) {
    const int32_t* Cm = a.C + static_cast<int64_t>(inst) * a.inst_stride;
    if (a.cmin[inst] < 0) {  // validate_instance (core.cpp:30-55)
      if (lane == 0) a.status[inst] = KMB_ENEGATIVE;
      continue;
    }
    const unsigned long long t0 = globaltimer_ns();
    WarpAuction<CPL> W;
#pragma unroll
    for (int q = 0; q < CPL; ++q) W.p[q] = 0.0;
    double eps = a.eps0, ef = a.eps_final;  // auction.cpp:189-190, 207-216
    if (a.scaled) {
      ef = a.eps_final > 0.0 ? a.eps_final : 1.0 / static_cast<double>(n + 1);
      eps = a.eps0 > 0.0 ? a.eps0 : dmax(static_cast<double>(a.cmax[inst]) / 2.0, ef);
      eps = dmax(eps, ef);
    }
    int64_t total_bids = 0;
    bool complete = false;
    for (;;) {  // auction.cpp:220-228
#pragma unroll
      for (int q = 0; q < CPL; ++q) W.own[q] = -1;
      W.ua = wmask;
      W.uc = wmask;
      W.unmatched = n;
      int32_t bidder = 0;
      int64_t bids = 0;
      const int64_t budget = a.max_bids - total_bids;
      complete = true;
      while (W.unmatched > 0) {  // AuctionCore::run (auction.cpp:133-158)
        if (W.unmatched <= 2) {  // try_complete (auction.cpp:79-120)
          int32_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
          const int nr = first_two(W.ua, r0, r1);
          first_two(W.uc, c0, c1);
          double bv0, bv1 = 0.0, sd;
          int32_t jd;
          W.scan(Cm + static_cast<int64_t>(r0) * a.ld, n, bv0, sd, jd);
          if (nr > 1) W.scan(Cm + static_cast<int64_t>(r1) * a.ld, n, bv1, sd, jd);
          bool ok = false;
          if (nr == 1) {
            if (W.edge_ok(Cm, a.ld, r0, c0, bv0, eps)) {
              W.commit(r0, c0);
              ok = true;
            }
          } else {
            const int64_t ld = a.ld;
            const int64_t straight = static_cast<int64_t>(__ldg(Cm + r0 * ld + c0)) + __ldg(Cm + r1 * ld + c1);
            const int64_t crossed = static_cast<int64_t>(__ldg(Cm + r0 * ld + c1)) + __ldg(Cm + r1 * ld + c0);
            const bool straight_first = straight <= crossed;
            for (int pass = 0; pass < 2 && !ok; ++pass) {
              const bool take_straight = (pass == 0) == straight_first;
              const int32_t j0 = take_straight ? c0 : c1;
              const int32_t j1 = take_straight ? c1 : c0;
              if (W.edge_ok(Cm, a.ld, r0, j0, bv0, eps) && W.edge_ok(Cm, a.ld, r1, j1, bv1, eps)) {
                W.commit(r0, j0);
                W.commit(r1, j1);
                ok = true;
              }
            }
          }
          if (ok) break;
        }
        if (bids >= budget) {
          complete = false;
          break;
        }
        if (a.budget_ns > 0 && (bids & 0x3FF) == 0) {  // auction.cpp:140-144
          const int expired = __shfl_sync(
              FULL, (globaltimer_ns() - t0) > static_cast<unsigned long long>(a.budget_ns) ? 1 : 0, 0);
          if (expired) {
            complete = false;
            break;
          }
        }
        // ---- bid (auction.cpp:44-74)
        const int32_t i = bidder;
        double best, second;
        int32_t j;
        W.scan(Cm + static_cast<int64_t>(i) * a.ld, n, best, second, j);
        if (n == 1) second = best;
        // the owner lane of column j raises p[j] and swaps its owner; every
        // register slot is written through a select so the arrays stay in
        // registers (a guarded p[j >> 5] store would be lowered to local memory)
        const double inc = __dadd_rn(__dsub_rn(best, second), eps);
        const uint32_t sel = lane == (j & 31) ? 1u << (j >> 5) : 0u;  // slot bit mask
        int32_t displaced = -1;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const bool hit = (sel >> q) & 1u;
          const double np = __dadd_rn(W.p[q], inc);
          displaced = hit ? W.own[q] : displaced;
          W.p[q] = hit ? np : W.p[q];
          W.own[q] = hit ? i : W.own[q];
        }
        displaced = __shfl_sync(FULL, displaced, j & 31);
        if (lane == (i >> 5)) W.ua &= ~(1u << (i & 31));
        if (displaced >= 0) {
          if (lane == (displaced >> 5)) W.ua |= 1u << (displaced & 31);
        } else {
          if (lane == (j >> 5)) W.uc &= ~(1u << (j & 31));
          --W.unmatched;
        }
        // next bidder: the smallest unassigned row (rows below i are assigned,
        // except a displaced one)
        if (displaced >= 0 && displaced < i) {
          bidder = displaced;
        } else {
          const int from = i + 1, fw = from >> 5;
          const uint32_t m = lane > fw ? W.ua : (lane == fw ? (W.ua & (~0u << (from & 31))) : 0u);
          const uint32_t bal = __ballot_sync(FULL, m != 0u);
          if (bal) {
            const int l = __ffs(bal) - 1;
            bidder = (l << 5) + __ffs(__shfl_sync(FULL, m, l)) - 1;
          } else {
            bidder = -1;
          }
        }
        ++bids;
      }
      total_bids += bids;
      if (!a.scaled || !complete || eps <= ef) break;
      eps = dmax(__ddiv_rn(eps, a.theta), ef);  // auction.cpp:226
    }
    // ---- outputs (finish, auction.cpp:161-179)
    long long tot = 0;
    if (a.row_to_col)
      for (int r = lane; r < n; r += 32) a.row_to_col[static_cast<int64_t>(inst) * n + r] = -1;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      if (c < n) {
        if (a.prices) a.prices[static_cast<int64_t>(inst) * n + c] = W.p[q];
        if (W.own[q] >= 0) {
          if (a.row_to_col) a.row_to_col[static_cast<int64_t>(inst) * n + W.own[q]] = c;
          tot += __ldg(Cm + static_cast<int64_t>(W.own[q]) * a.ld + c);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) {
      if (a.total_cost) a.total_cost[inst] = tot;
      if (a.bids) a.bids[inst] = total_bids;
      if (a.complete) a.complete[inst] = complete ? 1 : 0;
      if (a.eps_last) a.eps_last[inst] = eps;
      a.status[inst] = 0;
    }
  }
}

template <int CPL>
cudaError_t launch_warp(const AuctionArgs& a, int sm_count, cudaStream_t st) {
  auto k = k_auction_warp<CPL>;
  int per_sm = 0;
  cudaError_t e = prepare_launch(reinterpret_cast<const void*>(k), 32, 0, -1, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = static_cast<int>(std::min<int64_t>(a.batch, static_cast<int64_t>(per_sm) * sm_count));
  k<<<grid, 32, 0, st>>>(a);
  return cudaGetLastError();
}

// Per-instance min / max cost (atomics into cmin / cmax, preset to INT64_MAX / 0):
// one grid-wide pass, so a single large instance is read at full bandwidth.
__global__ void __launch_bounds__(256) k_auction_minmax(const int32_t* __restrict__ C, int32_t batch,
                                                        int32_t n, int64_t ld, int64_t inst_stride,
                                                        long long* cmin, long long* cmax) {
  const int rows_per_block = 8;
  const int xb = (n + rows_per_block - 1) / rows_per_block;
  for (int64_t t = blockIdx.x; t < static_cast<int64_t>(batch) * xb; t += gridDim.x) {
    const int inst = static_cast<int>(t / xb);
    const int r0 = static_cast<int>(t % xb) * rows_per_block;
    const int32_t* Cm = C + static_cast<int64_t>(inst) * inst_stride;
    int32_t lo = INT_MAX, hi = 0;
    for (int r = r0; r < min(n, r0 + rows_per_block); ++r)
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const int32_t x = __ldg(Cm + static_cast<int64_t>(r) * ld + c);
        lo = min(lo, x);
        hi = max(hi, x);
      }
    lo = __reduce_min_sync(FULL, lo);
    hi = __reduce_max_sync(FULL, hi);
    if ((threadIdx.x & 31) == 0) {
      if (lo != INT_MAX) atomicMin(cmin + inst, static_cast<long long>(lo));
      if (hi > 0) atomicMax(cmax + inst, static_cast<long long>(hi));
    }
  }
}

template <int NT>
cudaError_t launch_nt(const AuctionArgs& a, int sm_count, size_t smem, cudaStream_t st) {
  auto k = k_auction<NT>;
  int per_sm = 0;
  cudaError_t e = prepare_launch(reinterpret_cast<const void*>(k), NT, smem, -1, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = static_cast<int>(std::min<int64_t>(a.batch, static_cast<int64_t>(per_sm) * sm_count));
  k<<<grid, NT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t auction_smem_bytes(int n) {
  const size_t words = (static_cast<size_t>(n) + 31) / 32;
  return static_cast<size_t>(n) * 12 + words * 8;
}

int auction_max_n() { return 18000; }

cudaError_t launch_auction(const AuctionArgs& a, int sm_count, cudaStream_t st) {
  const size_t smem = auction_smem_bytes(a.n);
  cudaError_t e = cudaMemsetAsync(a.cmin, 0x7f, sizeof(long long) * a.batch, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.cmax, 0, sizeof(long long) * a.batch, st);
  if (e != cudaSuccess) return e;
  const int64_t tiles = static_cast<int64_t>(a.batch) * ((a.n + 7) / 8);
  k_auction_minmax<<<static_cast<int>(std::min<int64_t>(tiles, 16LL * sm_count)), 256, 0, st>>>(
      a.C, a.batch, a.n, a.ld, a.inst_stride, a.cmin, a.cmax);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (a.n <= 32) return launch_warp<1>(a, sm_count, st);
  if (a.n <= 64) return launch_warp<2>(a, sm_count, st);
  if (a.n <= 128) return launch_warp<4>(a, sm_count, st);
  if (a.n <= 256) return launch_warp<8>(a, sm_count, st);
  if (a.n <= 4096) return launch_nt<256>(a, sm_count, smem, st);
  return launch_nt<1024>(a, sm_count, smem, st);
}

}  // namespace kmb
