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

#include <cstdint>

#include "kmb_common.cuh"
#include "kmb_internal.h"

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

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// claim word for n <= 256: smaller is better; stamp decreases with the phase
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

template <int CPL, bool SMEM_C>
__device__ __forceinline__ RowVec<CPL> load_row(const int32_t* base) {
  RowVec<CPL> r;
  if constexpr (CPL == 4) {
    int4 t;
    if constexpr (SMEM_C) t = *reinterpret_cast<const int4*>(base);
    else t = __ldg(reinterpret_cast<const int4*>(base));
    r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
  } else if constexpr (CPL == 8) {
    int4 t0, t1;
    if constexpr (SMEM_C) {
      t0 = reinterpret_cast<const int4*>(base)[0];
      t1 = reinterpret_cast<const int4*>(base)[1];
    } else {
      t0 = __ldg(reinterpret_cast<const int4*>(base));
      t1 = __ldg(reinterpret_cast<const int4*>(base) + 1);
    }
    r.x[0] = t0.x; r.x[1] = t0.y; r.x[2] = t0.z; r.x[3] = t0.w;
    r.x[4] = t1.x; r.x[5] = t1.y; r.x[6] = t1.z; r.x[7] = t1.w;
  } else if constexpr (CPL == 2) {
    int2 t;
    if constexpr (SMEM_C) t = *reinterpret_cast<const int2*>(base);
    else t = __ldg(reinterpret_cast<const int2*>(base));
    r.x[0] = t.x; r.x[1] = t.y;
  } else {
    r.x[0] = SMEM_C ? *base : __ldg(base);
  }
  return r;
}

}  // namespace

// Per-warp shared state (n <= 256): u, w, root_row, match_row, match_col,
// tree_par, claim, found, list[2]  -> 10 * n int32.
__host__ __device__ constexpr int warp_state_words(int n) { return 10 * n; }

template <int CPL, bool SMEM_C>
__global__ void __launch_bounds__(128) k_warp_batch(WarpArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;  // warp in block
  const int wpb = blockDim.x >> 5;
  const int n = a.n, np = a.pitch;
  constexpr uint32_t FULL = 0xffffffffu;

  // carve this warp's slice
  const size_t cbytes = SMEM_C ? static_cast<size_t>(n) * np * 4 : 0;
  const size_t wbytes = cbytes + static_cast<size_t>(warp_state_words(n)) * 4 + 16;
  unsigned char* base = dyn + wib * ((wbytes + 15) & ~static_cast<size_t>(15));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base);
  int32_t* Cs = reinterpret_cast<int32_t*>(base + 16);
  int32_t* st = reinterpret_cast<int32_t*>(base + 16 + cbytes);
  int32_t* u = st;
  int32_t* w = u + n;
  int32_t* root_row = w + n;
  int32_t* match_row = root_row + n;
  int32_t* match_col = match_row + n;
  int32_t* tree_par = match_col + n;
  uint32_t* claim = reinterpret_cast<uint32_t*>(tree_par + n);
  int32_t* found = reinterpret_cast<int32_t*>(claim + n);
  int32_t* lists = found + n;

  if (SMEM_C && lane == 0) mbar_init1(bar);
  __syncwarp();
  uint32_t parity = 0;
  const int c0 = CPL * lane;  // first owned column

  for (int inst = blockIdx.x * wpb + wib; inst < a.batch; inst += gridDim.x * wpb) {
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
      match_row[k] = -1;
      match_col[k] = -1;
      claim[k] = 0xFFFFFFFFu;
      root_row[k] = k;
      lists[k] = k;
    }
    if constexpr (SMEM_C) {
      mbar_wait_parity(bar, parity);
      parity ^= 1;
    }
    __syncwarp();
    // validation (core.cpp:144-145 + device range) and row reductions
    // (hungarian.cpp:323-327): the warp walks the rows, lanes across columns
    int32_t lo_all = 0x7fffffff, hi_all = 0;
    for (int i = 0; i < n; ++i) {
      const RowVec<CPL> cv = load_row<CPL, SMEM_C>(Cm + static_cast<int64_t>(i) * np + c0);
      int32_t lo = 0x7fffffff, hi = 0;
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (c0 + q < n) {
          lo = min(lo, cv.x[q]);
          hi = max(hi, cv.x[q]);
        }
      lo = __reduce_min_sync(FULL, lo);
      lo_all = min(lo_all, lo);
      hi_all = max(hi_all, hi);
      if (lane == (i & 31)) {
        const int32_t u0 = a.seed == 1 ? lo : 0;
        u[i] = u0;
        w[i] = u0;
      }
    }
    hi_all = __reduce_max_sync(FULL, hi_all);
    const int32_t bad = lo_all < 0 ? 2 : (hi_all >= (1 << 29) ? 3 : 0);
    if (bad) {
      for (int k = lane; k < n; k += 32) a.row_to_col[static_cast<int64_t>(inst) * n + k] = -1;
      if (lane == 0) {
        a.status[inst] = bad;
        a.total_cost[inst] = 0;
      }
      __syncwarp();
      continue;
    }
    __syncwarp();

    uint64_t key[CPL];
    int32_t v[CPL], dc[CPL];
    uint32_t rch = 0;  // bit q: column c0+q reached (or padding)
#pragma unroll
    for (int q = 0; q < CPL; ++q) v[q] = 0;
    int32_t* list = lists;
    int32_t* next = lists + n;
    int nroots = n;
    int phases = 0, dual_steps = 0, rows_scanned = 0;
    bool fatal = false;

    for (int phase = 0; nroots > 0; ++phase) {
      uint32_t pad = 0;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        key[q] = KMB_KEY_INF;
        if (c0 + q >= n) pad |= 1u << q;
      }
      rch = pad;
      int32_t D = 0;
      int head = 0, tail = nroots, nfound = 0;
      for (int round = 0;; ++round) {
        // ---- relax rows list[head, tail)  (hungarian.cpp:164-172) ----
        int r = head;
        for (; r + 3 < tail; r += 4) {
          int32_t ii[4];
          uint32_t bb[4];
          RowVec<CPL> cv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            ii[k] = list[r + k];
            bb[k] = static_cast<uint32_t>(static_cast<int32_t>(KMB_BIAS) - w[ii[k]]);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            cv[k] = load_row<CPL, SMEM_C>(Cm + static_cast<int64_t>(ii[k]) * np + c0);
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int q = 0; q < CPL; ++q)
              key[q] = umin64(key[q], pack_key(static_cast<uint32_t>(cv[k].x[q]) + bb[k], ii[k]));
        }
        for (; r < tail; ++r) {
          const int32_t i = list[r];
          const uint32_t b = static_cast<uint32_t>(static_cast<int32_t>(KMB_BIAS) - w[i]);
          const RowVec<CPL> cv = load_row<CPL, SMEM_C>(Cm + static_cast<int64_t>(i) * np + c0);
#pragma unroll
          for (int q = 0; q < CPL; ++q)
            key[q] = umin64(key[q], pack_key(static_cast<uint32_t>(cv.x[q]) + b, i));
        }
        rows_scanned += tail - head;
        if (phase == 0 && round == 0 && a.seed == 1) {  // column reduction, :328-333
#pragma unroll
          for (int q = 0; q < CPL; ++q)
            if (!((pad >> q) & 1)) v[q] = static_cast<int32_t>(key_val(key[q]));
        }
        // ---- min unreached slack' (hungarian.cpp:203-206) ----
        int32_t s[CPL];
        int32_t lm = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          s[q] = static_cast<int32_t>(key_val(key[q])) - v[q];
          if (!((rch >> q) & 1)) lm = min(lm, s[q]);
        }
        const int32_t m = __reduce_min_sync(FULL, lm);
        if (m > D) {
          if (nfound > 0) break;  // closure exhausted (continue_bfs)
          if (m == 0x7fffffff) {
            fatal = true;
            break;
          }
          D = m;  // dual step (hungarian.cpp:207-215), applied lazily
          ++dual_steps;
        }
        // ---- absorb zero-slack columns (hungarian.cpp:186-199) ----
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const bool tight = !((rch >> q) & 1) && s[q] == D;
          bool newrow = false, newfree = false;
          int32_t i2 = -1;
          const int col = c0 + q;
          if (tight) {
            rch |= 1u << q;
            dc[q] = D;
            const int32_t par = key_row(key[q]);
            tree_par[col] = par;
            const int32_t root = root_row[par];
            i2 = match_col[col];
            if (i2 < 0) {
              newfree = true;
              atomicMin(claim + root, wclaim(phase, col));
            } else {
              newrow = true;
              w[i2] = u[i2] - D;
              root_row[i2] = root;
            }
          }
          const uint32_t rm = __ballot_sync(FULL, newrow);
          if (newrow) list[tail + __popc(rm & ((1u << lane) - 1))] = i2;
          tail += __popc(rm);
          const uint32_t fm = __ballot_sync(FULL, newfree);
          if (newfree) found[nfound + __popc(fm & ((1u << lane) - 1))] = col;
          nfound += __popc(fm);
        }
        __syncwarp();
        head = r;  // == old tail
        if (nfound > 0 && (!a.continue_bfs || head == tail)) break;
      }
      if (fatal) break;
      // ---- end of phase: finalise duals, next free rows, flips ----
      int nnext = 0;
      for (int rb = 0; rb < tail; rb += 32) {
        const int rr = rb + lane;
        bool keep = false;
        int32_t i = 0;
        if (rr < tail) {
          i = list[rr];
          const int32_t un = w[i] + D;
          u[i] = un;
          if (rr < nroots && !wclaimed_in(claim[i], phase)) {
            keep = true;
            w[i] = un;
            root_row[i] = i;
          }
        }
        const uint32_t km = __ballot_sync(FULL, keep);
        if (keep) next[nnext + __popc(km & ((1u << lane) - 1))] = i;
        nnext += __popc(km);
      }
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (((rch >> q) & 1) && !((pad >> q) & 1)) v[q] -= D - dc[q];
      __syncwarp();
      for (int f = lane; f < nfound; f += 32) {
        int32_t j = found[f];
        const int32_t root = root_row[tree_par[j]];
        if (claim[root] != wclaim(phase, j)) continue;
        for (;;) {
          const int32_t i = tree_par[j];
          const int32_t nx = match_row[i];
          match_row[i] = j;
          match_col[j] = i;
          if (nx < 0) break;
          j = nx;
        }
      }
      __syncwarp();
      int32_t* t = list;
      list = next;
      next = t;
      nroots = nnext;
      ++phases;
    }
    // ---- outputs ----
    int64_t tot = 0;
    for (int k = lane; k < n; k += 32) {
      const int32_t mr = match_row[k];
      a.row_to_col[static_cast<int64_t>(inst) * n + k] = mr;
      a.u[static_cast<int64_t>(inst) * n + k] = u[k];
      if (mr >= 0) tot += SMEM_C ? Cs[static_cast<int64_t>(k) * np + mr] : __ldg(Cg + static_cast<int64_t>(k) * np + mr);
    }
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (c0 + q < n) a.v[static_cast<int64_t>(inst) * n + c0 + q] = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) {
      a.total_cost[inst] = tot;
      a.status[inst] = fatal ? -2 : 0;
      if (a.stats) {
        a.stats[3 * static_cast<int64_t>(inst) + 0] = phases;
        a.stats[3 * static_cast<int64_t>(inst) + 1] = dual_steps;
        a.stats[3 * static_cast<int64_t>(inst) + 2] = rows_scanned;
      }
    }
    __syncwarp();
  }
}

int warp_max_n() { return 256; }

size_t warp_smem_per_warp(int n, int pitch, bool smem_c) {
  const size_t c = smem_c ? static_cast<size_t>(n) * pitch * 4 : 0;
  return (c + static_cast<size_t>(warp_state_words(n)) * 4 + 16 + 15) & ~static_cast<size_t>(15);
}

template <int CPL, bool SMEM_C>
static cudaError_t launch_t(const WarpArgs& a, int sm_count, int wpb, cudaStream_t st,
                            int* grid_out) {
  auto kern = k_warp_batch<CPL, SMEM_C>;
  const size_t smem = warp_smem_per_warp(a.n, a.pitch, SMEM_C) * wpb;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * wpb, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int warps_needed = a.batch;
  int grid = sm_count * occ;
  const int grid_needed = (warps_needed + wpb - 1) / wpb;
  if (grid > grid_needed) grid = grid_needed;
  if (grid_out) *grid_out = grid;
  kern<<<grid, 32 * wpb, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_warp_batch(const WarpArgs& a, int sm_count, bool smem_c, cudaStream_t st,
                              int* grid_out) {
  if (a.n < 1 || a.n > 256 || a.pitch % 4 != 0) return cudaErrorInvalidValue;
  const int cpl = a.n <= 32 ? 1 : a.n <= 64 ? 2 : a.n <= 128 ? 4 : 8;
  if (smem_c && warp_smem_per_warp(a.n, a.pitch, true) > 227 * 1024) smem_c = false;
  const int wpb = smem_c ? 1 : 4;
#define KMB_L(C)                                                                   \
  return smem_c ? launch_t<C, true>(a, sm_count, wpb, st, grid_out)                \
                : launch_t<C, false>(a, sm_count, wpb, st, grid_out)
  switch (cpl) {
    case 1: KMB_L(1);
    case 2: KMB_L(2);
    case 4: KMB_L(4);
    default: KMB_L(8);
  }
#undef KMB_L
}

}  // namespace kmb
