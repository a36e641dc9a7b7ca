// Batched small instances (BASELINE config 3: 4096 independent n=128 solves):
// one CTA per instance, the whole n x n cost matrix staged into shared memory
// by a TMA bulk copy (cp.async.bulk + mbarrier), every per-phase structure in
// SMEM, __syncthreads as the only barrier.  Persistent CTAs stride over the
// instances; several CTAs per SM overlap one instance's TMA load with the
// others' solves.
//
// The algorithm is exactly the engine of kmb_solver.cu with G = 1 (thread j
// owns column j, so the per-column min needs no cross-thread merge):
// multi-source search with lazy duals (hungarian.cpp:175-217 restated),
// argmin-parent forest augmentation in place of TightPhase
// (hungarian.cpp:223-309), reductions of hungarian.cpp:323-333 as seed 1.
#include <cuda_runtime.h>

#include <cstdint>

#include "kmb_common.cuh"
#include "kmb_internal.h"

namespace kmb {

constexpr int kBatchMaxN = 224;  // n*n*4 + per-row state must fit 227 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct BatchSmem {
  uint64_t bar;
  int32_t tail;
  int32_t ntail;
  int32_t nfound;
  int32_t status;
  int64_t part[8];
  int64_t m;
};

// dynamic smem: Cs[n*n] | u[n] w[n] (i64) | claim[n] (u64) | list[2][n]
//               match_row[n] match_col[n] root_row[n] tree_par[n] found[n] (i32)
__host__ __device__ inline size_t batch_smem_bytes(int n) {
  const size_t cs = ((static_cast<size_t>(n) * n * 4) + 15) & ~static_cast<size_t>(15);
  return cs + static_cast<size_t>(n) * (8 + 8 + 8 + 4 * 7);
}

__global__ void __launch_bounds__(256) k_batch_solve(BatchArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BatchSmem sm;
  const int n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int T = blockDim.x, nw = T >> 5;
  int32_t* Cs = reinterpret_cast<int32_t*>(dyn);
  const size_t cs_bytes = ((static_cast<size_t>(n) * n * 4) + 15) & ~static_cast<size_t>(15);
  int64_t* u = reinterpret_cast<int64_t*>(dyn + cs_bytes);
  int64_t* w = u + n;
  uint64_t* claim = reinterpret_cast<uint64_t*>(w + n);
  int32_t* lists = reinterpret_cast<int32_t*>(claim + n);
  int32_t* match_row = lists + 2 * n;
  int32_t* match_col = match_row + n;
  int32_t* root_row = match_col + n;
  int32_t* tree_par = root_row + n;
  int32_t* found = tree_par + n;

  const bool bulk = ((n * n) & 3) == 0;  // 16 B granularity of cp.async.bulk
  if (tid == 0) mbar_init(&sm.bar, 1);
  __syncthreads();
  uint32_t mbar_parity = 0;
  const int j = tid;  // owned column (and row, for per-row init)
  const bool own = j < n;

  for (int inst = blockIdx.x; inst < a.batch; inst += gridDim.x) {
    const int32_t* Cg = a.C + static_cast<int64_t>(inst) * n * n;
    // ---- stage the cost matrix: TMA bulk copy into SMEM ----
    if (bulk) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t total = static_cast<uint32_t>(n) * n * 4;
        mbar_arrive_expect_tx(&sm.bar, total);
        const uint32_t chunk = 32768;
        for (uint32_t off = 0; off < total; off += chunk) {
          const uint32_t b = total - off < chunk ? total - off : chunk;
          bulk_copy_g2s(reinterpret_cast<unsigned char*>(Cs) + off,
                        reinterpret_cast<const unsigned char*>(Cg) + off, b, &sm.bar);
        }
      }
    } else {
      for (int k = tid; k < n * n; k += T) Cs[k] = Cg[k];
    }
    // per-row / per-column init overlaps the copy
    if (own) {
      match_row[j] = -1;
      match_col[j] = -1;
      claim[j] = KMB_KEY_INF;
      root_row[j] = j;
      lists[j] = j;
    }
    if (tid == 0) {
      sm.tail = n;
      sm.ntail = 0;
      sm.nfound = 0;
      sm.status = 0;
    }
    if (bulk) {
      mbar_wait(&sm.bar, mbar_parity);
      mbar_parity ^= 1;
    }
    __syncthreads();
    // validation (core.cpp:144-145 + device range) and row reductions
    // (hungarian.cpp:323-327): one warp per row, conflict-free
    for (int i = wid; i < n; i += nw) {
      int32_t lo = 0x7fffffff, hi = 0;
      for (int k = lane; k < n; k += 32) {
        const int32_t x = Cs[i * n + k];
        lo = min(lo, x);
        hi = max(hi, x);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      const int64_t u0 = a.seed == 1 ? lo : 0;
      if (lane == 0) {
        if (lo < 0) atomicMax(&sm.status, 2);
        else if (hi >= (1 << 29)) atomicMax(&sm.status, 3);
        u[i] = u0;
        w[i] = u0;
      }
    }
    __syncthreads();
    if (sm.status != 0) {  // invalid instance: report, produce no assignment
      if (own) a.row_to_col[static_cast<int64_t>(inst) * n + j] = -1;
      if (tid == 0) {
        a.status[inst] = sm.status;
        a.total_cost[inst] = 0;
      }
      __syncthreads();
      continue;
    }

    int64_t v = 0, dc = 0;
    int64_t dual_steps = 0, rows_scanned = 0, phases = 0;
    int32_t* list = lists;
    int32_t* next = lists + n;
    bool fatal = false;
    for (int phase = 0;; ++phase) {
      const int nroots = sm.tail;
      if (nroots == 0) break;
      uint64_t key = KMB_KEY_INF;
      bool rch = !own;
      int64_t D = 0;
      int head = 0, tail = nroots, nfound = 0;
      for (int round = 0;; ++round) {
        // relax rows list[head, tail) for column j (hungarian.cpp:164-172)
        if (own) {
          int r = head;
          for (; r + 3 < tail; r += 4) {
            int32_t i[4];
            uint32_t c[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) i[k] = list[r + k];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              c[k] = static_cast<uint32_t>(Cs[i[k] * n + j]) + row_bias(w[i[k]]);
#pragma unroll
            for (int k = 0; k < 4; ++k) key = umin64(key, pack_key(c[k], i[k]));
          }
          for (; r < tail; ++r) {
            const int32_t i = list[r];
            key = umin64(key, pack_key(static_cast<uint32_t>(Cs[i * n + j]) + row_bias(w[i]), i));
          }
          if (phase == 0 && round == 0 && a.seed == 1) v = key_val(key);  // :328-333
        }
        rows_scanned += tail - head;
        int64_t s = (!rch) ? key_val(key) - v : KMB_I64_INF;
        s = warp_min_i64(s);
        if (lane == 0) sm.part[wid] = s;
        __syncthreads();
        int64_t m = KMB_I64_INF;
        for (int q = 0; q < nw; ++q) m = sm.part[q] < m ? sm.part[q] : m;
        if (m > D) {
          if (nfound > 0) break;  // closure exhausted (continue_bfs)
          if (m == KMB_I64_INF) {
            fatal = true;
            break;
          }
          D = m;
          ++dual_steps;
        }
        if (!rch && key_val(key) - v == D) {  // absorb (hungarian.cpp:186-199)
          rch = true;
          dc = D;
          const int32_t par = key_row(key);
          tree_par[j] = par;
          const int32_t root = root_row[par];
          const int32_t i2 = match_col[j];
          if (i2 < 0) {
            atomicMin(reinterpret_cast<unsigned long long*>(claim + root), claim_key(phase, j));
            found[atomicAdd(&sm.nfound, 1)] = j;
          } else {
            w[i2] = u[i2] - D;
            root_row[i2] = root;
            list[atomicAdd(&sm.tail, 1)] = i2;
          }
        }
        __syncthreads();
        head = tail;
        tail = sm.tail;
        nfound = sm.nfound;
        if (nfound > 0 && (!a.continue_bfs || head == tail)) break;
      }
      if (fatal) break;
      // ---- end of phase ----
      for (int r = tid; r < tail; r += T) {
        const int32_t i = list[r];
        const int64_t un = w[i] + D;
        u[i] = un;
        if (r < nroots && !claimed_in(claim[i], phase)) {
          const int pos = atomicAdd(&sm.ntail, 1);
          next[pos] = i;
          w[i] = un;
          root_row[i] = i;
        }
      }
      if (rch && own) v -= D - dc;
      for (int f = tid; f < nfound; f += T) {
        int32_t jj = found[f];
        const int32_t root = root_row[tree_par[jj]];
        if (claim[root] != claim_key(phase, jj)) continue;
        for (;;) {
          const int32_t i = tree_par[jj];
          const int32_t nxt = match_row[i];
          match_row[i] = jj;
          match_col[jj] = i;
          if (nxt < 0) break;
          jj = nxt;
        }
      }
      __syncthreads();
      if (tid == 0) {
        sm.tail = sm.ntail;
        sm.ntail = 0;
        sm.nfound = 0;
      }
      int32_t* t = list;
      list = next;
      next = t;
      ++phases;
      __syncthreads();
    }
    // ---- outputs ----
    int64_t tot = 0;
    if (own) {
      const int32_t mr = match_row[j];
      a.row_to_col[static_cast<int64_t>(inst) * n + j] = mr;
      a.u[static_cast<int64_t>(inst) * n + j] = u[j];
      a.v[static_cast<int64_t>(inst) * n + j] = v;
      tot = mr >= 0 ? Cs[j * n + mr] : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    __syncthreads();  // everyone done reading sm.part / Cs before reuse
    if (lane == 0) sm.part[wid] = tot;
    __syncthreads();
    if (tid == 0) {
      int64_t t = 0;
      for (int q = 0; q < nw; ++q) t += sm.part[q];
      a.total_cost[inst] = t;
      a.status[inst] = fatal ? -2 : 0;  // KMB_EINTERNAL
      if (a.stats) {
        int64_t* o = a.stats + KMB_ISTATS * static_cast<int64_t>(inst);
        o[0] = phases;
        o[1] = dual_steps;
        o[2] = rows_scanned;
        for (int k = 3; k < KMB_ISTATS; ++k) o[k] = 0;
      }
    }
    __syncthreads();
  }
}

int batch_max_n() { return kBatchMaxN; }

cudaError_t launch_batch(const BatchArgs& a, int sm_count, cudaStream_t st, int* grid_out) {
  if (a.n < 1 || a.n > kBatchMaxN) return cudaErrorInvalidValue;
  const int threads = ((a.n + 31) / 32) * 32;
  const size_t smem = batch_smem_bytes(a.n);
  cudaError_t e = cudaFuncSetAttribute(k_batch_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_batch_solve, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) occ = 1;
  int grid = sm_count * occ;
  if (grid > a.batch) grid = a.batch;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid;
  k_batch_solve<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace kmb
