// 64-bit cost path: the reference's own input type (OTInstance::cost is
// std::vector<int64_t>, core.hpp) end to end on the device.
//
// * k_minmax / k_convert: validation and the K11 quantization
//   chat = floor(C * B / N) with its lossless flag (quantize_costs,
//   hungarian.cpp:33-53), or a plain narrowing to int32, in one pass.
//   Instances whose (quantized) costs fit the 32-bit engines' range [0, 2^29)
//   run there; everything else runs the wide engine below.
// * k_wide ("wide engine", stats->engine 9): one CTA per instance, 64-bit
//   costs, duals and keys, for costs up to the reference's validate_instance
//   headroom (core.cpp:47-53: n * maxC * (2n + 2) <= 2^62, so every lazy dual
//   and reduced cost, bounded by 3 * maxC, fits int64).  Same search as the
//   32-bit engines (lazy duals, argmin-parent forest,
//   dual step only when the tight closure of the free rows holds no free
//   column, step over the whole closure by the minimum slack), so the duals
//   equal the reference's; the search restarts from the free
//   rows after every augmentation (the restart schedule, oracle/kmb_mirror.c
//   kmm_solve) — this path is for totality over the reference's inputs, the
//   fast engines carry the benchmark configs.
//   Keys are (int64 value, int32 row) pairs compared lexicographically, so the
//   argmin parent is the smallest row among equal reduced costs.  Per-column
//   and per-row state live in a global workspace slot per CTA.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "kmb_common.cuh"
#include "kmb_internal.h"
#include "kmb_launch.h"

namespace kmb {
namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr int64_t WINF = KMB_I64_INF;

// ---- validation / quantization -------------------------------------------------

__global__ void k_minmax(const int64_t* __restrict__ C, int64_t ld, int64_t rows, int32_t cols,
                         long long* __restrict__ out /* [0] min, [1] max */) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  const int64_t total = rows * cols;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = k / cols, j = k - r * cols;
    const long long x = __ldg(reinterpret_cast<const long long*>(C + r * ld + j));
    lo = x < lo ? x : lo;
    hi = x > hi ? x : hi;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long a = __shfl_xor_sync(FULL, lo, o), b = __shfl_xor_sync(FULL, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

// dst[r][j] = Q ? floor(C[r][j] * B / N) : C[r][j], written as int64 (chat,
// optional) and/or int32 (narrow, optional; the caller checked the range).
// lossy: set to 1 when some C * B is not a multiple of N (hungarian.cpp:49).
template <bool Q>
__global__ void k_convert(const int64_t* __restrict__ C, int64_t ld, int64_t rows, int32_t cols,
                          int64_t B, int64_t N, int64_t* __restrict__ chat,
                          int32_t* __restrict__ narrow, int32_t* __restrict__ lossy) {
  bool exact = true;
  const int64_t total = rows * cols;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = k / cols, j = k - r * cols;
    const int64_t x = __ldg(reinterpret_cast<const long long*>(C + r * ld + j));
    int64_t q = x;
    if (Q) {
      const int64_t p = x * B;  // no overflow: B <= INT64_MAX / N and 0 <= x <= N
      q = p / N;
      exact &= q * N == p;
    }
    if (chat) chat[k] = q;
    if (narrow) narrow[k] = static_cast<int32_t>(q);
  }
  if (Q && lossy && !__all_sync(FULL, exact) && (threadIdx.x & 31) == 0) *lossy = 1;
}

__global__ void k_scale(int64_t* __restrict__ x, int64_t count, int64_t k) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] *= k;
}

// total[b] = sum_i C_b[i][r2c_b[i]] over assigned rows (objective_int on the
// caller's costs, core.cpp:76-90); one warp per instance.
__global__ void k_total(const int64_t* __restrict__ C, int64_t ld, int64_t inst_stride, int32_t batch,
                        int32_t n, const int32_t* __restrict__ r2c, int64_t* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < batch;
       b += (gridDim.x * blockDim.x) >> 5) {
    long long s = 0;
    for (int i = lane; i < n; i += 32) {
      const int32_t j = r2c[static_cast<int64_t>(b) * n + i];
      if (j >= 0) s += C[b * inst_stride + i * ld + j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) total[b] = s;
  }
}

// ---- the wide engine ------------------------------------------------------------

__device__ __forceinline__ bool key_less(int64_t av, int32_t ar, int64_t bv, int32_t br) {
  return av < bv || (av == bv && ar < br);
}

struct WideShared {
  long long red[33];
  int32_t nrows, nfound, won, stop;
  long long lo, hi;
  unsigned long long tot;
};

// block-wide minimum of x (every thread gets it); `red` is reused per call
template <int T>
__device__ __forceinline__ long long block_min(long long x, long long* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long y = __shfl_xor_sync(FULL, x, o);
    x = y < x ? y : x;
  }
  if (lane == 0) red[wid] = x;
  __syncthreads();
  if (wid == 0) {
    x = lane < T / 32 ? red[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const long long y = __shfl_xor_sync(FULL, x, o);
      x = y < x ? y : x;
    }
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  x = red[32];
  __syncthreads();  // red is free again
  return x;
}

template <int T>
__global__ void __launch_bounds__(T) k_wide(WideArgs a) {
  __shared__ WideShared sm;
  const int n = a.n;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  // workspace slot of this CTA
  const int64_t so = static_cast<int64_t>(blockIdx.x) * n;
  int64_t* keyv = a.ws64 + so * 6;  // per column
  int64_t* v = keyv + n;
  int64_t* dc = v + n;
  int64_t* u = dc + n;              // per row
  int64_t* w = u + n;
  uint64_t* claim = reinterpret_cast<uint64_t*>(w + n);
  int32_t* keyr = a.ws32 + so * 8;  // per column
  int32_t* rch = keyr + n;
  int32_t* tree_par = rch + n;
  int32_t* match_col = tree_par + n;
  int32_t* found = match_col + n;
  int32_t* match_row = found + n;   // per row
  int32_t* root_row = match_row + n;
  int32_t* rows = root_row + n;

  for (int inst = blockIdx.x; inst < a.batch; inst += gridDim.x) {
    const int64_t* Cm = a.C + static_cast<int64_t>(inst) * a.inst_stride;
    const int64_t ld = a.ld;
    const unsigned long long t0 = globaltimer_ns();
    if (t == 0) {
      sm.lo = LLONG_MAX;
      sm.hi = 0;
      sm.tot = 0;
      sm.stop = 0;
    }
    __syncthreads();
    // validation (core.cpp:38-53) and the row reductions (hungarian.cpp:323-327)
    {
      long long lo_all = LLONG_MAX, hi_all = 0;
      for (int i = wid; i < n; i += T / 32) {
        long long lo = LLONG_MAX, hi = 0;
        for (int k = lane; k < n; k += 32) {
          const long long x = __ldg(reinterpret_cast<const long long*>(Cm + i * ld + k));
          lo = x < lo ? x : lo;
          hi = x > hi ? x : hi;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const long long p = __shfl_xor_sync(FULL, lo, o), q = __shfl_xor_sync(FULL, hi, o);
          lo = p < lo ? p : lo;
          hi = q > hi ? q : hi;
        }
        lo_all = lo < lo_all ? lo : lo_all;
        hi_all = hi > hi_all ? hi : hi_all;
        if (lane == 0) {
          u[i] = a.seed == 1 ? lo : 0;
          w[i] = u[i];
          match_row[i] = -1;
          root_row[i] = i;
          rows[i] = i;
          claim[i] = ~0ull;
        }
      }
      if (lane == 0) {
        atomicMin(&sm.lo, lo_all);
        atomicMax(&sm.hi, hi_all);
      }
    }
    for (int j = t; j < n; j += T) {
      keyv[j] = WINF;
      keyr[j] = INT_MAX;
      v[j] = 0;
      dc[j] = 0;
      rch[j] = 0;
      match_col[j] = -1;
    }
    __syncthreads();
    // the host checked validate_instance's headroom; this guards the int64 bound
    const int status0 = sm.lo < 0 ? 2 : (sm.hi > a.max_cost ? 3 : 0);
    if (status0) {
      if (t == 0) {
        a.status[inst] = status0;
        a.total_cost[inst] = 0;
        if (a.converged) a.converged[inst] = 0;
      }
      if (a.stats && t < KMB_ISTATS) a.stats[KMB_ISTATS * static_cast<int64_t>(inst) + t] = 0;
      for (int k = t; k < n; k += T) a.row_to_col[static_cast<int64_t>(inst) * n + k] = -1;
      __syncthreads();
      continue;
    }
    if (t == 0) {
      sm.nrows = n;
      sm.nfound = 0;
    }
    int nrows = n, head = 0, nfree = n;
    int64_t D = 0;
    int epochs = 0, dual_steps = 0;
    int64_t rounds = 0, rows_scanned = 0;
    bool first = true, stopped = false;
    int status = 0;
    __syncthreads();

    while (nfree > 0) {
      if (rounds > 4ll * n * n + 64) {  // a valid search ends in n epochs of <= 2n + 1 rounds
        status = -2;
        break;
      }
      ++rounds;
      // ---- relax the rows reached last round (hungarian.cpp:164-172) ----
      for (int j = t; j < n; j += T) {
        if (rch[j]) continue;
        int64_t bv = keyv[j];
        int32_t br = keyr[j];
        int r = head;
        for (; r + 4 <= nrows; r += 4) {
          int32_t i[4];
          int64_t c[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) i[k] = rows[r + k];
#pragma unroll
          for (int k = 0; k < 4; ++k) c[k] = __ldg(reinterpret_cast<const long long*>(Cm + i[k] * ld + j));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int64_t x = c[k] - w[i[k]];
            if (key_less(x, i[k], bv, br)) {
              bv = x;
              br = i[k];
            }
          }
        }
        for (; r < nrows; ++r) {
          const int32_t i = rows[r];
          const int64_t x = __ldg(reinterpret_cast<const long long*>(Cm + i * ld + j)) - w[i];
          if (key_less(x, i, bv, br)) {
            bv = x;
            br = i;
          }
        }
        keyv[j] = bv;
        keyr[j] = br;
        if (first && a.seed == 1) v[j] = bv;  // column reductions, :328-333
      }
      rows_scanned += nrows - head;
      head = nrows;
      first = false;
      // ---- min unreached slack' (hungarian.cpp:203-206) ----
      long long lm = LLONG_MAX;
      for (int j = t; j < n; j += T)
        if (!rch[j] && keyv[j] != WINF) {
          const long long s = keyv[j] - v[j];
          lm = s < lm ? s : lm;
        }
      const long long m = block_min<T>(lm, sm.red);
      if (m > D) {
        if (m == LLONG_MAX) {  // no unreached column is reachable: invariant broken
          status = -2;
          break;
        }
        D = m;  // dual step (hungarian.cpp:207-215), applied lazily
        ++dual_steps;
      }
      // ---- absorb zero-slack columns (hungarian.cpp:186-199) ----
      for (int j = t; j < n; j += T) {
        if (rch[j] || keyv[j] == WINF || keyv[j] - v[j] != D) continue;
        rch[j] = 1;
        dc[j] = D;
        const int32_t par = keyr[j];
        tree_par[j] = par;
        const int32_t root = root_row[par];
        const int32_t i2 = match_col[j];
        if (i2 < 0) {
          atomicMin(reinterpret_cast<unsigned long long*>(claim + root),
                    static_cast<unsigned long long>(claim_key(epochs, j)));
          found[atomicAdd(&sm.nfound, 1)] = j;
        } else {
          w[i2] = u[i2] - D;
          root_row[i2] = root;
          rows[atomicAdd(&sm.nrows, 1)] = i2;
        }
      }
      __syncthreads();
      nrows = sm.nrows;
      const int nfound = sm.nfound;
      if (nfound == 0) continue;

      // ---- augment: each claimed tree flips the path to its smallest free column
      if (t == 0) sm.won = 0;
      __syncthreads();
      int won = 0;
      for (int f = t; f < nfound; f += T) {
        int32_t j = found[f];
        if (claim[root_row[tree_par[j]]] != claim_key(epochs, j)) continue;
        ++won;
        for (;;) {
          const int32_t i = tree_par[j];
          const int32_t nx = match_row[i];
          match_row[i] = j;
          match_col[j] = i;
          if (nx < 0) break;
          j = nx;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) won += __shfl_xor_sync(FULL, won, o);
      if (lane == 0 && won) atomicAdd(&sm.won, won);
      // ---- restart: finalise every lazy dual, the free rows seed the next search
      for (int r = t; r < nrows; r += T) {
        const int32_t i = rows[r];
        u[i] = w[i] + D;
      }
      for (int j = t; j < n; j += T) {
        if (rch[j]) v[j] -= D - dc[j];
        rch[j] = 0;
        dc[j] = 0;
        keyv[j] = WINF;
        keyr[j] = INT_MAX;
      }
      if (t == 0 && a.deadline_ns > 0 &&
          globaltimer_ns() - t0 > static_cast<unsigned long long>(a.deadline_ns))
        sm.stop = 1;
      __syncthreads();
      nfree -= sm.won;
      if (t == 0) {
        sm.nrows = 0;
        sm.nfound = 0;
      }
      __syncthreads();
      for (int i = t; i < n; i += T)
        if (match_row[i] < 0) {
          w[i] = u[i];
          root_row[i] = i;
          rows[atomicAdd(&sm.nrows, 1)] = i;
        }
      __syncthreads();
      nrows = sm.nrows;
      head = 0;
      D = 0;
      ++epochs;
      if (sm.stop && nfree > 0) {
        stopped = true;
        break;
      }
    }
    __syncthreads();
    // ---- outputs ----
    long long tot = 0;
    for (int k = t; k < n; k += T) {
      const int32_t mr = match_row[k];
      a.row_to_col[static_cast<int64_t>(inst) * n + k] = mr;
      a.u[static_cast<int64_t>(inst) * n + k] = u[k];
      a.v[static_cast<int64_t>(inst) * n + k] = v[k];
      if (mr >= 0) tot += Cm[k * ld + mr];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) atomicAdd(&sm.tot, static_cast<unsigned long long>(tot));
    __syncthreads();
    if (t == 0) {
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
    __syncthreads();
  }
}

constexpr int kWideThreads = 512;

int grid_for(int64_t work, int sm_count) {
  const int64_t g = (work + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count) * 8;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

int wide_slots(int batch, int sm_count) {
  const int cap = sm_count * 2;  // 2 CTAs of 512 threads per SM
  return batch < cap ? batch : cap;
}
size_t wide_ws64_bytes(int n, int slots) { return static_cast<size_t>(slots) * n * 6 * 8; }
size_t wide_ws32_bytes(int n, int slots) { return static_cast<size_t>(slots) * n * 8 * 4; }

cudaError_t launch_wide(const WideArgs& a, int slots, cudaStream_t st) {
  k_wide<kWideThreads><<<slots, kWideThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_minmax_i64(const int64_t* C, int64_t ld, int64_t rows, int32_t cols, long long* out,
                              int sm_count, cudaStream_t st) {
  k_minmax<<<grid_for(rows * cols, sm_count), 256, 0, st>>>(C, ld, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_convert_i64(const int64_t* C, int64_t ld, int64_t rows, int32_t cols, bool quantize,
                               int64_t B, int64_t N, int64_t* chat, int32_t* narrow, int32_t* lossy,
                               int sm_count, cudaStream_t st) {
  const int g = grid_for(rows * cols, sm_count);
  if (quantize)
    k_convert<true><<<g, 256, 0, st>>>(C, ld, rows, cols, B, N, chat, narrow, lossy);
  else
    k_convert<false><<<g, 256, 0, st>>>(C, ld, rows, cols, B, N, chat, narrow, lossy);
  return cudaGetLastError();
}

cudaError_t launch_scale_i64(int64_t* x, int64_t count, int64_t k, int sm_count, cudaStream_t st) {
  k_scale<<<grid_for(count, sm_count), 256, 0, st>>>(x, count, k);
  return cudaGetLastError();
}

cudaError_t launch_total_i64(const int64_t* C, int64_t ld, int64_t inst_stride, int32_t batch, int32_t n,
                             const int32_t* r2c, int64_t* total, int sm_count, cudaStream_t st) {
  const int g = grid_for(static_cast<int64_t>(batch) * 32, sm_count);
  k_total<<<g, 256, 0, st>>>(C, ld, inst_stride, batch, n, r2c, total);
  return cudaGetLastError();
}

}  // namespace kmb
