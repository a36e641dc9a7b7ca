// Shared device helpers for the KM / batched-KM engine (sm_100a).
//
// Key packing.  A column's running minimum over reached rows is one 64-bit
// unsigned key  ((C_ij - w_i + 2^30) << 32) | i  (w_i = u_i - D_at_reach, see
// kmb_solver.cu).  With 0 <= C < 2^30 every dual stays in [-maxC, maxC]
// (SURVEY.md §7 "Integer widths"; argued in DESIGN.md), so C - w + 2^30 lies in
// (0, 3*2^30) and fits the high word.  Unsigned 64-bit min then gives the
// minimum reduced cost with ties broken by the smallest row — a deterministic
// argmin parent independent of scheduling.
#pragma once

#include <cstdint>

#define KMB_BIAS (1LL << 30)
#define KMB_KEY_INF 0xFFFFFFFFFFFFFFFFull
#define KMB_I64_INF 0x7FFFFFFFFFFFFFFFLL

namespace kmb {

__device__ __forceinline__ uint64_t pack_key(uint32_t hi, int32_t row) {
  return (static_cast<uint64_t>(hi) << 32) | static_cast<uint32_t>(row);
}
__device__ __forceinline__ int64_t key_val(uint64_t k) {
  return static_cast<int64_t>(k >> 32) - KMB_BIAS;
}
__device__ __forceinline__ int32_t key_row(uint64_t k) {
  return static_cast<int32_t>(k & 0xffffffffu);
}
// high word for row i: C_ij + (2^30 - w_i), computed in 32 bits.
__device__ __forceinline__ uint32_t row_bias(int64_t w) {
  return static_cast<uint32_t>(KMB_BIAS - w);
}
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// claim word of a tree root: smallest free column reaching it in phase `ph`
// wins; keys of later phases are smaller so stale claims never block, and the
// stamp ~(ph+1) never equals the all-ones "unclaimed" word.
__device__ __forceinline__ uint32_t claim_stamp(int32_t ph) {
  return ~static_cast<uint32_t>(ph + 1);
}
__device__ __forceinline__ uint64_t claim_key(int32_t ph, int32_t col) {
  return (static_cast<uint64_t>(claim_stamp(ph)) << 32) | static_cast<uint32_t>(col);
}
__device__ __forceinline__ bool claimed_in(uint64_t c, int32_t ph) {
  return static_cast<uint32_t>(c >> 32) == claim_stamp(ph);
}

// L1-bypassing loads for state other CTAs write (L1 is not coherent).
__device__ __forceinline__ int32_t ldcg(const int32_t* p) { return __ldcg(p); }
__device__ __forceinline__ int64_t ldcg(const int64_t* p) {
  return static_cast<int64_t>(__ldcg(reinterpret_cast<const long long*>(p)));
}
__device__ __forceinline__ uint64_t ldcg(const uint64_t* p) {
  return static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(p)));
}

// Streaming 128-bit load of immutable cost data: no L1 allocation.
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// relaxed polls (no L1 invalidation per iteration); the acquire is done once
// after the poll succeeds
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x < v ? x : v;
  }
  return v;
}

// Software grid barrier over a monotonically increasing 64-bit counter:
// barrier k completes when the counter reaches k*G; one atomic per CTA, then
// every CTA polls the same L2 line.  `epoch` is the CTA-local barrier count
// (all CTAs start from the same counter value, which is a multiple of G).
struct GridBarrier {
  unsigned long long* counter;
  unsigned long long target;
  unsigned int G;

  __device__ static GridBarrier make(unsigned long long* counter, unsigned int G) {
    return GridBarrier{counter, 0ull, G};
  }

  // bar.sync makes the CTA's writes visible to thread 0, whose release
  // reduction (cumulative) publishes them at gpu scope; the acquire poll orders
  // every later read after the other CTAs' releases.  No full fences.
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      target += G;
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(counter) : "memory");
      while (ld_acquire_u64(counter) < target) {
      }
    }
    __syncthreads();
  }
};

// All CTAs of the launch form ONE thread-block cluster (G <= 16): the hardware
// cluster barrier (release/acquire at cluster scope, covers global memory).
struct ClusterBarrier {
  __device__ static ClusterBarrier make(unsigned long long*, unsigned int) { return ClusterBarrier{}; }
  __device__ __forceinline__ void sync() {
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n"
        "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
};

}  // namespace kmb
