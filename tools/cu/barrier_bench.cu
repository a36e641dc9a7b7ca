// Grid-barrier microbenchmark (tools only): cost per barrier for G persistent
// CTAs, for the engine's GridBarrier and variants.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2005_01182_b200/csrc/kmb_common.cuh"

using namespace kmb;

__device__ __forceinline__ unsigned long long ldacq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// variant 0: engine GridBarrier
__global__ void k_b0(unsigned long long* ctr, int iters, unsigned long long* out) {
  GridBarrier bar = GridBarrier::make(ctr, gridDim.x);
  const unsigned long long t0 = globaltimer_ns();
  for (int k = 0; k < iters; ++k) bar.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = globaltimer_ns() - t0;
}

// variant 1: poll with nanosleep backoff
__global__ void k_b1(unsigned long long* ctr, int iters, unsigned long long* out, int ns) {
  unsigned long long target = 0;
  const unsigned long long t0 = globaltimer_ns();
  for (int k = 0; k < iters; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      target += gridDim.x;
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
      while (ldacq(ctr) < target) __nanosleep(ns);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = globaltimer_ns() - t0;
}

// variant 2: hierarchical: cluster barrier, one red per cluster, leader polls, cluster barrier
__global__ void k_b2(unsigned long long* ctr, int iters, unsigned long long* out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned ncl = gridDim.x / cl.num_blocks();
  unsigned long long target = 0;
  const bool lead = cl.block_rank() == 0 && threadIdx.x == 0;
  const unsigned long long t0 = globaltimer_ns();
  for (int k = 0; k < iters; ++k) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (lead) {
      target += ncl;
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
      while (ldacq(ctr) < target) {
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = globaltimer_ns() - t0;
}

// variant 3: last arriver flips a generation word; others poll it (acq)
__global__ void k_b3(unsigned long long* ctr, int iters, unsigned long long* out) {
  unsigned long long* gen = ctr + 16;  // separate 128-B line
  const unsigned long long t0 = globaltimer_ns();
  for (int k = 0; k < iters; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long old;
      asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
      if (old == (unsigned long long)(k + 1) * gridDim.x - 1) {
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(gen), "l"((unsigned long long)(k + 1)) : "memory");
      } else {
        while (ldacq(gen) < (unsigned long long)(k + 1)) {
        }
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = globaltimer_ns() - t0;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long *ctr, *out;
  cudaMalloc(&ctr, 4096);
  cudaMalloc(&out, 64);
  const int iters = 20000;
  for (int G : {sms, 74, 37, 16}) {
    for (int v = 0; v < 6; ++v) {
      cudaMemset(ctr, 0, 4096);
      void* args0[] = {&ctr, (void*)&iters, &out};
      int ns = v == 1 ? 32 : 128;
      void* args1[] = {&ctr, (void*)&iters, &out, &ns};
      cudaError_t e = cudaSuccess;
      if (v == 0) e = cudaLaunchCooperativeKernel((void*)k_b0, G, 512, args0, 0, 0);
      else if (v == 1 || v == 2) e = cudaLaunchCooperativeKernel((void*)k_b1, G, 512, args1, 0, 0);
      else if (v == 3) e = cudaLaunchCooperativeKernel((void*)k_b3, G, 512, args0, 0, 0);
      else {
        const int cs = v == 4 ? 2 : 4;
        if (G % cs) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = G; cfg.blockDim = 512;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
        cfg.attrs = at; cfg.numAttrs = 2;
        e = cudaLaunchKernelEx(&cfg, k_b2, ctr, iters, out);
      }
      cudaError_t e2 = cudaDeviceSynchronize();
      unsigned long long ns_total = 0;
      cudaMemcpy(&ns_total, out, 8, cudaMemcpyDeviceToHost);
      const char* name[] = {"engine", "sleep32", "sleep128", "lastflip", "cluster2", "cluster4"};
      printf("G=%3d %-9s %s %s: %.3f us/barrier\n", G, name[v], cudaGetErrorString(e), cudaGetErrorString(e2),
             ns_total / 1e3 / iters);
    }
  }
  return 0;
}
