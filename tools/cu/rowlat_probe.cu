// Memory-side model of the warp engine's relax (config 3): 4096 resident warps
// (28 per SM), each chasing dependent random rows inside its own matrix.
// Varies the row size (512 B int32 rows vs 256 B 16-bit rows), the footprint
// per warp (64 KiB vs 32 KiB) and the rows in flight per dependent step, and
// prints rows/us - what a 16-bit resident encoding could buy on the memory
// side.  Build: nvcc -O3 -std=c++17 -arch=sm_100a -o rowlat_probe rowlat_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <int LB, int K>  // LB: bytes per lane per row (16 or 8); K rows in flight
__global__ void __launch_bounds__(128, 7) chase(const char* base, uint32_t region, uint32_t rows_per_region,
                                                int steps, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const char* reg = base + static_cast<size_t>(warp) * region + lane * LB;
  uint32_t s = warp * 2654435761u + 12345u, acc = 0;
  for (int it = 0; it < steps; ++it) {
    uint32_t r[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      s = s * 1664525u + 1013904223u;
      r[k] = ((s >> 8) + (acc & 1u)) % rows_per_region;  // depends on the previous loads
    }
    if constexpr (LB == 16) {
      int4 v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = __ldg(reinterpret_cast<const int4*>(reg + r[k] * (32u * LB)));
#pragma unroll
      for (int k = 0; k < K; ++k) acc += v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    } else {
      int2 v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = __ldg(reinterpret_cast<const int2*>(reg + r[k] * (32u * LB)));
#pragma unroll
      for (int k = 0; k < K; ++k) acc += v[k].x ^ v[k].y;
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
  }
  if (lane == 0) out[warp] = acc;
}

template <int LB, int K>
static void run(const char* d, uint32_t region, int warps, int steps, uint32_t* out, const char* name) {
  cudaFuncSetAttribute(chase<LB, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 72);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    chase<LB, K><<<warps / 4, 128>>>(d, region, region / (32 * LB), steps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double rows = double(warps) * steps * K;
  printf("%-34s region %3u KiB rows/step %d: %.3f ms, %.1f rows/us, %.2f TB/s requested, %.2f us per dependent step\n", name,
         region >> 10, K, best, rows / best / 1e3, rows * 32 * LB / best / 1e9, best * 1e3 / steps);
}

int main() {
  const int warps = 4096;
  char* d;
  uint32_t* out;
  cudaMalloc(&d, size_t(warps) * 65536);
  cudaMemset(d, 1, size_t(warps) * 65536);
  cudaMalloc(&out, warps * 4);
  const int steps = 800;
  run<16, 1>(d, 65536, warps, steps, out, "512 B rows (int32), footprint 256M");
  run<8, 1>(d, 32768, warps, steps, out, "256 B rows (u16), footprint 128M");
  run<16, 1>(d, 32768, warps, steps, out, "512 B rows, footprint 128M");
  run<16, 1>(d, 4096, warps, steps, out, "512 B rows, footprint 16M (L2)");
  run<16, 5>(d, 65536, warps, steps / 4, out, "512 B rows (int32), footprint 256M");
  run<8, 5>(d, 32768, warps, steps / 4, out, "256 B rows (u16), footprint 128M");
  run<8, 10>(d, 32768, warps, steps / 4, out, "256 B rows (u16), footprint 128M");
  run<16, 5>(d, 32768, warps, steps / 4, out, "512 B rows, footprint 128M");
  run<16, 5>(d, 4096, warps, steps / 4, out, "512 B rows, footprint 16M (L2)");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
