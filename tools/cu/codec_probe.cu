// Host-side probe for a 16-bit transport codec of host cost batches (config 3:
// 4096 x n=128 int32, 256 MiB).  Measures on the GPU box: host encode
// throughput (row min + 16-bit offsets) by thread count, plain memcpy by thread
// count, bare H2D of the raw and encoded sizes, and encode pipelined with the
// DMA chunk by chunk.  Build: nvcc -O3 -std=c++17 -o codec_probe codec_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

__attribute__((target_clones("arch=skylake-avx512", "avx2", "default")))
static int64_t encode_rows(const int32_t* src, int64_t rows, int n, uint16_t* off, int32_t* base) {
  int64_t wide = 0;
  for (int64_t r = 0; r < rows; ++r) {
    const int32_t* p = src + r * n;
    int32_t lo = p[0], hi = p[0];
    for (int j = 1; j < n; ++j) {
      lo = std::min(lo, p[j]);
      hi = std::max(hi, p[j]);
    }
    uint16_t* o = off + r * n;
    if (lo < 0 || hi - lo > 65535) {
      base[r] = INT32_MIN;
      ++wide;
      continue;
    }
    for (int j = 0; j < n; ++j) o[j] = static_cast<uint16_t>(p[j] - lo);
    base[r] = lo;
  }
  return wide;
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
static void par(int T, int64_t items, F f) {
  std::vector<std::thread> th;
  const int64_t per = (items + T - 1) / T;
  for (int t = 1; t < T; ++t) th.emplace_back([&, t] { f(per * t, std::min(items, per * (t + 1))); });
  f(0, std::min(items, per));
  for (auto& x : th) x.join();
}

int main() {
  const int B = 4096, n = 128;
  const int64_t rows = int64_t(B) * n, elems = rows * n;
  int32_t *h, *base;
  uint16_t* off;
  void* raw2;
  cudaMallocHost(&h, elems * 4);
  cudaMallocHost(&raw2, elems * 4);
  cudaMallocHost(&off, elems * 2);
  cudaMallocHost(&base, rows * 4);
  par(16, rows, [&](int64_t lo, int64_t hi) {
    uint64_t s = 0x9E3779B97F4A7C15ull * (lo + 1);
    for (int64_t k = lo * n; k < hi * n; ++k) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[k] = 245000 + static_cast<int32_t>(s % 50000) - 25000;
    }
  });
  void *d_raw, *d_enc;
  cudaMalloc(&d_raw, elems * 4);
  cudaMalloc(&d_enc, elems * 2 + rows * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  // bare H2D
  for (int rep = 0; rep < 3; ++rep) {
    for (size_t bytes : {size_t(elems) * 4, size_t(elems) * 2 + rows * 4}) {
      cudaEventRecord(e0, st);
      cudaMemcpyAsync(d_raw, h, bytes, cudaMemcpyHostToDevice, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("h2d %zu MiB: %.3f ms (%.1f GB/s)\n", bytes >> 20, ms, bytes / ms / 1e6);
    }
  }
  const int Ts[] = {1, 2, 4, 8, 12, 16, 24, 32};
  for (int T : Ts) {
    double best = 1e9, bestc = 1e9;
    int64_t wide = 0;
    for (int rep = 0; rep < 4; ++rep) {
      double t0 = now_ms();
      std::vector<int64_t> w(T, 0);
      par(T, rows, [&](int64_t lo, int64_t hi) {
        const int64_t per = (rows + T - 1) / T;
        w[lo / std::max<int64_t>(per, 1)] = encode_rows(h + lo * n, hi - lo, n, off + lo * n, base + lo);
      });
      best = std::min(best, now_ms() - t0);
      wide = 0;
      for (auto x : w) wide += x;
      t0 = now_ms();
      par(T, rows, [&](int64_t lo, int64_t hi) {
        std::memcpy(static_cast<char*>(raw2) + lo * n * 4, h + lo * n, (hi - lo) * n * 4);
      });
      bestc = std::min(bestc, now_ms() - t0);
    }
    printf("T=%2d encode %.3f ms (%.1f GB/s in)  memcpy %.3f ms (%.1f GB/s)  wide rows %lld\n", T, best,
           elems * 4 / best / 1e6, bestc, elems * 4 / bestc / 1e6, (long long)wide);
  }
  // pipelined: K chunks; threads encode chunk k, then its DMA is enqueued
  for (int T : {8, 12, 16}) {
    for (int K : {8, 16, 32}) {
      double best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaStreamSynchronize(st);
        const double t0 = now_ms();
        const int64_t cr = (rows + K - 1) / K;
        for (int k = 0; k < K; ++k) {
          const int64_t lo = k * cr, hi = std::min(rows, lo + cr);
          par(T, hi - lo, [&](int64_t a, int64_t b) {
            encode_rows(h + (lo + a) * n, b - a, n, off + (lo + a) * n, base + lo + a);
          });
          cudaMemcpyAsync(static_cast<char*>(d_enc) + lo * n * 2, off + lo * n, (hi - lo) * n * 2,
                          cudaMemcpyHostToDevice, st);
          cudaMemcpyAsync(static_cast<char*>(d_enc) + elems * 2 + lo * 4, base + lo, (hi - lo) * 4,
                          cudaMemcpyHostToDevice, st);
        }
        cudaStreamSynchronize(st);
        best = std::min(best, now_ms() - t0);
      }
      printf("pipelined T=%2d K=%2d: %.3f ms\n", T, K, best);
    }
  }
  return 0;
}
