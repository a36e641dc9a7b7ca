// C++ host side of the stream-ordered and multi-context batch calls, through
// the C ABI only (include/kmb.h) and the CUDA runtime:
//   * kmb_solve_batch_async_i32 on a caller stream equals kmb_solve_batch_i32;
//   * the same call captured in a CUDA graph (cudaStreamBeginCapture) and
//     replayed on new costs written into the captured input buffer;
//   * kmb_solve_batch_multi_i32 over two contexts equals the single-context call;
//   * per-instance statuses of the stream-ordered call (a negative cost).
// Exit code 0 = pass.  Run by tests/test_cpp_drop_in.py on the GPU box.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "kmb.h"

#define CHECK(x)                                                                        \
  do {                                                                                  \
    if (!(x)) {                                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s (%s)\n", __FILE__, __LINE__, #x, kmb_last_error()); \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)
#define CUDA(x) CHECK((x) == cudaSuccess)

namespace {

struct HostOut {
  std::vector<int32_t> r2c;
  std::vector<int64_t> u, v, tot;
  HostOut(int b, int n) : r2c(size_t(b) * n), u(size_t(b) * n), v(size_t(b) * n), tot(b) {}
  bool operator==(const HostOut& o) const { return r2c == o.r2c && u == o.u && v == o.v && tot == o.tot; }
};

struct DevBatch {
  int32_t *c = nullptr, *r2c = nullptr, *status = nullptr;
  int64_t *u = nullptr, *v = nullptr, *tot = nullptr;
  int b, n;
  DevBatch(int b_, int n_) : b(b_), n(n_) {
    const size_t bn = size_t(b) * n;
    cudaMalloc(&c, bn * n * 4);
    cudaMalloc(&r2c, bn * 4);
    cudaMalloc(&u, bn * 8);
    cudaMalloc(&v, bn * 8);
    cudaMalloc(&tot, size_t(b) * 8);
    cudaMalloc(&status, size_t(b) * 4);
  }
  ~DevBatch() {
    cudaFree(c); cudaFree(r2c); cudaFree(u); cudaFree(v); cudaFree(tot); cudaFree(status);
  }
  void fetch(HostOut& h) const {
    const size_t bn = size_t(b) * n;
    cudaMemcpy(h.r2c.data(), r2c, bn * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h.u.data(), u, bn * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h.v.data(), v, bn * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h.tot.data(), tot, size_t(b) * 8, cudaMemcpyDeviceToHost);
  }
};

std::vector<int32_t> random_batch(int b, int n, uint32_t seed) {
  std::mt19937 g(seed);
  std::uniform_int_distribution<int32_t> d(0, 100000);
  std::vector<int32_t> c(size_t(b) * n * n);
  for (auto& x : c) x = d(g);
  return c;
}

int sync_solve(kmb_context* ctx, const std::vector<int32_t>& c, int b, int n, HostOut& h) {
  return kmb_solve_batch_i32(ctx, c.data(), b, n, KMB_SEED_BATCHED, h.r2c.data(), h.u.data(),
                             h.v.data(), h.tot.data(), nullptr);
}

}  // namespace

int main() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    std::fprintf(stderr, "no CUDA device\n");
    return 2;
  }
  const int b = 40, n = 96;
  kmb_context* ctx = nullptr;
  CHECK(kmb_create(0, &ctx) == KMB_OK);
  cudaStream_t st;
  CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CHECK(kmb_set_stream(ctx, st) == KMB_OK);

  // 1. stream-ordered == synchronous
  const std::vector<int32_t> c1 = random_batch(b, n, 1);
  HostOut ref1(b, n), got(b, n);
  CHECK(sync_solve(ctx, c1, b, n, ref1) == KMB_OK);
  DevBatch d(b, n);
  CUDA(cudaMemcpy(d.c, c1.data(), c1.size() * 4, cudaMemcpyHostToDevice));
  CUDA(cudaMemset(d.status, 0xff, size_t(b) * 4));
  CHECK(kmb_solve_batch_async_i32(ctx, d.c, b, n, KMB_SEED_BATCHED, d.r2c, d.u, d.v, d.tot, d.status) == KMB_OK);
  CUDA(cudaStreamSynchronize(st));
  d.fetch(got);
  CHECK(got == ref1);
  std::vector<int32_t> status(b);
  CUDA(cudaMemcpy(status.data(), d.status, size_t(b) * 4, cudaMemcpyDeviceToHost));
  for (int t = 0; t < b; ++t) CHECK(status[t] == 0);

  // 2. captured in a CUDA graph, replayed on new costs
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  CHECK(kmb_solve_batch_async_i32(ctx, d.c, b, n, KMB_SEED_BATCHED, d.r2c, d.u, d.v, d.tot, d.status) == KMB_OK);
  CUDA(cudaStreamEndCapture(st, &graph));
  CUDA(cudaGraphInstantiate(&exec, graph, 0));
  const std::vector<int32_t> c2 = random_batch(b, n, 2);
  HostOut ref2(b, n);
  CHECK(sync_solve(ctx, c2, b, n, ref2) == KMB_OK);
  CUDA(cudaMemcpyAsync(d.c, c2.data(), c2.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA(cudaGraphLaunch(exec, st));
  CUDA(cudaStreamSynchronize(st));
  d.fetch(got);
  CHECK(got == ref2);
  CUDA(cudaGraphExecDestroy(exec));
  CUDA(cudaGraphDestroy(graph));

  // 3. two contexts (one per GPU in production; here both on device 0)
  kmb_context* ctx2 = nullptr;
  CHECK(kmb_create(ndev > 1 ? 1 : 0, &ctx2) == KMB_OK);
  kmb_context* both[2] = {ctx, ctx2};
  HostOut multi(b, n);
  CHECK(kmb_solve_batch_multi_i32(both, 2, c1.data(), b, n, KMB_SEED_BATCHED, multi.r2c.data(),
                                  multi.u.data(), multi.v.data(), multi.tot.data(), nullptr) == KMB_OK);
  CHECK(multi == ref1);

  // 4. statuses: a negative cost in instance 3 fails that instance only
  std::vector<int32_t> c3 = c1;
  c3[size_t(3) * n * n + 5] = -1;
  CUDA(cudaMemcpy(d.c, c3.data(), c3.size() * 4, cudaMemcpyHostToDevice));
  CHECK(kmb_solve_batch_async_i32(ctx, d.c, b, n, KMB_SEED_BATCHED, d.r2c, d.u, d.v, d.tot, d.status) == KMB_OK);
  CUDA(cudaStreamSynchronize(st));
  CUDA(cudaMemcpy(status.data(), d.status, size_t(b) * 4, cudaMemcpyDeviceToHost));
  for (int t = 0; t < b; ++t) CHECK(status[t] == (t == 3 ? KMB_ENEGATIVE : 0));
  // host buffers are rejected by the stream-ordered call
  CHECK(kmb_solve_batch_async_i32(ctx, c1.data(), b, n, KMB_SEED_BATCHED, d.r2c, d.u, d.v, d.tot,
                                  d.status) == KMB_EINVAL);

  kmb_destroy(ctx2);
  kmb_destroy(ctx);
  cudaStreamDestroy(st);
  std::printf("test_stream: ok\n");
  return 0;
}
