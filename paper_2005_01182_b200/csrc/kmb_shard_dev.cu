// Column-sharded single instance with the exchange on the device (BASELINE
// config 5's multi-GPU mode; hungarian.cpp:175-217 per
// round): one persistent kernel per rank, k_solve_sharded (kmb_solver.cu, the
// grid engine with its row-side state replicated, RMem).  Per round each rank
// relaxes the new rows over its column slab, publishes its min-slack partial
// and its appends by storing them into every rank's replica, and meets the
// others at a system-scope counting barrier in rank 0's home block — no host
// round trip and no collective call per round (the host-driven protocol of
// kmb_shard.cu needs five per round).
//
// Ranks are GPUs (kmb_shard_dev_open / _connect exchange CUDA IPC handles of
// each rank's window, so replicas and the home block are peer-mapped over
// NVLink) or CTA groups of one cooperative launch on one GPU
// (kmb_solve_sharded_local_i32: the same kernel and the same stores, the
// replicas side by side in one allocation — the test and world-1 vehicle on a
// one-GPU box, where several kernels that wait on each other must not run as
// separate launches).
//
// Window of a rank: its replica (shard_rep_bytes) | home block: Ctrl, claims
// (n x u64), slab row minima (R x n x i32).  Only rank 0's home block is used.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "kmb.h"
#include "kmb_internal.h"

namespace kmb {
namespace {

int dfail(int code, const std::string& msg) {
  set_last_error(msg);
  return code;
}

size_t al256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

struct Plan {
  int W = 4, G = 0, Gr = 0, Gt = 0;
  int64_t slab_cols() const { return static_cast<int64_t>(Gr) * W; }
};

// The single-GPU engine's slab width and CTA count (kmb_capi.cu prepare_grid),
// the CTAs split evenly over the ranks; `max_total` bounds R * Gr (all ranks
// on one GPU: cooperative residency) or, per rank, Gr.
Plan make_plan(int n, int R, int max_ctas, bool one_gpu) {
  Plan p;
  for (;;) {
    p.G = (n + p.W - 1) / p.W;
    p.Gr = (p.G + R - 1) / R;
    p.Gt = p.Gr * R;
    const bool fits = one_gpu ? p.Gt <= max_ctas : (p.G <= max_ctas && p.Gr <= max_ctas);
    if (fits) return p;
    p.W <<= 1;
  }
}

size_t home_bytes(int n, int R) {
  return al256(sizeof(Ctrl)) + al256(8ull * n) + al256(4ull * R * n);
}

struct HomePtrs {
  Ctrl* ctrl;
  uint64_t* claim;
  int32_t* rowmin;
};
HomePtrs home_at(unsigned char* h, int n) {
  HomePtrs p;
  p.ctrl = reinterpret_cast<Ctrl*>(h);
  p.claim = reinterpret_cast<uint64_t*>(h + al256(sizeof(Ctrl)));
  p.rowmin = reinterpret_cast<int32_t*>(h + al256(sizeof(Ctrl)) + al256(8ull * n));
  return p;
}

}  // namespace

// Per-context state of the device-sharded solve (owned by the context).
struct ShardDevState {
  int device = 0;
  int R = 0, rank = 0, n = 0;
  bool local = false;  // all ranks on this GPU (one launch)
  Plan plan;
  size_t rep_bytes = 0;
  unsigned char* window = nullptr;  // own replica(s) + home block
  unsigned char* peer[KMB_MAX_RANKS] = {};
  bool ipc_open[KMB_MAX_RANKS] = {};
  int32_t* slab = nullptr;  // pitched copy of the caller's slab (all slabs when local)
  size_t slab_bytes = 0;
  int64_t* vbuf = nullptr;
  ShardDevArgs* args_dev = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~ShardDevState() {
    cudaSetDevice(device);
    for (int r = 0; r < KMB_MAX_RANKS; ++r)
      if (ipc_open[r]) cudaIpcCloseMemHandle(peer[r]);
    if (window) cudaFree(window);
    if (slab) cudaFree(slab);
    if (vbuf) cudaFree(vbuf);
    if (args_dev) cudaFree(args_dev);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
  unsigned char* home() const { return peer[0] + al256(rep_bytes); }
};

void destroy_shard_dev(ShardDevState* p) { delete p; }

namespace {

#define DEV_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t e__ = (call);                                                  \
    if (e__ != cudaSuccess)                                                    \
      return kmb::dfail(KMB_ECUDA, std::string(who) + ": " #call ": " + cudaGetErrorString(e__)); \
  } while (0)

// Allocate the window(s): one rank's (GPU ranks) or all R replicas + one home
// block (local).
int alloc_state(ShardDevState& s, int n, int R, int rank, bool local, int max_ctas, const char* who) {
  s.n = n;
  s.R = R;
  s.rank = rank;
  s.local = local;
  s.plan = make_plan(n, R, max_ctas, local);
  s.rep_bytes = shard_rep_bytes(n, s.plan.Gt);
  const size_t reps = local ? static_cast<size_t>(R) : 1;
  DEV_CUDA(cudaMalloc(&s.window, al256(s.rep_bytes) * reps + home_bytes(n, R)));
  if (local) {
    // replicas side by side; the home block after them (peer[0] + rep stride)
    for (int r = 0; r < R; ++r) s.peer[r] = s.window + al256(s.rep_bytes) * r;
  } else {
    s.peer[rank] = s.window;
  }
  DEV_CUDA(cudaMalloc(&s.args_dev, sizeof(ShardDevArgs)));
  DEV_CUDA(cudaMalloc(&s.vbuf, 8ull * (local ? s.plan.Gt : s.plan.Gr) * s.plan.W));
  DEV_CUDA(cudaEventCreate(&s.e0));
  DEV_CUDA(cudaEventCreate(&s.e1));
  return KMB_OK;
}

// GPU ranks: every rank reaches this host vote before launching, so a rank
// that failed locally (bad arguments, staging) makes every rank return an
// error instead of leaving the others' kernels waiting at the first barrier.
// Returns 0 when every rank is ready.
int vote(Exchange* ex, bool ok) {
  if (!ex || ex->nranks <= 1) return ok ? 0 : -1;
  int64_t x = ok ? 0 : -1;
  if (ex->allreduce_min(&x, 1) != 0) return -2;
  return x < 0 ? -1 : 0;
}

// Run the kernel over this process's ranks; slab pointers already staged.
int run(kmb_context* c, ShardDevState& s, int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
        int64_t* total_cost, kmb_stats* stats, const char* who, Exchange* ex) {
  cudaStream_t st = context_stream(c);
  const Plan& p = s.plan;
  const int n = s.n;
  // the local (emulated) layout keeps the home block after all replicas: for
  // the kernel rank 0's "window" extends over them, so home() is computed from
  // the last replica there
  unsigned char* home = s.local ? s.window + al256(s.rep_bytes) * s.R : s.home();
  const HomePtrs h = home_at(home, n);
  ShardDevArgs A{};
  A.R = s.R;
  A.rank_base = s.local ? 0 : s.rank;
  A.Gr = p.Gr;
  A.sys = s.local ? 0 : 1;
  A.slab_pitch = s.local ? static_cast<int64_t>(p.Gt) * p.W : p.slab_cols();
  for (int r = 0; r < s.R; ++r) {
    A.rep[r] = s.peer[r];
    if (s.local) {
      A.slab[r] = s.slab + p.slab_cols() * r;
      A.vout[r] = s.vbuf + p.slab_cols() * r;
    } else if (r == s.rank) {
      A.slab[r] = s.slab;
      A.vout[r] = s.vbuf;
    }
  }
  A.rowmin = h.rowmin;
  const bool staged = cudaMemcpyAsync(s.args_dev, &A, sizeof(A), cudaMemcpyHostToDevice, st) == cudaSuccess;
  SolverArgs a{};
  a.n = n;
  a.W = p.W;
  a.seed = seed;
  // prefetch appended rows into L2 when this rank's slab exceeds it (as the
  // single-GPU engine does)
  a.prefetch_rows = static_cast<double>(A.slab_pitch) * n * 4 > 96.0 * (1 << 20) ? 1 : 0;
  a.slab_cache = n <= 40960 ? 1 : 0;
  a.claim = h.claim;
  a.ctrl = h.ctrl;
  bool ready = staged && (!(s.local || s.rank == 0) || cudaMemsetAsync(h.ctrl, 0, sizeof(Ctrl), st) == cudaSuccess);
  ready = ready && cudaStreamSynchronize(st) == cudaSuccess;
  // GPU ranks: rank 0's reset of the home block precedes every launch, and
  // nobody launches unless everybody is ready
  if (int vr = vote(ex, ready)) {
    cudaGetLastError();
    return dfail(KMB_ECUDA, std::string(who) + (vr == -2 ? ": host barrier failed"
                                                : ready ? ": another rank failed before the solve"
                                                        : ": staging the solve failed"));
  }
  DEV_CUDA(cudaEventRecord(s.e0, st));
  DEV_CUDA(launch_solver_sharded(a, s.args_dev, s.local ? p.Gt : p.Gr, st));
  DEV_CUDA(cudaEventRecord(s.e1, st));
  Ctrl hc;
  DEV_CUDA(cudaMemcpyAsync(&hc, h.ctrl, sizeof(hc), cudaMemcpyDeviceToHost, st));
  const unsigned char* mine = s.local ? s.peer[0] : s.peer[s.rank];
  const size_t o32 = static_cast<size_t>((8ull * (3ull * n + p.Gt) + 15) & ~15ull);
  if (row_to_col)
    DEV_CUDA(cudaMemcpyAsync(row_to_col, mine + o32 + 4ull * n, 4ull * n, cudaMemcpyDefault, st));
  if (u) DEV_CUDA(cudaMemcpyAsync(u, mine, 8ull * n, cudaMemcpyDefault, st));
  const int64_t vcols = s.local ? n : std::min<int64_t>(p.slab_cols(), n - p.slab_cols() * s.rank);
  if (v && vcols > 0) DEV_CUDA(cudaMemcpyAsync(v, s.vbuf, 8ull * vcols, cudaMemcpyDefault, st));
  DEV_CUDA(cudaStreamSynchronize(st));
  if (s.local && s.R > 1) {
    // every replica must hold the same row side: u and the matching
    std::unique_ptr<unsigned char[]> a0(new unsigned char[o32 + 8ull * n]), ar(new unsigned char[o32 + 8ull * n]);
    DEV_CUDA(cudaMemcpy(a0.get(), s.peer[0], 8ull * n, cudaMemcpyDeviceToHost));
    DEV_CUDA(cudaMemcpy(a0.get() + o32, s.peer[0] + o32 + 4ull * n, 8ull * n, cudaMemcpyDeviceToHost));
    for (int r = 1; r < s.R; ++r) {
      DEV_CUDA(cudaMemcpy(ar.get(), s.peer[r], 8ull * n, cudaMemcpyDeviceToHost));
      DEV_CUDA(cudaMemcpy(ar.get() + o32, s.peer[r] + o32 + 4ull * n, 8ull * n, cudaMemcpyDeviceToHost));
      if (std::memcmp(a0.get(), ar.get(), 8ull * n) != 0 ||
          std::memcmp(a0.get() + o32, ar.get() + o32, 8ull * n) != 0)
        return dfail(KMB_EINTERNAL, std::string(who) + ": replica " + std::to_string(r) + " diverged");
    }
  }
  // GPU ranks: nobody resets the home block before everyone read it
  if (ex && ex->nranks > 1) {
    int64_t x = 0;
    if (ex->allreduce_min(&x, 1) != 0) return dfail(KMB_ECUDA, std::string(who) + ": host barrier failed");
  }
  if (hc.status == KMB_ENEGATIVE) return dfail(KMB_ENEGATIVE, std::string(who) + ": costs must be nonnegative");
  if (hc.status == KMB_ERANGE)
    return dfail(KMB_ERANGE, std::string(who) + ": cost exceeds the device range [0, 2^29)");
  if (hc.status == -3)
    return dfail(KMB_ECUDA, std::string(who) + ": a rank did not reach the barrier within 20 s");
  if (hc.status != 0) return dfail(KMB_EINTERNAL, std::string(who) + ": engine invariant violated");
  if (total_cost) *total_cost = static_cast<int64_t>(hc.obj);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->phases = hc.phases;
    stats->dual_steps = hc.dual_steps;
    stats->rows_scanned = hc.rows_scanned;
    stats->segment_rows = hc.seg_rows;
    stats->rounds = hc.rounds;
    stats->cost_bytes_read = 4ll * n * (hc.rows_scanned + (seed == KMB_SEED_BATCHED ? n : 0)) + 16ll * hc.seg_rows;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s.e0, s.e1);
    stats->seconds = ms * 1e-3;
    stats->converged = hc.free_rows == 0 ? 1 : 0;
    stats->engine = 10;
    for (int k = 0; k < 6; ++k) stats->stage_ns[k] = hc.stage_ns[k];
  }
  return KMB_OK;
}

}  // namespace
}  // namespace kmb

extern "C" {

int kmb_solve_sharded_local_i32(kmb_context* c, const int32_t* cost, int32_t n, int64_t ld,
                                int32_t nranks, int32_t seed, int32_t* row_to_col, int64_t* u,
                                int64_t* v, int64_t* total_cost, kmb_stats* stats) {
  const char* who = "kmb_solve_sharded_local_i32";
  if (!c) return kmb::dfail(KMB_EINVAL, std::string(who) + ": NULL context");
  if (n <= 0 || !cost || ld < n || nranks < 1 || nranks > kmb::KMB_MAX_RANKS ||
      (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED))
    return kmb::dfail(KMB_EINVAL, std::string(who) + ": bad arguments");
  cudaSetDevice(kmb::context_device(c));
  auto& sp = kmb::context_shard_dev(c);
  if (!sp || !sp->local || sp->n != n || sp->R != nranks) {
    sp.reset(new kmb::ShardDevState());
    sp->device = kmb::context_device(c);
    if (int r = kmb::alloc_state(*sp, n, nranks, 0, true, kmb::context_sm_count(c), who)) {
      sp.reset();
      return r;
    }
  }
  kmb::ShardDevState& s = *sp;
  const kmb::Plan& p = s.plan;
  // the whole matrix, pitched: rank r's slab is columns [r * Gr * W, ...)
  const int64_t pitch = static_cast<int64_t>(p.Gt) * p.W;
  const size_t need = static_cast<size_t>(n) * pitch * 4;
  if (s.slab_bytes < need) {
    if (s.slab) cudaFree(s.slab);
    s.slab = nullptr;
    s.slab_bytes = 0;
    DEV_CUDA(cudaMalloc(&s.slab, need));
    s.slab_bytes = need;
  }
  cudaStream_t st = kmb::context_stream(c);
  DEV_CUDA(cudaMemsetAsync(s.slab, 0, need, st));
  DEV_CUDA(cudaMemcpy2DAsync(s.slab, pitch * 4, cost, ld * 4, static_cast<size_t>(n) * 4, n,
                             cudaMemcpyDefault, st));
  return kmb::run(c, s, seed, row_to_col, u, v, total_cost, stats, who, nullptr);
}

int kmb_shard_dev_open(kmb_context* c, int32_t n, int32_t nranks, int32_t rank, int32_t* slab_cols,
                       uint8_t* handle64) {
  const char* who = "kmb_shard_dev_open";
  if (!c || n <= 0 || nranks < 1 || nranks > kmb::KMB_MAX_RANKS || rank < 0 || rank >= nranks)
    return kmb::dfail(KMB_EINVAL, std::string(who) + ": bad arguments");
  cudaSetDevice(kmb::context_device(c));
  auto& sp = kmb::context_shard_dev(c);
  sp.reset(new kmb::ShardDevState());
  sp->device = kmb::context_device(c);
  if (int r = kmb::alloc_state(*sp, n, nranks, rank, false, kmb::context_sm_count(c), who)) {
    sp.reset();
    return r;
  }
  if (slab_cols) *slab_cols = static_cast<int32_t>(sp->plan.slab_cols());
  if (handle64) {
    cudaIpcMemHandle_t h;
    DEV_CUDA(cudaIpcGetMemHandle(&h, sp->window));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle64, &h, 64);
  }
  return KMB_OK;
}

int kmb_shard_dev_connect(kmb_context* c, const uint8_t* handles64) {
  const char* who = "kmb_shard_dev_connect";
  if (!c) return kmb::dfail(KMB_EINVAL, std::string(who) + ": NULL context");
  auto& sp = kmb::context_shard_dev(c);
  if (!sp || sp->local) return kmb::dfail(KMB_EINVAL, std::string(who) + ": call kmb_shard_dev_open first");
  cudaSetDevice(kmb::context_device(c));
  kmb::ShardDevState& s = *sp;
  for (int r = 0; r < s.R; ++r) {
    if (r == s.rank || s.ipc_open[r]) continue;
    if (!handles64) return kmb::dfail(KMB_EINVAL, std::string(who) + ": handles is NULL");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles64 + 64ull * r, 64);
    void* p = nullptr;
    DEV_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    s.peer[r] = static_cast<unsigned char*>(p);
    s.ipc_open[r] = true;
  }
  return KMB_OK;
}

int kmb_solve_sharded_dev_i32(kmb_context* c, const int32_t* slab, int32_t n, int64_t ld,
                              int32_t col_begin, int32_t ncols, int32_t seed, int32_t* row_to_col,
                              int64_t* u, int64_t* v_slab, int64_t* total_cost, kmb_stats* stats) {
  const char* who = "kmb_solve_sharded_dev_i32";
  if (!c) return kmb::dfail(KMB_EINVAL, std::string(who) + ": NULL context");
  auto& sp = kmb::context_shard_dev(c);
  if (!sp || sp->local) return kmb::dfail(KMB_EINVAL, std::string(who) + ": call kmb_shard_dev_open first");
  kmb::ShardDevState& s = *sp;
  auto& ex = kmb::context_exchange(c);
  if (s.R > 1 && !ex) return kmb::dfail(KMB_EINVAL, std::string(who) + ": call kmb_shard_init_* first");
  // a rank-local argument error is voted on, so the other ranks return too
  for (int r = 0; r < s.R; ++r)
    if (!s.peer[r]) {
      kmb::vote(ex.get(), false);
      return kmb::dfail(KMB_EINVAL, std::string(who) + ": call kmb_shard_dev_connect first");
    }
  const int64_t w = s.plan.slab_cols();
  const int64_t want = std::max<int64_t>(0, std::min<int64_t>(w, n - w * s.rank));
  if (n != s.n || col_begin != w * s.rank || ncols != want || !slab || ld < ncols ||
      (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED)) {
    kmb::vote(ex.get(), false);
    return kmb::dfail(KMB_EINVAL, std::string(who) + ": bad arguments (rank r holds columns [r * slab_cols, ...))");
  }
  cudaSetDevice(kmb::context_device(c));
  // staging failures are voted on in run()'s pre-launch barrier like any other
  const size_t need = static_cast<size_t>(n) * w * 4;
  cudaError_t e = cudaSuccess;
  if (s.slab_bytes < need) {
    if (s.slab) cudaFree(s.slab);
    s.slab = nullptr;
    s.slab_bytes = 0;
    e = cudaMalloc(&s.slab, need);
    if (e == cudaSuccess) s.slab_bytes = need;
  }
  cudaStream_t st = kmb::context_stream(c);
  if (e == cudaSuccess) e = cudaMemsetAsync(s.slab, 0, need, st);
  if (e == cudaSuccess && ncols > 0)
    e = cudaMemcpy2DAsync(s.slab, w * 4, slab, ld * 4, static_cast<size_t>(ncols) * 4, n, cudaMemcpyDefault, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    kmb::vote(ex.get(), false);
    return kmb::dfail(KMB_ECUDA, std::string(who) + ": staging the slab: " + cudaGetErrorString(e));
  }
  return kmb::run(c, s, seed, row_to_col, u, v_slab, total_cost, stats, who, ex.get());
}

}  // extern "C"
