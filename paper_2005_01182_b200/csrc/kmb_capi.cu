// C ABI of include/kmb.h: context, device workspace, engine selection, host <->
// device staging.  Host code only; the kernels live in kmb_solver.cu (grid
// engine) and kmb_batch.cu (SMEM engine).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "kmb.h"
#include "kmb_internal.h"
#include "kmb_stage.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(KMB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define KMB_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e__ = (call);                           \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, need);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

struct kmb_context {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t max_ctas = 0;
  int64_t warps_per_sm = 0;  // warp engine residency bound (0 = occupancy limit)
  int64_t pipeline = 0;      // host-input batches: chunk schedule (0 = tapered auto)
  int64_t resident16 = 0;    // warp engine 16-bit resident copy (0 auto, 1 on, -1 off)
  int engine = 0;
  int64_t last_batch = 0;  // instances of the last batch solve (kmb_last_instance_stats)
  // grid-engine workspace
  DevBuf cost, u, v, mrow, mcol, tpar, root, claim, lrow0, lrow1, lw0, lw1, found, partial,
      ctrl, obj;
  // batch workspace
  DevBuf bcost, bpad, br2c, bu, bv, btot, bstat, bstatus, b16;
  // cost construction workspace (host-resident points / output)
  DevBuf pa, pb, pout, pbad;
  // auction workspace
  DevBuf aprice, ar2c, atot, abids, acomp, aeps, amin, amax;
  // 64-bit cost path: staged costs, chat, narrowed costs, min/max + lossy flag,
  // device-side results, wide-engine slots
  DevBuf w64in, wchat, wnar, wmm, wr2c, wu, wv, wtot, wws64, wws32;
  // batch summary (device fold + pinned host copy)
  DevBuf bsum;
  int64_t* hsum = nullptr;
  // column-sharded solve: the collective (NCCL or caller callbacks)
  std::unique_ptr<kmb::Exchange> exchange;
  // device-resident column-sharded solve (replicas, IPC mappings)
  kmb::ShardDevPtr shard_dev;
  // pageable host buffers: pinned staging ring + copy threads (kmb_stage.h)
  std::unique_ptr<kmb::HostStager> stager;
  // chunked host-input pipeline of the batch engines
  static constexpr int kAux = 4, kMaxChunks = 64;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t aux_ev[kAux] = {};
  cudaStream_t cin = nullptr;             // H2D copies of the chunks, in order
  cudaEvent_t in_ev[kMaxChunks] = {};     // chunk k landed
};

namespace kmb {
std::unique_ptr<Exchange>& context_exchange(kmb_context* c) { return c->exchange; }
ShardDevPtr& context_shard_dev(kmb_context* c) { return c->shard_dev; }
int context_sm_count(kmb_context* c) { return c->sm_count; }
cudaStream_t context_stream(kmb_context* c) { return c->stream; }
int context_device(kmb_context* c) { return c->device; }
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace kmb

extern "C" {

const char* kmb_last_error(void) { return g_err.c_str(); }
int kmb_abi_version(void) { return KMB_ABI_VERSION; }

int kmb_create(int device, kmb_context** out) {
  if (!out) return fail(KMB_EINVAL, "kmb_create: out is NULL");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count <= device || device < 0)
    return fail(KMB_ENODEVICE, std::string("kmb_create: no CUDA device ") + std::to_string(device) +
                                   (e != cudaSuccess ? std::string(" (") + cudaGetErrorString(e) + ")"
                                                     : std::string()));
  cudaDeviceProp prop;
  KMB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(KMB_ENODEVICE, std::string("kmb_create: device is sm_") + std::to_string(prop.major) +
                                   std::to_string(prop.minor) + ", this build targets sm_100a");
  KMB_CUDA(cudaSetDevice(device));
  kmb_context* c = new kmb_context();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);
  *out = c;
  return KMB_OK;
}

void kmb_destroy(kmb_context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  c->shard_dev.reset();
  c->stager.reset();
  for (DevBuf* b : {&c->cost, &c->u, &c->v, &c->mrow, &c->mcol, &c->tpar, &c->root, &c->claim,
                    &c->lrow0, &c->lrow1, &c->lw0, &c->lw1, &c->found, &c->partial, &c->ctrl,
                    &c->obj, &c->bcost, &c->bpad, &c->br2c, &c->bu, &c->bv, &c->btot, &c->bstat,
                    &c->bstatus, &c->b16, &c->pa, &c->pb, &c->pout, &c->pbad, &c->aprice, &c->ar2c, &c->atot,
                    &c->abids, &c->acomp, &c->aeps, &c->amin, &c->amax, &c->bsum, &c->w64in, &c->wchat,
                    &c->wnar, &c->wmm, &c->wr2c, &c->wu, &c->wv, &c->wtot, &c->wws64, &c->wws32})
    b->release();
  if (c->hsum) cudaFreeHost(c->hsum);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (int k = 0; k < kmb_context::kAux; ++k) {
    if (c->aux_ev[k]) cudaEventDestroy(c->aux_ev[k]);
    if (c->aux[k]) cudaStreamDestroy(c->aux[k]);
  }
  for (int k = 0; k < kmb_context::kMaxChunks; ++k)
    if (c->in_ev[k]) cudaEventDestroy(c->in_ev[k]);
  if (c->cin) cudaStreamDestroy(c->cin);
  delete c;
}

int kmb_set_stream(kmb_context* c, void* s) {
  if (!c) return fail(KMB_EINVAL, "kmb_set_stream: NULL context");
  c->stream = static_cast<cudaStream_t>(s);
  return KMB_OK;
}

int kmb_set_option(kmb_context* c, int option, int64_t value) {
  if (!c) return fail(KMB_EINVAL, "kmb_set_option: NULL context");
  switch (option) {
    case KMB_OPT_MAX_CTAS: c->max_ctas = value; return KMB_OK;
    case KMB_OPT_WARPS_PER_SM: c->warps_per_sm = value; return KMB_OK;
    case KMB_OPT_RESIDENT16:
      if (value < -1 || value > 1) return fail(KMB_EINVAL, "kmb_set_option: resident16 must be -1, 0 or 1");
      c->resident16 = value;
      return KMB_OK;
    case KMB_OPT_PIPELINE:
      if (value < -(kmb_context::kMaxChunks / 2) || value > kmb_context::kMaxChunks)
        return fail(KMB_EINVAL, "kmb_set_option: pipeline chunk count out of range");
      c->pipeline = value;
      return KMB_OK;
    case KMB_OPT_ENGINE:
      if (value < 0 || value > 11 || value == 2 || value == 3 || value == 7 || value == 9 || value == 10)
        return fail(KMB_EINVAL, "kmb_set_option: engine must be 0, 1, 4, 5, 6, 8 or 11");
      c->engine = static_cast<int>(value);
      return KMB_OK;
    default: return fail(KMB_EINVAL, "kmb_set_option: unknown option");
  }
}

static int copy_out(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!dst || bytes == 0) return KMB_OK;
  KMB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  return KMB_OK;
}

static int status_message(int status, const char* who) {
  if (status == KMB_ENEGATIVE) return fail(status, std::string(who) + ": costs must be nonnegative");
  if (status == KMB_ERANGE)
    return fail(status, std::string(who) + ": cost exceeds the device range [0, 2^29)");
  return fail(KMB_EINTERNAL, std::string(who) + ": engine invariant violated (status " +
                                 std::to_string(status) + ")");
}

#ifndef KMB_TAPER_MIN  // the tapered schedule halves the last chunk down to this size
#define KMB_TAPER_MIN 64
#endif

// instance status of a time budget that expired (single-CTA engine): not an error
constexpr int64_t kStopped = 4;

static int solve_batch_impl(kmb_context* c, const int32_t* costs, int32_t batch, int32_t n,
                            int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
                            int64_t* total_cost, kmb_stats* stats, const char* who, int engine,
                            double time_budget_s = 0.0, int32_t* async_status = nullptr) {
  cudaStream_t st = c->stream;
  const size_t cbytes = static_cast<size_t>(batch) * n * n * sizeof(int32_t);
  // auto: a batch (or pipeline chunk) that fits the CTA engine's residency in
  // one wave runs one CTA per instance (shorter rounds: 0.38 vs 0.47 ms for a
  // 512-instance config-3 shard); larger batches one warp per instance, all
  // resident (0.78 ms at 4096 vs 1.7 for CTAs).  The warp engine is ahead from
  // ~11/12 of that residency on (config 3, warp / CTA: 1,024 0.479 / 0.469 ms,
  // 1,184 0.473 / 0.493)
  const bool auto_engine = engine == 0 || engine == 1 || engine == 5;
  const int cap6 = auto_engine ? kmb::cta_batch_capacity(n, c->sm_count) : 0;
  // n > 256: one 512-thread CTA per instance (single-CTA engine, n <= 4096),
  // or, for up to #SMs / 32 instances with 1792 < n <= 4608, one replicated
  // 16-CTA cluster each (4 x n = 3072: 43.6 -> 26.0 ms; at 9 clusters the
  // single-CTA engine is ahead again: 9 x n = 2500 38.5 vs 40.9 ms)
  auto pick = [&](int cnt) {
    if (n <= kmb::warp_max_n()) return cnt * 12 <= cap6 * 11 ? 6 : 4;
    return (n > 1792 && n <= 4608 && cnt * 32 <= c->sm_count) ? 11 : 8;
  };
  if (auto_engine) engine = pick(batch);
  // Host input: stream the batch in chunks, each chunk's kernel starting as soon
  // as its H2D copy lands and its results leaving as soon as it ends, so the
  // PCIe transfers overlap the solves (the transfer bounds the end-to-end rate).
  const bool host_in = !is_device_ptr(costs);
  const bool warp_eng = engine == 4;
  // row pitch of the vector-load engines: the warp engine's 128-bit loads need
  // rows padded to the warp width, the single-CTA engine's (up to 128-bit)
  // loads a pitch that is a multiple of 4; both a 16-byte aligned base.  A
  // buffer that is neither is copied into the aligned, padded workspace (a
  // misaligned vector load would fault).
  const bool vec_eng = warp_eng || engine == 8;
  const int np = warp_eng ? kmb::warp_pitch(n) : engine == 8 ? (n + 3) & ~3 : n;
  const bool repack = vec_eng && (np != n || (!host_in && (reinterpret_cast<uintptr_t>(costs) & 15) != 0));
  const bool pipelined = host_in && batch >= 256 && np == n;
  // chunk schedule [lo, lo + cnt): K equal chunks, and (tapered) the last one
  // split by halving down to KMB_TAPER_MIN instances, so the solve left after the final
  // copy lands is a short one
  std::vector<std::pair<int, int>> sched;
  if (pipelined) {
    const int64_t opt = c->pipeline;
    const int K = opt > 0 ? static_cast<int>(std::min<int64_t>(opt, batch))
                          : opt < 0 ? std::min<int>(static_cast<int>(-opt), batch / 64)
                                    : std::max(2, std::min(8, batch / 128));
    const bool taper = opt <= 0;
    const int chunk = (batch + K - 1) / K;
    int lo = 0;
    for (int k = 0; k < K && lo < batch; ++k) {
      int cnt = std::min(chunk, batch - lo);
      if (taper && lo + cnt >= batch) {  // the last chunk: halve it down
        while (cnt > KMB_TAPER_MIN && static_cast<int>(sched.size()) < kmb_context::kMaxChunks - 1) {
          const int h = cnt / 2;
          sched.emplace_back(lo, h);
          lo += h;
          cnt -= h;
        }
      }
      sched.emplace_back(lo, cnt);
      lo += cnt;
    }
  }
  const int32_t* dcost = costs;
  if (host_in) {
    KMB_CUDA(c->bcost.ensure(cbytes));
    dcost = c->bcost.as<int32_t>();
  }
  const size_t nb = static_cast<size_t>(batch) * n;
  int32_t* dr2c = row_to_col;
  int64_t *du = u, *dv = v, *dtot = total_cost;
  if (!is_device_ptr(row_to_col)) { KMB_CUDA(c->br2c.ensure(nb * 4)); dr2c = c->br2c.as<int32_t>(); }
  if (!is_device_ptr(u)) { KMB_CUDA(c->bu.ensure(nb * 8)); du = c->bu.as<int64_t>(); }
  if (!is_device_ptr(v)) { KMB_CUDA(c->bv.ensure(nb * 8)); dv = c->bv.as<int64_t>(); }
  if (!is_device_ptr(total_cost)) { KMB_CUDA(c->btot.ensure(batch * 8)); dtot = c->btot.as<int64_t>(); }
  KMB_CUDA(c->bstat.ensure(static_cast<size_t>(batch) * kmb::KMB_ISTATS * 8));
  c->last_batch = batch;
  KMB_CUDA(c->bstatus.ensure(static_cast<size_t>(batch) * 4));
  // stream-ordered calls write the statuses straight into the caller's buffer
  int32_t* const status_base = async_status ? async_status : c->bstatus.as<int32_t>();
  const int32_t* src = dcost;  // vector-load engines: rows padded to np
  // warp engine: 16-bit resident copy of the rows (KMB_OPT_RESIDENT16)
  // decided per launch (a pipelined call's chunks are launches of their own)
  uint16_t* c16 = nullptr;
  auto want16 = [&](int cnt) {
    if (n <= 64 || n > kmb::warp_max_n()) return false;
    const size_t mat_bytes = static_cast<size_t>(cnt) * n * np * 4;
    // auto (measured on one B200, ms without / with the copy):
    //  n > 128 (8 columns a lane): from 128 MiB of matrices up - n = 256 x 700
    //    1.22 / 1.11, x 1,024 1.49 / 1.22, x 4,096 5.63 / 2.89; n = 200 x 2,000
    //    1.62 / 1.24; n = 160 x 4,096 2.43 / 1.60;
    //  n <= 128: between 1.5 x the L2 and 448 MiB - config 3 (64 KiB matrices)
    //    x 2,560 0.721 / 0.747, x 3,072 0.785 / 0.772, x 3,584 0.856 / 0.821,
    //    x 4,096 0.956 / 0.899, x 6,000 1.452 / 1.370, x 8,192 1.753 / 1.790
    //    (instances that start later pack while the others search); uniform
    //    U{0..50000} x 4,096 0.603 / 0.592, x 8,192 1.092 / 1.194.
    // Instances whose rows do not fit 16 bits fall back per instance.
    const size_t mib = static_cast<size_t>(1) << 20;
    const bool auto16 = n > 128 ? mat_bytes >= 128 * mib : (mat_bytes >= 192 * mib && mat_bytes < 448 * mib);
    return c->resident16 > 0 || (c->resident16 == 0 && auto16);
  };
  {
    bool any16 = false;  // does any launch of this call run the warp engine with the copy?
    if (sched.empty()) {
      any16 = warp_eng && want16(batch);
    } else {
      for (const auto& ch : sched) any16 = any16 || ((auto_engine ? pick(ch.second) : engine) == 4 && want16(ch.second));
    }
    if (any16) {
      KMB_CUDA(c->b16.ensure(nb * np * 2));
      c16 = c->b16.as<uint16_t>();
    }
  }
  int grid = 0;
  // the chunks of a pipelined call size their carveout for the largest chunk
  const int carve_batch = sched.empty() ? 0 : sched[0].second;
  // instances [lo, lo + cnt) on engine eng, stream s
  auto launch = [&](int lo, int cnt, int eng, cudaStream_t s) -> cudaError_t {
    const size_t ro = static_cast<size_t>(lo) * n;
    if (eng == 11) {  // replicated cluster engine: one <=16-CTA cluster per instance
      kmb::BigArgs a{};
      a.C = dcost + ro * n;
      a.ld = n;
      a.inst_stride = static_cast<int64_t>(n) * n;
      a.batch = cnt;
      a.n = n;
      a.seed = seed;
      a.deadline_ns = time_budget_s > 0.0 ? static_cast<int64_t>(time_budget_s * 1e9) : 0;
      a.row_to_col = dr2c + ro;
      a.u = du + ro;
      a.v = dv + ro;
      a.total_cost = dtot + lo;
      a.stats = c->bstat.as<int64_t>() + static_cast<size_t>(lo) * kmb::KMB_ISTATS;
      a.status = status_base + lo;
      const int G = c->max_ctas > 0 ? static_cast<int>(std::min<int64_t>(c->max_ctas, 16)) : 16;
      return kmb::launch_cluster(a, G, c->sm_count, s);
    }
    if (eng == 8) {
      kmb::BigArgs a{};
      a.C = src + ro * np;
      a.ld = np;
      a.inst_stride = static_cast<int64_t>(n) * np;
      a.batch = cnt;
      a.n = n;
      a.seed = seed;
      a.deadline_ns = time_budget_s > 0.0 ? static_cast<int64_t>(time_budget_s * 1e9) : 0;
      a.row_to_col = dr2c + ro;
      a.u = du + ro;
      a.v = dv + ro;
      a.total_cost = dtot + lo;
      a.stats = c->bstat.as<int64_t>() + static_cast<size_t>(lo) * kmb::KMB_ISTATS;
      a.status = status_base + lo;
      a.carve_batch = carve_batch;
      return kmb::launch_big(a, c->sm_count, s);
    }
    if (eng == 6) {
      kmb::BatchArgs a{};
      a.C = dcost + ro * n;
      a.batch = cnt;
      a.n = n;
      a.seed = seed;
      a.row_to_col = dr2c + ro;
      a.u = du + ro;
      a.v = dv + ro;
      a.total_cost = dtot + lo;
      a.stats = c->bstat.as<int64_t>() + static_cast<size_t>(lo) * kmb::KMB_ISTATS;
      a.status = status_base + lo;
      a.carve_batch = carve_batch;
      return kmb::launch_batch(a, c->sm_count, static_cast<int>(c->warps_per_sm), s, &grid);
    }
    kmb::WarpArgs a{};
    a.C = src + ro * np;
    a.batch = cnt;
    a.n = n;
    a.pitch = np;
    a.seed = seed;
    a.row_to_col = dr2c + ro;
    a.u = du + ro;
    a.v = dv + ro;
    a.total_cost = dtot + lo;
    a.stats = c->bstat.as<int64_t>() + static_cast<size_t>(lo) * kmb::KMB_ISTATS;
    a.status = status_base + lo;
    a.C16 = c16 && want16(cnt) ? c16 + ro * np : nullptr;
    return kmb::launch_warp_batch(a, c->sm_count, static_cast<int>(c->warps_per_sm), s, &grid);
  };
  // Pageable host memory (numpy arrays, std::vectors): the costs are staged
  // through pinned slots by the copy threads, and results bound for pageable
  // arrays land in a pinned buffer first (a D2H into pageable memory blocks
  // the host until the stream reaches it, which would serialise the chunks).
  const bool page_in = host_in && !async_status && !kmb::is_pinned_host(costs);
  int32_t* orow = row_to_col;
  int64_t *ou = u, *ov = v, *otot = total_cost;
  const bool pg_row = row_to_col && dr2c != row_to_col && !kmb::is_pinned_host(row_to_col);
  const bool pg_u = u && du != u && !kmb::is_pinned_host(u);
  const bool pg_v = v && dv != v && !kmb::is_pinned_host(v);
  const bool pg_tot = total_cost && dtot != total_cost && !kmb::is_pinned_host(total_cost);
  if (page_in || pg_row || pg_u || pg_v || pg_tot) {
    if (!c->stager) c->stager = std::make_unique<kmb::HostStager>();
  }
  if (pg_row || pg_u || pg_v || pg_tot) {
    unsigned char* pb = nullptr;
    KMB_CUDA(c->stager->out_buffer(nb * 20 + static_cast<size_t>(batch) * 8, &pb));
    if (pg_u) ou = reinterpret_cast<int64_t*>(pb);
    if (pg_v) ov = reinterpret_cast<int64_t*>(pb + nb * 8);
    if (pg_tot) otot = reinterpret_cast<int64_t*>(pb + nb * 16);
    if (pg_row) orow = reinterpret_cast<int32_t*>(pb + nb * 16 + static_cast<size_t>(batch) * 8);
  }
  // results of instances [lo, lo + cnt) to the caller's host buffers
  auto results_out = [&](int lo, int cnt, cudaStream_t s) -> cudaError_t {
    const size_t ro = static_cast<size_t>(lo) * n, rn = static_cast<size_t>(cnt) * n;
    cudaError_t e = cudaSuccess;
    if (dr2c != row_to_col && row_to_col)
      e = cudaMemcpyAsync(orow + ro, dr2c + ro, rn * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && du != u && u) e = cudaMemcpyAsync(ou + ro, du + ro, rn * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dv != v && v) e = cudaMemcpyAsync(ov + ro, dv + ro, rn * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dtot != total_cost && total_cost)
      e = cudaMemcpyAsync(otot + lo, dtot + lo, static_cast<size_t>(cnt) * 8, cudaMemcpyDeviceToHost, s);
    return e;
  };
  int used = engine;
  if (async_status) {  // stream-ordered: enqueue and return (device buffers only)
    if (repack) {
      KMB_CUDA(c->bpad.ensure(nb * np * 4));
      KMB_CUDA(cudaMemcpy2DAsync(c->bpad.p, np * 4, dcost, n * 4, n * 4, nb, cudaMemcpyDeviceToDevice, st));
      src = c->bpad.as<int32_t>();
    }
    KMB_CUDA(launch(0, batch, engine, st));
    return KMB_OK;
  }
  KMB_CUDA(cudaEventRecord(c->ev0, st));
  if (!pipelined) {
    if (page_in) KMB_CUDA(c->stager->h2d(c->bcost.p, costs, cbytes, st));
    else if (host_in) KMB_CUDA(cudaMemcpyAsync(c->bcost.p, costs, cbytes, cudaMemcpyHostToDevice, st));
    if (repack) {  // rows padded to np (in-bounds, aligned vector loads): pad once
      KMB_CUDA(c->bpad.ensure(nb * np * 4));
      KMB_CUDA(cudaMemcpy2DAsync(c->bpad.p, np * 4, dcost, n * 4, n * 4, nb, cudaMemcpyDeviceToDevice, st));
      src = c->bpad.as<int32_t>();
    }
    KMB_CUDA(launch(0, batch, engine, st));
    KMB_CUDA(cudaEventRecord(c->ev1, st));
    KMB_CUDA(results_out(0, batch, st));
  } else {
    if (!c->aux[0]) {
      for (int k = 0; k < kmb_context::kAux; ++k) {
        KMB_CUDA(cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking));
        KMB_CUDA(cudaEventCreateWithFlags(&c->aux_ev[k], cudaEventDisableTiming));
      }
    }
    if (!c->cin) {
      KMB_CUDA(cudaStreamCreateWithFlags(&c->cin, cudaStreamNonBlocking));
      for (int k = 0; k < kmb_context::kMaxChunks; ++k)
        KMB_CUDA(cudaEventCreateWithFlags(&c->in_ev[k], cudaEventDisableTiming));
    }
    // copies in order on one stream; chunk k's solve and result copies on an
    // auxiliary stream once its copy has landed (solves of successive chunks
    // may overlap each other; the D2H engine runs beside the H2D one)
    KMB_CUDA(cudaStreamWaitEvent(c->cin, c->ev0, 0));
    auto copy_in = [&](size_t k) -> cudaError_t {
      const int lo = sched[k].first, cnt = sched[k].second;
      const size_t off = static_cast<size_t>(lo) * n * n, len = static_cast<size_t>(cnt) * n * n * 4;
      cudaError_t e = page_in ? c->stager->h2d(c->bcost.as<int32_t>() + off, costs + off, len, c->cin)
                              : cudaMemcpyAsync(c->bcost.as<int32_t>() + off, costs + off, len,
                                                cudaMemcpyHostToDevice, c->cin);
      return e == cudaSuccess ? cudaEventRecord(c->in_ev[k], c->cin) : e;
    };
    // pinned input: every copy enqueued up front; pageable: the host stages
    // chunk k + 1 while chunk k's copy and solve run
    if (!page_in)
      for (size_t k = 0; k < sched.size(); ++k) KMB_CUDA(copy_in(k));
    for (size_t k = 0; k < sched.size(); ++k) {
      if (page_in) KMB_CUDA(copy_in(k));
      const int lo = sched[k].first, cnt = sched[k].second;
      cudaStream_t s2 = c->aux[k % kmb_context::kAux];
      KMB_CUDA(cudaStreamWaitEvent(s2, c->in_ev[k], 0));
      const int eng = auto_engine ? pick(cnt) : engine;  // chunks are small: CTA engine
      if (k == 0) used = eng;
      KMB_CUDA(launch(lo, cnt, eng, s2));
      KMB_CUDA(results_out(lo, cnt, s2));
    }
    for (int k = 0; k < kmb_context::kAux; ++k) {
      KMB_CUDA(cudaEventRecord(c->aux_ev[k], c->aux[k]));
      KMB_CUDA(cudaStreamWaitEvent(st, c->aux_ev[k], 0));
    }
    KMB_CUDA(cudaEventRecord(c->ev1, st));  // includes the transfers
  }
  engine = used;
  // status is always checked: invalid input must not pass silently.  Status and
  // per-instance stats are folded on the device; one small copy comes back.
  KMB_CUDA(c->bsum.ensure(16 * 8));
  if (!c->hsum) KMB_CUDA(cudaMallocHost(&c->hsum, 16 * 8));
  KMB_CUDA(kmb::launch_batch_summary(c->bstat.as<int64_t>(), c->bstatus.as<int32_t>(), batch,
                                     c->bsum.as<int64_t>(), st));
  KMB_CUDA(cudaMemcpyAsync(c->hsum, c->bsum.p, 11 * 8, cudaMemcpyDeviceToHost, st));
  {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, who);
  }
  if (pg_u) c->stager->memcpy_par(u, ou, nb * 8);
  if (pg_v) c->stager->memcpy_par(v, ov, nb * 8);
  if (pg_row) c->stager->memcpy_par(row_to_col, orow, nb * 4);
  if (pg_tot) std::memcpy(total_cost, otot, static_cast<size_t>(batch) * 8);
  const int64_t* h = c->hsum;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->phases = h[1];
    stats->dual_steps = h[2];
    stats->rows_scanned = h[3];
    stats->rounds = h[4];
    stats->sum_instance_cycles = h[5];
    stats->max_instance_cycles = h[6];
    for (int k = 0; k < 4; ++k) stats->stage_ns[k] = h[7 + k];  // batch: SM cycles, summed
    stats->cost_bytes_read = static_cast<int64_t>(batch) * n * n * 4;  // HBM: each matrix once
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    stats->seconds = ms * 1e-3;
    stats->converged = h[0] == kStopped ? 0 : 1;
    stats->engine = engine;
  }
  if (h[0] && h[0] != kStopped) return status_message(static_cast<int>(h[0]), who);
  return KMB_OK;
}

int kmb_solve_batch_i32(kmb_context* c, const int32_t* costs, int32_t batch, int32_t n,
                        int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
                        int64_t* total_cost, kmb_stats* stats) {
  const char* who = "kmb_solve_batch_i32";
  if (!c) return fail(KMB_EINVAL, "kmb_solve_batch_i32: NULL context");
  if (batch <= 0 || n <= 0) return fail(KMB_EINVAL, "kmb_solve_batch_i32: dimensions must be positive");
  if (!costs) return fail(KMB_EINVAL, "kmb_solve_batch_i32: costs is NULL");
  if (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED) return fail(KMB_EINVAL, "kmb_solve_batch_i32: bad seed");
  if (n > kmb::big_max_n())
    return fail(KMB_EINVAL, "kmb_solve_batch_i32: n > " + std::to_string(kmb::big_max_n()) +
                                " (use kmb_solve_i32 per instance)");
  if (n > kmb::warp_max_n() && c->engine != 0 && c->engine != 8 && c->engine != 11)
    return fail(KMB_EINVAL, "kmb_solve_batch_i32: n > 256 needs the single-CTA (8) or cluster (11) engine");
  if (c->engine == 11 && n > kmb::cluster_max_n())
    return fail(KMB_EINVAL, "kmb_solve_batch_i32: engine 11 takes n <= " + std::to_string(kmb::cluster_max_n()));
  KMB_CUDA(cudaSetDevice(c->device));
  return solve_batch_impl(c, costs, batch, n, seed, row_to_col, u, v, total_cost, stats, who,
                          c->engine);
}

// Stream-ordered batch solve (graph-capturable once the workspace is sized):
// device buffers only, no host synchronisation, per-instance statuses to the
// caller's device buffer.
int kmb_solve_batch_async_i32(kmb_context* c, const int32_t* costs, int32_t batch, int32_t n,
                              int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
                              int64_t* total_cost, int32_t* status) {
  const char* who = "kmb_solve_batch_async_i32";
  if (!c) return fail(KMB_EINVAL, std::string(who) + ": NULL context");
  if (batch <= 0 || n <= 0) return fail(KMB_EINVAL, std::string(who) + ": dimensions must be positive");
  if (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED) return fail(KMB_EINVAL, std::string(who) + ": bad seed");
  if (n > kmb::big_max_n())
    return fail(KMB_EINVAL, std::string(who) + ": n > " + std::to_string(kmb::big_max_n()));
  if (n > kmb::warp_max_n() && c->engine != 0 && c->engine != 8 && c->engine != 11)
    return fail(KMB_EINVAL, std::string(who) + ": n > 256 needs the single-CTA (8) or cluster (11) engine");
  KMB_CUDA(cudaSetDevice(c->device));
  for (const void* p : {static_cast<const void*>(costs), static_cast<const void*>(row_to_col),
                        static_cast<const void*>(u), static_cast<const void*>(v),
                        static_cast<const void*>(total_cost), static_cast<const void*>(status)})
    if (!p || !is_device_ptr(p))
      return fail(KMB_EINVAL, std::string(who) + ": every buffer must be device memory");
  return solve_batch_impl(c, costs, batch, n, seed, row_to_col, u, v, total_cost, nullptr, who,
                          c->engine, 0.0, status);
}

// Several contexts (normally one per GPU): contiguous slices of the batch, each
// solved by kmb_solve_batch_i32 on its own context, concurrently (one host
// thread per extra context).  Across devices the buffers must be host memory.
int kmb_solve_batch_multi_i32(kmb_context* const* ctxs, int32_t nctx, const int32_t* costs,
                              int32_t batch, int32_t n, int32_t seed, int32_t* row_to_col,
                              int64_t* u, int64_t* v, int64_t* total_cost, kmb_stats* stats) {
  const char* who = "kmb_solve_batch_multi_i32";
  if (!ctxs || nctx <= 0) return fail(KMB_EINVAL, std::string(who) + ": no contexts");
  for (int k = 0; k < nctx; ++k)
    if (!ctxs[k]) return fail(KMB_EINVAL, std::string(who) + ": NULL context");
  if (batch <= 0 || n <= 0) return fail(KMB_EINVAL, std::string(who) + ": dimensions must be positive");
  if (!costs) return fail(KMB_EINVAL, std::string(who) + ": costs is NULL");
  bool one_device = true;
  for (int k = 1; k < nctx; ++k) one_device &= ctxs[k]->device == ctxs[0]->device;
  if (!one_device) {
    cudaSetDevice(ctxs[0]->device);
    for (const void* p : {static_cast<const void*>(costs), static_cast<const void*>(row_to_col),
                          static_cast<const void*>(u), static_cast<const void*>(v),
                          static_cast<const void*>(total_cost)})
      if (p && is_device_ptr(p))
        return fail(KMB_EINVAL, std::string(who) + ": contexts on several devices need host buffers");
  }
  const int parts = std::min<int>(nctx, batch);
  std::vector<int> lo(parts + 1);
  for (int k = 0; k <= parts; ++k) lo[k] = static_cast<int>(static_cast<int64_t>(batch) * k / parts);
  std::vector<int> rc(parts, KMB_OK);
  std::vector<std::string> msg(parts);
  std::vector<kmb_stats> st(parts);
  auto run = [&](int k) {
    const size_t o = static_cast<size_t>(lo[k]) * n;
    rc[k] = kmb_solve_batch_i32(ctxs[k], costs + o * n, lo[k + 1] - lo[k], n, seed,
                                row_to_col ? row_to_col + o : nullptr, u ? u + o : nullptr,
                                v ? v + o : nullptr, total_cost ? total_cost + lo[k] : nullptr,
                                &st[k]);
    if (rc[k] != KMB_OK) msg[k] = g_err;
  };
  std::vector<std::thread> th;
  th.reserve(parts - 1);
  for (int k = 1; k < parts; ++k) th.emplace_back(run, k);
  run(0);
  for (auto& t : th) t.join();
  for (int k = 0; k < parts; ++k)
    if (rc[k] != KMB_OK) return fail(rc[k], msg[k] + " (slice " + std::to_string(k) + ")");
  if (stats) {
    *stats = st[0];
    for (int k = 1; k < parts; ++k) {
      stats->phases += st[k].phases;
      stats->dual_steps += st[k].dual_steps;
      stats->rows_scanned += st[k].rows_scanned;
      stats->cost_bytes_read += st[k].cost_bytes_read;
      stats->rounds += st[k].rounds;
      stats->seconds = std::max(stats->seconds, st[k].seconds);
      stats->converged = stats->converged && st[k].converged;
      for (int q = 0; q < 6; ++q) stats->stage_ns[q] += st[k].stage_ns[q];
      stats->max_instance_cycles = std::max(stats->max_instance_cycles, st[k].max_instance_cycles);
      stats->sum_instance_cycles += st[k].sum_instance_cycles;
    }
  }
  return KMB_OK;
}

// Grid engine staging: slab width W (power of two) and CTA count G, pitched
// cost copy when the caller's buffer is not already in that layout, workspace.
static int prepare_grid(kmb_context* c, const int32_t* cost, int32_t n, int64_t ld, int32_t seed,
                        kmb::SolverArgs* out, int* G_out, bool cluster = false) {
  cudaStream_t st = c->stream;
  int64_t maxg = c->max_ctas > 0 ? c->max_ctas : c->sm_count;
  if (maxg > c->sm_count) maxg = c->sm_count;  // cooperative: one CTA per SM
  if (cluster && maxg > 16) maxg = 16;          // one thread-block cluster
  int W = 4;
  while ((n + W - 1) / W > maxg) W <<= 1;
  const int G = (n + W - 1) / W;
  const int64_t pitch = static_cast<int64_t>(G) * W;
  const size_t nn = static_cast<size_t>(n);
  const int32_t* dC = cost;
  const bool dev_in = is_device_ptr(cost);
  const bool aligned = (reinterpret_cast<uintptr_t>(cost) & 15) == 0;
  if (!(dev_in && aligned && ld == pitch)) {
    KMB_CUDA(c->cost.ensure(nn * pitch * 4));
    KMB_CUDA(cudaMemcpy2DAsync(c->cost.p, pitch * 4, cost, ld * 4, nn * 4, nn, cudaMemcpyDefault, st));
    dC = c->cost.as<int32_t>();
  }
  KMB_CUDA(c->u.ensure(nn * 8));
  KMB_CUDA(c->v.ensure(nn * 8));
  KMB_CUDA(c->mrow.ensure(nn * 4));
  KMB_CUDA(c->mcol.ensure(nn * 4));
  KMB_CUDA(c->tpar.ensure(nn * 4));
  KMB_CUDA(c->root.ensure(nn * 4));
  KMB_CUDA(c->claim.ensure(nn * 8));
  KMB_CUDA(c->lrow0.ensure(nn * 4));
  KMB_CUDA(c->lrow1.ensure(nn * 4));
  KMB_CUDA(c->lw0.ensure(nn * 8));
  KMB_CUDA(c->lw1.ensure(nn * 8));
  KMB_CUDA(c->found.ensure(nn * 4));
  KMB_CUDA(c->partial.ensure(static_cast<size_t>(G) * 8));
  KMB_CUDA(c->ctrl.ensure(sizeof(kmb::Ctrl)));
  KMB_CUDA(c->obj.ensure(8));
  kmb::SolverArgs& a = *out;
  a.C = dC;
  a.pitch = pitch;
  a.n = n;
  a.W = W;
  a.seed = seed;
  // prefetching the rows each round appends pays when they come from HBM (c5:
  // 121.7 -> 117.2 ms); on an L2-resident matrix it only adds traffic (c4: +5%)
  a.prefetch_rows = static_cast<double>(pitch) * n * 4 > 96.0 * (1 << 20) ? 1 : 0;
#ifndef KMB_SLAB_CACHE
#define KMB_SLAB_CACHE 1
#endif
  // the grid engine keeps the rows' roots and its slab's matches in shared
  // memory (4 (n + W) bytes; one CTA per SM), the cluster engine does not
  a.slab_cache = (KMB_SLAB_CACHE && !cluster && n <= 40960) ? 1 : 0;
  a.u = c->u.as<int64_t>();
  a.v = c->v.as<int64_t>();
  a.match_row = c->mrow.as<int32_t>();
  a.match_col = c->mcol.as<int32_t>();
  a.tree_par = c->tpar.as<int32_t>();
  a.root_row = c->root.as<int32_t>();
  a.claim = c->claim.as<uint64_t>();
  a.list_row[0] = c->lrow0.as<int32_t>();
  a.list_row[1] = c->lrow1.as<int32_t>();
  a.list_w[0] = c->lw0.as<int64_t>();
  a.list_w[1] = c->lw1.as<int64_t>();
  a.found = c->found.as<int32_t>();
  a.partial = c->partial.as<int64_t>();
  a.ctrl = c->ctrl.as<kmb::Ctrl>();
  *G_out = G;
  return KMB_OK;
}

int kmb_solve_i32(kmb_context* c, const int32_t* cost, int32_t n, int64_t ld, int32_t seed,
                  double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                  int64_t* total_cost, kmb_stats* stats) {
  const char* who = "kmb_solve_i32";
  if (!c) return fail(KMB_EINVAL, "kmb_solve_i32: NULL context");
  if (n <= 0) return fail(KMB_EINVAL, "kmb_solve_i32: dimensions must be positive");
  if (!cost) return fail(KMB_EINVAL, "kmb_solve_i32: cost is NULL");
  if (ld < n) return fail(KMB_EINVAL, "kmb_solve_i32: ld < n");
  if (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED) return fail(KMB_EINVAL, "kmb_solve_i32: bad seed");
  KMB_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;

  int engine = c->engine;
  // auto (measured crossovers): one CTA per instance up to
  // n = 256 (no time budget there; c1 0.20 ms vs 0.55 for one warp), one
  // 512-thread CTA up to n = 1792 (c2 8.5 ms vs 24 on a cluster), one
  // thread-block cluster with replicated row state up to n = 4608, the
  // whole-GPU grid beyond (n = 6144: 64 vs 78 ms uniform, 269 vs 298 geometric)
  // round 2: the replicated cluster engine takes 1792 < n <= 4608 (c4 84 ms vs
  // 130 on engine 5; uniform n = 3072 23 vs 34 ms on the single CTA, n = 4096 31
  // vs 43 on engine 5; at n = 5120 it ties the grid engine)
  if (engine == 0)
    engine = (n <= 256 && time_budget_s <= 0.0) ? 6 : n <= 1792 ? 8 : (n <= 4608 ? 11 : 1);
  if (engine == 6 && n > kmb::batch_max_n()) engine = 1;
  if (engine == 4 && n > kmb::warp_max_n()) engine = 1;
  if (engine == 8 && n > kmb::big_max_n()) engine = 1;
  if (engine == 11 && n > kmb::cluster_max_n()) engine = 1;
  if (engine == 4 || engine == 6 || engine == 8 || engine == 11) {
    if (time_budget_s > 0.0 && engine != 8 && engine != 11)
      return fail(KMB_EINVAL, "kmb_solve_i32: the per-instance engines have no time budget; use engine 1");
    const int32_t* src = cost;
    if (ld != n) {  // compact into the batch buffer
      KMB_CUDA(c->bcost.ensure(static_cast<size_t>(n) * n * 4));
      KMB_CUDA(cudaMemcpy2DAsync(c->bcost.p, n * 4, cost, ld * 4, n * 4, n, cudaMemcpyDefault, st));
      src = c->bcost.as<int32_t>();
    }
    return solve_batch_impl(c, src, 1, n, seed, row_to_col, u, v, total_cost, stats, who, engine,
                            time_budget_s);
  }

  const bool cluster = engine == 5;
  kmb::SolverArgs a{};
  int G = 0;
  if (int r = prepare_grid(c, cost, n, ld, seed, &a, &G, cluster)) return r;
  const size_t nn = static_cast<size_t>(n);
  const int32_t* dC = a.C;
  const int64_t pitch = a.pitch;
  a.deadline_ns = 0;
  if (time_budget_s > 0.0) {
    // relative budget (top bit set): the kernel adds it to its own %globaltimer
    a.deadline_ns = (1ull << 63) | static_cast<unsigned long long>(time_budget_s * 1e9);
  }
  KMB_CUDA(cudaMemsetAsync(c->ctrl.p, 0, sizeof(kmb::Ctrl), st));
  KMB_CUDA(cudaEventRecord(c->ev0, st));
  KMB_CUDA(kmb::launch_solver(a, G, cluster, st));
  KMB_CUDA(kmb::launch_objective(dC, pitch, n, a.match_row, c->obj.as<unsigned long long>(), st));
  KMB_CUDA(cudaEventRecord(c->ev1, st));
  int r;
  if ((r = copy_out(row_to_col, a.match_row, nn * 4, st))) return r;
  if ((r = copy_out(u, a.u, nn * 8, st))) return r;
  if ((r = copy_out(v, a.v, nn * 8, st))) return r;
  if ((r = copy_out(total_cost, c->obj.p, 8, st))) return r;
  kmb::Ctrl h;
  KMB_CUDA(cudaMemcpyAsync(&h, c->ctrl.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  KMB_CUDA(cudaStreamSynchronize(st));
  if (h.status != 0) return status_message(h.status, who);
  if (stats) {
    stats->phases = h.phases;
    stats->dual_steps = h.dual_steps;
    stats->rows_scanned = h.rows_scanned;
    stats->segment_rows = h.seg_rows;
    stats->cost_bytes_read =
        4ll * n * (h.rows_scanned + (seed == KMB_SEED_BATCHED ? n : 0)) + 16ll * h.seg_rows;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    stats->seconds = ms * 1e-3;
    stats->converged = h.free_rows == 0 ? 1 : 0;
    stats->engine = cluster ? 5 : 1;
    stats->rounds = h.rounds;
    for (int k = 0; k < 6; ++k) stats->stage_ns[k] = h.stage_ns[k];
  }
  return KMB_OK;
}

}  // extern "C"

// ---- 64-bit costs (the reference's own cost type) ------------------------------

namespace {

constexpr int64_t kNarrowMax = (int64_t{1} << 29) - 1;  // the 32-bit engines' range
constexpr int64_t kWideMax = int64_t{1} << 60;          // |reduced costs| <= 4 * max < 2^63

// validate_instance's headroom (core.cpp:47-53) for a unit square instance:
// S * N * (n + m + 2) <= 2^62 with S = n, m = n
int64_t headroom_max(int32_t n) {
  const int64_t h = ((int64_t{1} << 62) / n) / (2 * static_cast<int64_t>(n) + 2);
  return h < kWideMax ? h : kWideMax;
}

// the caller's costs as one contiguous device block (rows x cols)
int stage_i64(kmb_context* c, const int64_t* cost, int64_t rows, int32_t cols, int64_t ld,
              const int64_t** out) {
  if (is_device_ptr(cost) && ld == cols) {
    *out = cost;
    return KMB_OK;
  }
  KMB_CUDA(c->w64in.ensure(static_cast<size_t>(rows) * cols * 8));
  if (ld == cols) {
    KMB_CUDA(cudaMemcpyAsync(c->w64in.p, cost, static_cast<size_t>(rows) * cols * 8, cudaMemcpyDefault,
                             c->stream));
    *out = c->w64in.as<int64_t>();
    return KMB_OK;
  }
  KMB_CUDA(cudaMemcpy2DAsync(c->w64in.p, static_cast<size_t>(cols) * 8, cost, static_cast<size_t>(ld) * 8,
                             static_cast<size_t>(cols) * 8, rows, cudaMemcpyDefault, c->stream));
  *out = c->w64in.as<int64_t>();
  return KMB_OK;
}

int minmax_i64(kmb_context* c, const int64_t* d, int64_t rows, int32_t cols, long long* lo, long long* hi) {
  KMB_CUDA(c->wmm.ensure(32));
  const long long init[2] = {LLONG_MAX, LLONG_MIN};
  KMB_CUDA(cudaMemcpyAsync(c->wmm.p, init, 16, cudaMemcpyHostToDevice, c->stream));
  KMB_CUDA(kmb::launch_minmax_i64(d, cols, rows, cols, c->wmm.as<long long>(), c->sm_count, c->stream));
  long long h[2];
  KMB_CUDA(cudaMemcpyAsync(h, c->wmm.p, 16, cudaMemcpyDeviceToHost, c->stream));
  KMB_CUDA(cudaStreamSynchronize(c->stream));
  *lo = h[0];
  *hi = h[1];
  return KMB_OK;
}

template <class T>
int dev_or_ws(T* user, DevBuf& ws, size_t count, T** out) {
  if (user && is_device_ptr(user)) {
    *out = user;
    return KMB_OK;
  }
  KMB_CUDA(ws.ensure(count * sizeof(T) > 0 ? count * sizeof(T) : 8));
  *out = ws.as<T>();
  return KMB_OK;
}

// Wide engine on contiguous device costs, device outputs; stats summed.
int solve_wide(kmb_context* c, const int64_t* dC, int32_t batch, int32_t n, int32_t seed,
               double time_budget_s, int32_t* dr2c, int64_t* du, int64_t* dv, int64_t* dtot,
               kmb_stats* stats, const char* who) {
  cudaStream_t st = c->stream;
  const int slots = kmb::wide_slots(batch, c->sm_count);
  KMB_CUDA(c->wws64.ensure(kmb::wide_ws64_bytes(n, slots)));
  KMB_CUDA(c->wws32.ensure(kmb::wide_ws32_bytes(n, slots)));
  KMB_CUDA(c->bstat.ensure(static_cast<size_t>(batch) * kmb::KMB_ISTATS * 8));
  KMB_CUDA(c->bstatus.ensure(static_cast<size_t>(batch) * 4));
  c->last_batch = batch;
  kmb::WideArgs a{};
  a.C = dC;
  a.ld = n;
  a.inst_stride = static_cast<int64_t>(n) * n;
  a.batch = batch;
  a.n = n;
  a.seed = seed;
  a.deadline_ns = time_budget_s > 0.0 ? static_cast<int64_t>(time_budget_s * 1e9) : 0;
  a.row_to_col = dr2c;
  a.u = du;
  a.v = dv;
  a.total_cost = dtot;
  a.stats = c->bstat.as<int64_t>();
  a.status = c->bstatus.as<int32_t>();
  a.ws64 = c->wws64.as<int64_t>();
  a.ws32 = c->wws32.as<int32_t>();
  a.max_cost = kWideMax;
  KMB_CUDA(cudaEventRecord(c->ev0, st));
  KMB_CUDA(kmb::launch_wide(a, slots, st));
  KMB_CUDA(cudaEventRecord(c->ev1, st));
  KMB_CUDA(c->bsum.ensure(16 * 8));
  if (!c->hsum) KMB_CUDA(cudaMallocHost(&c->hsum, 16 * 8));
  KMB_CUDA(kmb::launch_batch_summary(c->bstat.as<int64_t>(), c->bstatus.as<int32_t>(), batch,
                                     c->bsum.as<int64_t>(), st));
  KMB_CUDA(cudaMemcpyAsync(c->hsum, c->bsum.p, 11 * 8, cudaMemcpyDeviceToHost, st));
  {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, who);
  }
  const int64_t* h = c->hsum;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->phases = h[1];
    stats->dual_steps = h[2];
    stats->rows_scanned = h[3];
    stats->rounds = h[4];
    stats->sum_instance_cycles = h[5];
    stats->max_instance_cycles = h[6];
    stats->cost_bytes_read = 8 * static_cast<int64_t>(n) * (h[3] + static_cast<int64_t>(batch) * n);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    stats->seconds = ms * 1e-3;
    stats->converged = h[0] == kStopped ? 0 : 1;
    stats->engine = 9;
  }
  if (h[0] == KMB_ERANGE)
    return fail(KMB_ERANGE, std::string(who) + ": supply * cost magnitude too large for 64-bit arithmetic");
  if (h[0] && h[0] != kStopped) return status_message(static_cast<int>(h[0]), who);
  return KMB_OK;
}

// Solve `batch` contiguous device instances whose costs lie in [0, hi]: the
// 32-bit engines on a narrowed copy when hi < 2^29, the wide engine otherwise.
// Outputs are device buffers.
// the narrowed copy in c->wnar on the 32-bit engines
int solve_narrow_dev(kmb_context* c, int32_t batch, int32_t n, int32_t seed, double time_budget_s,
                     int32_t* dr2c, int64_t* du, int64_t* dv, int64_t* dtot, kmb_stats* stats,
                     const char* who) {
  if (batch == 1)
    return kmb_solve_i32(c, c->wnar.as<int32_t>(), n, n, seed, time_budget_s, dr2c, du, dv, dtot, stats);
  return solve_batch_impl(c, c->wnar.as<int32_t>(), batch, n, seed, dr2c, du, dv, dtot, stats, who,
                          c->engine, time_budget_s);
}

int solve_dev_i64(kmb_context* c, const int64_t* dC, int32_t batch, int32_t n, int32_t seed,
                  double time_budget_s, long long hi, int32_t* dr2c, int64_t* du, int64_t* dv,
                  int64_t* dtot, kmb_stats* stats, const char* who) {
  if (hi <= kNarrowMax) {
    const size_t cnt = static_cast<size_t>(batch) * n * n;
    KMB_CUDA(c->wnar.ensure(cnt * 4));
    KMB_CUDA(kmb::launch_convert_i64(dC, n, static_cast<int64_t>(batch) * n, n, false, 1, 1, nullptr,
                                     c->wnar.as<int32_t>(), nullptr, c->sm_count, c->stream));
    return solve_narrow_dev(c, batch, n, seed, time_budget_s, dr2c, du, dv, dtot, stats, who);
  }
  return solve_wide(c, dC, batch, n, seed, time_budget_s, dr2c, du, dv, dtot, stats, who);
}

int copy_results(kmb_context* c, int32_t batch, int32_t n, int32_t* r2c, int64_t* u, int64_t* v,
                 int64_t* tot, const int32_t* dr2c, const int64_t* du, const int64_t* dv,
                 const int64_t* dtot) {
  const size_t nb = static_cast<size_t>(batch) * n;
  int r;
  if (r2c != dr2c && (r = copy_out(r2c, dr2c, nb * 4, c->stream))) return r;
  if (u != du && (r = copy_out(u, du, nb * 8, c->stream))) return r;
  if (v != dv && (r = copy_out(v, dv, nb * 8, c->stream))) return r;
  if (tot != dtot && (r = copy_out(tot, dtot, static_cast<size_t>(batch) * 8, c->stream))) return r;
  KMB_CUDA(cudaStreamSynchronize(c->stream));
  return KMB_OK;
}

int solve_i64_common(kmb_context* c, const int64_t* costs, int32_t batch, int32_t n, int64_t ld,
                     int32_t seed, double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                     int64_t* total_cost, kmb_stats* stats, const char* who) {
  if (!c) return fail(KMB_EINVAL, std::string(who) + ": NULL context");
  if (batch <= 0 || n <= 0) return fail(KMB_EINVAL, std::string(who) + ": dimensions must be positive");
  if (!costs) return fail(KMB_EINVAL, std::string(who) + ": cost is NULL");
  if (ld < n) return fail(KMB_EINVAL, std::string(who) + ": ld < n");
  if (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED) return fail(KMB_EINVAL, std::string(who) + ": bad seed");
  KMB_CUDA(cudaSetDevice(c->device));
  const int64_t* dC = nullptr;
  int r;
  if ((r = stage_i64(c, costs, static_cast<int64_t>(batch) * n, n, ld, &dC))) return r;
  long long lo = 0, hi = 0;
  if ((r = minmax_i64(c, dC, static_cast<int64_t>(batch) * n, n, &lo, &hi))) return r;
  if (lo < 0) return fail(KMB_ENEGATIVE, std::string(who) + ": costs must be nonnegative");
  if (hi > headroom_max(n))
    return fail(KMB_ERANGE, std::string(who) + ": supply * cost magnitude too large for 64-bit arithmetic");
  if (batch > 1 && hi <= kNarrowMax && n > kmb::big_max_n())
    return fail(KMB_EINVAL, std::string(who) + ": n > " + std::to_string(kmb::big_max_n()) +
                                " (use kmb_solve_i64 per instance)");
  const size_t nb = static_cast<size_t>(batch) * n;
  int32_t* dr2c;
  int64_t *du, *dv, *dtot;
  if ((r = dev_or_ws(row_to_col, c->wr2c, nb, &dr2c)) || (r = dev_or_ws(u, c->wu, nb, &du)) ||
      (r = dev_or_ws(v, c->wv, nb, &dv)) || (r = dev_or_ws(total_cost, c->wtot, batch, &dtot)))
    return r;
  if ((r = solve_dev_i64(c, dC, batch, n, seed, time_budget_s, hi, dr2c, du, dv, dtot, stats, who)))
    return r;
  return copy_results(c, batch, n, row_to_col, u, v, total_cost, dr2c, du, dv, dtot);
}

// K11 on the device (quantize_costs, hungarian.cpp:33-53): N = max cost (hi),
// chat = floor(C * B / N) into `chat` (device, optional) and, when B < 2^29 so
// every chat fits the 32-bit engines, also narrowed into c->wnar; lossless
// flag.  All-zero costs: N = 1, chat = C, lossless.
int quantize_dev(kmb_context* c, const int64_t* dC, int64_t rows, int32_t cols, long long hi, int64_t B,
                 int64_t* chat, bool want_narrow, int64_t* N_out, int32_t* lossless_out) {
  if (B <= 0) return fail(KMB_EINVAL, "quantize_costs: B must be positive");
  const size_t cnt = static_cast<size_t>(rows) * cols;
  int64_t N = hi;
  if (N <= 0) {
    *N_out = 1;
    *lossless_out = 1;
    if (chat) KMB_CUDA(cudaMemcpyAsync(chat, dC, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
    if (want_narrow) {
      KMB_CUDA(c->wnar.ensure(cnt * 4));
      KMB_CUDA(kmb::launch_convert_i64(dC, cols, rows, cols, false, 1, 1, nullptr, c->wnar.as<int32_t>(),
                                       nullptr, c->sm_count, c->stream));
    }
    return KMB_OK;
  }
  if (B > INT64_MAX / N) return fail(KMB_EINVAL, "quantize_costs: B * max cost overflows");
  KMB_CUDA(c->wmm.ensure(32));
  int32_t* lossy = reinterpret_cast<int32_t*>(c->wmm.as<char>() + 16);
  KMB_CUDA(cudaMemsetAsync(lossy, 0, 4, c->stream));
  int32_t* nar = nullptr;
  if (want_narrow) {
    KMB_CUDA(c->wnar.ensure(cnt * 4));
    nar = c->wnar.as<int32_t>();
  }
  KMB_CUDA(kmb::launch_convert_i64(dC, cols, rows, cols, true, B, N, chat, nar, lossy, c->sm_count, c->stream));
  int32_t h = 0;
  KMB_CUDA(cudaMemcpyAsync(&h, lossy, 4, cudaMemcpyDeviceToHost, c->stream));
  KMB_CUDA(cudaStreamSynchronize(c->stream));
  *N_out = N;
  *lossless_out = h ? 0 : 1;
  return KMB_OK;
}

}  // namespace

extern "C" {

int kmb_solve_i64(kmb_context* c, const int64_t* cost, int32_t n, int64_t ld, int32_t seed,
                  double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                  int64_t* total_cost, kmb_stats* stats) {
  return solve_i64_common(c, cost, 1, n, ld, seed, time_budget_s, row_to_col, u, v, total_cost, stats,
                          "kmb_solve_i64");
}

int kmb_solve_batch_i64(kmb_context* c, const int64_t* costs, int32_t batch, int32_t n, int32_t seed,
                        int32_t* row_to_col, int64_t* u, int64_t* v, int64_t* total_cost,
                        kmb_stats* stats) {
  return solve_i64_common(c, costs, batch, n, n, seed, 0.0, row_to_col, u, v, total_cost, stats,
                          "kmb_solve_batch_i64");
}

int kmb_quantize_i64(kmb_context* c, const int64_t* cost, int64_t count, int64_t B, int64_t* chat,
                     int64_t* N, int32_t* lossless) {
  if (!c) return fail(KMB_EINVAL, "kmb_quantize_i64: NULL context");
  if (count < 0 || (count > 0 && !cost)) return fail(KMB_EINVAL, "kmb_quantize_i64: bad arguments");
  if (B <= 0) return fail(KMB_EINVAL, "quantize_costs: B must be positive");
  if (count == 0) {
    if (N) *N = 1;
    if (lossless) *lossless = 1;
    return KMB_OK;
  }
  KMB_CUDA(cudaSetDevice(c->device));
  const int64_t* dC = nullptr;
  int r;
  if ((r = stage_i64(c, cost, count, 1, 1, &dC))) return r;
  long long lo = 0, hi = 0;
  if ((r = minmax_i64(c, dC, count, 1, &lo, &hi))) return r;
  int64_t* dchat = nullptr;
  if ((r = dev_or_ws(chat, c->wchat, static_cast<size_t>(count), &dchat))) return r;
  int64_t n_out = 1;
  int32_t ll = 1;
  if ((r = quantize_dev(c, dC, count, 1, hi, B, dchat, false, &n_out, &ll))) return r;
  if (chat && chat != dchat) {
    KMB_CUDA(cudaMemcpyAsync(chat, dchat, static_cast<size_t>(count) * 8, cudaMemcpyDeviceToHost, c->stream));
    KMB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (N) *N = n_out;
  if (lossless) *lossless = ll;
  return KMB_OK;
}

int kmb_solve_batched_km_i64(kmb_context* c, const int64_t* cost, int32_t n, int64_t B,
                             double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                             int64_t* total_cost, int64_t* chat, int64_t* N, int32_t* lossless,
                             kmb_stats* stats) {
  const char* who = "solve_batched_km";
  if (!c) return fail(KMB_EINVAL, "kmb_solve_batched_km_i64: NULL context");
  if (n <= 0) return fail(KMB_EINVAL, std::string(who) + ": dimensions must be positive");
  if (!cost) return fail(KMB_EINVAL, "kmb_solve_batched_km_i64: cost is NULL");
  KMB_CUDA(cudaSetDevice(c->device));
  const int64_t* dC = nullptr;
  int r;
  const int64_t nn = static_cast<int64_t>(n) * n;
  if ((r = stage_i64(c, cost, n, n, n, &dC))) return r;
  long long lo = 0, hi = 0;
  if ((r = minmax_i64(c, dC, n, n, &lo, &hi))) return r;
  // require_unit_square (hungarian.cpp:15-21) before quantize_costs (:318)
  if (lo < 0) return fail(KMB_ENEGATIVE, std::string(who) + ": costs must be nonnegative");
  if (hi > headroom_max(n))
    return fail(KMB_ERANGE, std::string(who) + ": supply * cost magnitude too large for 64-bit arithmetic");
  const size_t nb = static_cast<size_t>(n);
  int32_t* dr2c;
  int64_t *du, *dv, *dtot;
  if ((r = dev_or_ws(row_to_col, c->wr2c, nb, &dr2c)) || (r = dev_or_ws(u, c->wu, nb, &du)) ||
      (r = dev_or_ws(v, c->wv, nb, &dv)) || (r = dev_or_ws(total_cost, c->wtot, 1, &dtot)))
    return r;
  // B a multiple of N (the lossless B = N * n among them): chat = k * C exactly
  // and the search is scale-equivariant (every reduced cost, slack and dual
  // step scales by k, ties stay ties), so C is solved and the duals scaled.
  const int64_t k = (hi > 0 && B > 0 && B % hi == 0) ? B / hi : 0;
  int64_t n_q = 1;
  int32_t ll = 1;
  int64_t* dchat = nullptr;
  const bool need_chat = chat != nullptr || (k == 0 && hi > 0 && B > kNarrowMax);
  if (need_chat && (r = dev_or_ws(chat, c->wchat, static_cast<size_t>(nn), &dchat))) return r;
  if (k > 0 || hi <= 0) {
    if ((r = quantize_dev(c, dC, n, n, hi, B, dchat, false, &n_q, &ll))) return r;
    if ((r = solve_dev_i64(c, dC, 1, n, KMB_SEED_BATCHED, time_budget_s, hi, dr2c, du, dv, dtot, stats, who)))
      return r;
    if (k > 1) {
      KMB_CUDA(kmb::launch_scale_i64(du, n, k, c->sm_count, c->stream));
      KMB_CUDA(kmb::launch_scale_i64(dv, n, k, c->sm_count, c->stream));
    }
  } else {
    // every chat <= B: the 32-bit engines take it when B < 2^29
    const bool narrow = B <= kNarrowMax;
    if (!narrow && B > kWideMax)
      return fail(KMB_ERANGE, std::string(who) + ": quantized cost exceeds the device range [0, 2^60]");
    if ((r = quantize_dev(c, dC, n, n, hi, B, dchat, narrow, &n_q, &ll))) return r;
    if (narrow)
      r = solve_narrow_dev(c, 1, n, KMB_SEED_BATCHED, time_budget_s, dr2c, du, dv, dtot, stats, who);
    else
      r = solve_wide(c, dchat, 1, n, KMB_SEED_BATCHED, time_budget_s, dr2c, du, dv, dtot, stats, who);
    if (r) return r;
  }
  // the objective on the caller's costs (make_result, core.cpp:76-90)
  KMB_CUDA(kmb::launch_total_i64(dC, n, nn, 1, n, dr2c, dtot, c->sm_count, c->stream));
  if (chat && chat != dchat) KMB_CUDA(cudaMemcpyAsync(chat, dchat, nn * 8, cudaMemcpyDeviceToHost, c->stream));
  if ((r = copy_results(c, 1, n, row_to_col, u, v, total_cost, dr2c, du, dv, dtot))) return r;
  if (N) *N = n_q;
  if (lossless) *lossless = ll;
  return KMB_OK;
}

int kmb_last_instance_stats(kmb_context* c, int64_t* out, int64_t capacity, int64_t* count) {
  if (!c || !out || !count) return fail(KMB_EINVAL, "kmb_last_instance_stats: bad arguments");
  KMB_CUDA(cudaSetDevice(c->device));
  // the last batch's instances only, read in order with the context's stream
  // (a non-blocking stream is not ordered with the legacy default stream)
  const int64_t have = c->last_batch * kmb::KMB_ISTATS;
  const int64_t k = capacity < have ? capacity : have;
  *count = c->last_batch;
  if (k > 0) {
    KMB_CUDA(cudaMemcpyAsync(out, c->bstat.p, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, c->stream));
    KMB_CUDA(cudaStreamSynchronize(c->stream));
  }
  return KMB_OK;
}

int kmb_auction_i32(kmb_context* c, const int32_t* costs, int32_t batch, int32_t n,
                    const kmb_auction_config* cfg, double* prices, int32_t* row_to_col,
                    int64_t* total_cost, int64_t* bids, int32_t* converged,
                    double* epsilon_last, double* seconds) {
  if (!c) return fail(KMB_EINVAL, "kmb_auction_i32: NULL context");
  if (!cfg) return fail(KMB_EINVAL, "kmb_auction_i32: NULL config");
  const char* who = cfg->scaled ? "solve_auction_scaled" : "solve_auction";
  if (batch <= 0 || n <= 0 || !costs) return fail(KMB_EINVAL, std::string(who) + ": bad arguments");
  // auction.cpp:190-191, 205-206
  if (!cfg->scaled && !(cfg->epsilon > 0.0))
    return fail(KMB_EINVAL, "solve_auction: epsilon must be positive");
  if (cfg->scaled && !(cfg->theta > 1.0))
    return fail(KMB_EINVAL, "solve_auction_scaled: theta must exceed 1");
  if (n > kmb::auction_max_n())
    return fail(KMB_EINVAL, std::string(who) + ": n > " + std::to_string(kmb::auction_max_n()) +
                                " (prices and owners must fit in shared memory)");
  KMB_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const size_t nb = static_cast<size_t>(batch) * n;
  const int32_t* dcost = costs;
  KMB_CUDA(cudaEventRecord(c->ev0, st));
  if (!is_device_ptr(costs)) {
    KMB_CUDA(c->bcost.ensure(nb * n * 4));
    KMB_CUDA(cudaMemcpyAsync(c->bcost.p, costs, nb * n * 4, cudaMemcpyHostToDevice, st));
    dcost = c->bcost.as<int32_t>();
  }
  auto dev = [&](void* user, DevBuf& buf, size_t bytes, void** out) -> cudaError_t {
    if (user && is_device_ptr(user)) {
      *out = user;
      return cudaSuccess;
    }
    *out = nullptr;
    if (!user) return cudaSuccess;
    cudaError_t e = buf.ensure(bytes);
    *out = buf.p;
    return e;
  };
  void *dp, *dr, *dt, *db, *dc, *de;
  KMB_CUDA(dev(prices, c->aprice, nb * 8, &dp));
  KMB_CUDA(dev(row_to_col, c->ar2c, nb * 4, &dr));
  KMB_CUDA(dev(total_cost, c->atot, batch * 8, &dt));
  KMB_CUDA(dev(bids, c->abids, batch * 8, &db));
  KMB_CUDA(dev(converged, c->acomp, batch * 4, &dc));
  KMB_CUDA(dev(epsilon_last, c->aeps, batch * 8, &de));
  KMB_CUDA(c->amin.ensure(batch * 8));
  KMB_CUDA(c->amax.ensure(batch * 8));
  KMB_CUDA(c->bstatus.ensure(batch * 4));
  kmb::AuctionArgs a{};
  a.C = dcost;
  a.ld = n;
  a.inst_stride = static_cast<int64_t>(n) * n;
  a.batch = batch;
  a.n = n;
  a.scaled = cfg->scaled ? 1 : 0;
  a.eps0 = cfg->epsilon;
  a.theta = cfg->theta;
  a.eps_final = cfg->epsilon_final;
  a.max_bids = cfg->max_bids;
  a.budget_ns = cfg->time_budget_s > 0.0 ? static_cast<int64_t>(cfg->time_budget_s * 1e9) : 0;
  a.cmin = c->amin.as<long long>();
  a.cmax = c->amax.as<long long>();
  a.prices = static_cast<double*>(dp);
  a.row_to_col = static_cast<int32_t*>(dr);
  a.total_cost = static_cast<int64_t*>(dt);
  a.bids = static_cast<int64_t*>(db);
  a.complete = static_cast<int32_t*>(dc);
  a.eps_last = static_cast<double*>(de);
  a.status = c->bstatus.as<int32_t>();
  KMB_CUDA(kmb::launch_auction(a, c->sm_count, st));
  KMB_CUDA(cudaEventRecord(c->ev1, st));
  if (dp != prices) { int r = copy_out(prices, dp, nb * 8, st); if (r) return r; }
  if (dr != row_to_col) { int r = copy_out(row_to_col, dr, nb * 4, st); if (r) return r; }
  if (dt != total_cost) { int r = copy_out(total_cost, dt, batch * 8, st); if (r) return r; }
  if (db != bids) { int r = copy_out(bids, db, batch * 8, st); if (r) return r; }
  if (dc != converged) { int r = copy_out(converged, dc, batch * 4, st); if (r) return r; }
  if (de != epsilon_last) { int r = copy_out(epsilon_last, de, batch * 8, st); if (r) return r; }
  std::vector<int32_t> hs(batch);
  KMB_CUDA(cudaMemcpyAsync(hs.data(), c->bstatus.p, batch * 4, cudaMemcpyDeviceToHost, st));
  KMB_CUDA(cudaStreamSynchronize(st));
  if (seconds) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    *seconds = ms * 1e-3;
  }
  for (int32_t b = 0; b < batch; ++b)
    if (hs[b]) return status_message(hs[b], who);
  return KMB_OK;
}

int kmb_costs_from_points(kmb_context* c, const void* a, const void* b, int32_t dtype,
                          int32_t batch, int32_t n, int32_t m, int32_t dim, double scale,
                          int32_t squared, int32_t* out) {
  if (!c) return fail(KMB_EINVAL, "kmb_costs_from_points: NULL context");
  if (!a || !b || !out || batch <= 0 || n <= 0 || m <= 0 || dim <= 0 ||
      (dtype != KMB_F64 && dtype != KMB_F32))
    return fail(KMB_EINVAL, "kmb_costs_from_points: bad arguments");
  if (!(scale > 0.0)) return fail(KMB_EINVAL, "quantization scale must be positive");
  KMB_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const size_t es = dtype == KMB_F64 ? 8 : 4;
  const size_t abytes = es * batch * static_cast<size_t>(n) * dim;
  const size_t bbytes = es * batch * static_cast<size_t>(m) * dim;
  const size_t obytes = 4 * static_cast<size_t>(batch) * n * m;
  const void* da = a;
  const void* db = b;
  if (!is_device_ptr(a)) {
    KMB_CUDA(c->pa.ensure(abytes));
    KMB_CUDA(cudaMemcpyAsync(c->pa.p, a, abytes, cudaMemcpyHostToDevice, st));
    da = c->pa.p;
  }
  if (!is_device_ptr(b)) {
    KMB_CUDA(c->pb.ensure(bbytes));
    KMB_CUDA(cudaMemcpyAsync(c->pb.p, b, bbytes, cudaMemcpyHostToDevice, st));
    db = c->pb.p;
  }
  const bool host_out = !is_device_ptr(out);
  int32_t* dout = out;
  if (host_out) {
    KMB_CUDA(c->pout.ensure(obytes));
    dout = c->pout.as<int32_t>();
  }
  KMB_CUDA(c->pbad.ensure(sizeof(int32_t)));
  KMB_CUDA(cudaMemsetAsync(c->pbad.p, 0, sizeof(int32_t), st));
  if (dtype == KMB_F64)
    KMB_CUDA(kmb::launch_costs<double>(static_cast<const double*>(da), static_cast<const double*>(db),
                                       batch, n, m, dim, scale, squared, dout,
                                       c->pbad.as<int32_t>(), st));
  else
    KMB_CUDA(kmb::launch_costs<float>(static_cast<const float*>(da), static_cast<const float*>(db),
                                      batch, n, m, dim, scale, squared, dout,
                                      c->pbad.as<int32_t>(), st));
  if (host_out) KMB_CUDA(cudaMemcpyAsync(out, dout, obytes, cudaMemcpyDeviceToHost, st));
  int32_t bad = 0;
  KMB_CUDA(cudaMemcpyAsync(&bad, c->pbad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  KMB_CUDA(cudaStreamSynchronize(st));
  if (bad) return fail(KMB_ERANGE, "kmb_costs_from_points: a cost does not fit int32");
  return KMB_OK;
}

int kmb_bench_scan(kmb_context* c, const int32_t* cost, int32_t n, int64_t ld, int32_t iters,
                   double* seconds_per_pass, double* gbytes_per_s) {
  if (!c) return fail(KMB_EINVAL, "kmb_bench_scan: NULL context");
  if (n <= 0 || !cost || ld < n || iters <= 0) return fail(KMB_EINVAL, "kmb_bench_scan: bad arguments");
  KMB_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  kmb::SolverArgs a{};
  int G = 0;
  if (int r = prepare_grid(c, cost, n, ld, KMB_SEED_BATCHED, &a, &G)) return r;
  KMB_CUDA(c->tpar.ensure(static_cast<size_t>(n) * 8));  // reused as the key output
  KMB_CUDA(cudaMemsetAsync(c->ctrl.p, 0, sizeof(kmb::Ctrl), st));
  KMB_CUDA(kmb::launch_solver_init(a, st));  // row list 0..n-1 with the row minima as w
  KMB_CUDA(kmb::launch_scan_all(a, G, c->tpar.as<uint64_t>(), st));  // warm-up
  KMB_CUDA(cudaEventRecord(c->ev0, st));
  for (int32_t k = 0; k < iters; ++k)
    KMB_CUDA(kmb::launch_scan_all(a, G, c->tpar.as<uint64_t>(), st));
  KMB_CUDA(cudaEventRecord(c->ev1, st));
  KMB_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  const double t = ms * 1e-3 / iters;
  if (seconds_per_pass) *seconds_per_pass = t;
  if (gbytes_per_s) *gbytes_per_s = 4.0 * n * static_cast<double>(n) / t / 1e9;
  return KMB_OK;
}

}  // extern "C"
