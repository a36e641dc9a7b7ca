// Column-sharded single instance over several GPUs (BASELINE config 5's
// multi-GPU mode).  Rank r owns columns [col_begin,
// col_begin + ncols) of every row: an n x ncols slab in its HBM, and that
// slab's per-column search state (key, v, Dc, reached, tree parent, match).
// The row side (u, root, match_row, the reached-row list) is replicated and
// kept identical on every rank by applying the same exchanged entries in the
// same (rank-major) order.
//
// Per round (the same round as kmb_solver.cu, hungarian.cpp:175-217):
//   device  relax the new rows over the slab (reduced-cost scan) + local min
//   comm    allreduce(MIN) of the local min slack'          -> m, dual step
//   device  absorb tight slab columns -> (col, parent) list
//   host    turn them into new-row / free-column entries (row side is replicated)
//   comm    allgather of the entries                          -> same list everywhere
// Epoch end (a free column was reached anywhere): claims are computed from the
// gathered free-column entries, the claimed trees' (col, parent) pairs are
// allgathered so every rank can walk the augmenting paths, the slab dissolves
// its claimed columns on the device, the row side dissolves on the host.
//
// The exchange is an interface: NCCL (ncclAllReduce ncclMin / ncclAllGather
// over NVLink; libnccl is resolved at run time so the process shares the NCCL
// that torch already loaded) or caller-supplied callbacks (e.g. torch gloo),
// which lets two ranks share one GPU in tests.  Duals and total cost are the
// engine's (bit-identical to the reference, tests/test_sharded.py).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "kmb.h"
#include "kmb_common.cuh"
#include "kmb_internal.h"

namespace kmb {

// ---- device kernels on the slab --------------------------------------------------

__global__ void k_sh_rowmin(const int32_t* C, int64_t ld, int32_t n, int32_t ncols, int64_t* rowmin,
                            int32_t* status) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < n; i += nwarps) {
    const int32_t* row = C + static_cast<int64_t>(i) * ld;
    int32_t lo = 0x7fffffff, hi = 0;
    for (int j = lane; j < ncols; j += 32) {
      lo = min(lo, row[j]);
      hi = max(hi, row[j]);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      rowmin[i] = lo;
      if (lo < 0) atomicMax(status, 2);
      else if (hi >= (1 << 29)) atomicMax(status, 3);
    }
  }
}

// relax rows ent[0, cnt) (row, w) over the slab: thread = column, rows streamed
// in order (coalesced across the warp), then the local min of unreached slack'
__global__ void k_sh_relax(const int32_t* C, int64_t ld, int32_t ncols, const int32_t* rows,
                           const int64_t* ws, int32_t cnt, uint64_t* key, const int64_t* v,
                           const uint8_t* rch, int set_v, int64_t* v_out, unsigned long long* lmin) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t s = KMB_I64_INF;
  if (j < ncols) {
    uint64_t k = key[j];
    for (int r = 0; r < cnt; ++r) {
      const int32_t i = rows[r];
      const uint32_t c = static_cast<uint32_t>(C[static_cast<int64_t>(i) * ld + j]);
      k = umin64(k, pack_key(c + row_bias(ws[r]), i));
    }
    key[j] = k;
    int64_t vj = v[j];
    if (set_v) {  // column reduction (hungarian.cpp:328-333) is the first relax
      vj = key_val(k);
      v_out[j] = vj;
    }
    if (!rch[j]) s = key_val(k) - vj;
  }
  s = warp_min_i64(s);
  // slack' >= 0 for unreached columns; store biased so an unsigned min works
  if ((threadIdx.x & 31) == 0 && s != KMB_I64_INF)
    atomicMin(lmin, static_cast<unsigned long long>(s));
}

__global__ void k_sh_absorb(int32_t ncols, const uint64_t* key, const int64_t* v, uint8_t* rch,
                            int64_t* dc, int32_t* tree_par, int64_t D, int32_t* out_cols,
                            int32_t* out_par, int32_t* out_cnt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols || rch[j]) return;
  if (key_val(key[j]) - v[j] != D) return;
  rch[j] = 1;
  dc[j] = D;
  const int32_t par = key_row(key[j]);
  tree_par[j] = par;
  const int pos = atomicAdd(out_cnt, 1);
  out_cols[pos] = j;
  out_par[pos] = par;
}

// dissolve claimed trees on the slab; reset keys whose argmin row leaves
__global__ void k_sh_dissolve(int32_t ncols, uint64_t* key, int64_t* v, uint8_t* rch,
                              const int64_t* dc, const int32_t* tree_par, const int32_t* root_row,
                              const uint8_t* claimed, int64_t D) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  if (rch[j]) {
    if (claimed[root_row[tree_par[j]]]) {
      v[j] -= D - dc[j];
      rch[j] = 0;
      key[j] = KMB_KEY_INF;
    }
  } else if (key[j] != KMB_KEY_INF && claimed[root_row[key_row(key[j])]]) {
    key[j] = KMB_KEY_INF;
  }
}

__global__ void k_sh_finish(int32_t ncols, int64_t* v, const uint8_t* rch, const int64_t* dc,
                            int64_t D) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ncols && rch[j]) v[j] -= D - dc[j];
}

__global__ void k_sh_cost(const int32_t* C, int64_t ld, int32_t n, int32_t col_begin, int32_t ncols,
                          const int32_t* row_to_col, unsigned long long* out) {
  int64_t s = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = row_to_col[i] - col_begin;
    if (j >= 0 && j < ncols) s += C[static_cast<int64_t>(i) * ld + j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(s));
}

}  // namespace kmb

namespace {

// ncclUniqueId is a struct of 128 bytes passed by value
struct NcclId {
  char internal[128];
};
typedef int (*nccl_init_rank_fn)(void**, int, NcclId, int);

struct NcclLib {
  void* h = nullptr;
  int (*get_id)(NcclId*) = nullptr;
  nccl_init_rank_fn init_rank = nullptr;
  int (*allreduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*allgather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*destroy)(void*) = nullptr;
  const char* (*errstr)(int) = nullptr;
  bool load(std::string* err) {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      *err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return false;
    }
    get_id = reinterpret_cast<int (*)(NcclId*)>(dlsym(h, "ncclGetUniqueId"));
    init_rank = reinterpret_cast<nccl_init_rank_fn>(dlsym(h, "ncclCommInitRank"));
    allreduce = reinterpret_cast<decltype(allreduce)>(dlsym(h, "ncclAllReduce"));
    allgather = reinterpret_cast<decltype(allgather)>(dlsym(h, "ncclAllGather"));
    destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    errstr = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    if (!get_id || !init_rank || !allreduce || !allgather || !destroy) {
      *err = "libnccl.so.2 lacks a required symbol";
      return false;
    }
    return true;
  }
};
NcclLib g_nccl;

// enum values from nccl.h (stable ABI): ncclInt64 = 4, ncclUint8 = 1, ncclMin = 3
constexpr int kNcclInt64 = 4, kNcclUint8 = 1, kNcclMin = 3;

struct NcclExchange : kmb::Exchange {
  void* comm = nullptr;
  cudaStream_t st = nullptr;
  int64_t* dbuf = nullptr;
  size_t dcap = 0;
  ~NcclExchange() override {
    if (comm) g_nccl.destroy(comm);
    if (dbuf) cudaFree(dbuf);
  }
  bool ensure(size_t bytes) {
    if (bytes <= dcap) return true;
    if (dbuf) cudaFree(dbuf);
    dcap = 0;
    if (cudaMalloc(&dbuf, bytes) != cudaSuccess) return false;
    dcap = bytes;
    return true;
  }
  int allreduce_min(int64_t* p, int32_t count) override {
    const size_t b = static_cast<size_t>(count) * 8;
    if (!ensure(b)) return -1;
    if (cudaMemcpyAsync(dbuf, p, b, cudaMemcpyHostToDevice, st) != cudaSuccess) return -1;
    if (g_nccl.allreduce(dbuf, dbuf, count, kNcclInt64, kNcclMin, comm, st) != 0) return -1;
    if (cudaMemcpyAsync(p, dbuf, b, cudaMemcpyDeviceToHost, st) != cudaSuccess) return -1;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : -1;
  }
  int allgather(const void* s, int64_t bytes, void* r) override {
    const size_t total = static_cast<size_t>(bytes) * nranks;
    if (!ensure(total + bytes)) return -1;
    char* send = reinterpret_cast<char*>(dbuf) + total;
    if (cudaMemcpyAsync(send, s, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return -1;
    if (g_nccl.allgather(send, dbuf, bytes, kNcclUint8, comm, st) != 0) return -1;
    if (cudaMemcpyAsync(r, dbuf, total, cudaMemcpyDeviceToHost, st) != cudaSuccess) return -1;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : -1;
  }
};

}  // namespace

namespace {

int sfail(int code, const std::string& m) {
  kmb::set_last_error(m);
  return code;
}

template <class T>
struct DArr {
  T* p = nullptr;
  explicit DArr(size_t n) {
    if (cudaMalloc(&p, sizeof(T) * (n ? n : 1)) != cudaSuccess) p = nullptr;
  }
  ~DArr() {
    if (p) cudaFree(p);
  }
  DArr(const DArr&) = delete;
};


// CUDA slab operations for kmb::sharded_solve (kmb_shard_proto.h)
struct CudaSlabOps {
  cudaStream_t st;
  int32_t n, ncols;
  int64_t lds;
  std::string err;
  DArr<int32_t> C, rows, tree, cols, pars, cnt, status, root, r2c;
  DArr<int64_t> v, dc, drowmin, ws;
  DArr<uint64_t> key;
  DArr<uint8_t> rch, claimed;
  DArr<unsigned long long> mn, cost_acc;
  int GB;
  CudaSlabOps(cudaStream_t s, int32_t n_, int32_t nc_)
      : st(s), n(n_), ncols(nc_), lds((nc_ + 3) & ~3),
        C(static_cast<size_t>(n_) * std::max<int64_t>((nc_ + 3) & ~3, 1)), rows(n_), tree(nc_),
        cols(nc_), pars(nc_), cnt(1), status(1), root(n_), r2c(n_), v(nc_), dc(nc_), drowmin(n_),
        ws(n_), key(nc_), rch(nc_), claimed(n_), mn(1), cost_acc(1),
        GB(std::max(1, (nc_ + 255) / 256)) {}
  bool ok() const {
    return C.p && rows.p && tree.p && cols.p && pars.p && cnt.p && status.p && root.p && r2c.p &&
           v.p && dc.p && drowmin.p && ws.p && key.p && rch.p && claimed.p && mn.p && cost_acc.p;
  }
  int chk(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return 0;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return -1;
  }
  int load(const int32_t* slab, int64_t ld) {
    if (ncols > 0 &&
        chk(cudaMemcpy2DAsync(C.p, lds * 4, slab, ld * 4, static_cast<size_t>(ncols) * 4, n,
                              cudaMemcpyDefault, st), "slab copy"))
      return -1;
    if (chk(cudaMemsetAsync(key.p, 0xff, static_cast<size_t>(ncols) * 8, st), "init")) return -1;
    if (chk(cudaMemsetAsync(v.p, 0, static_cast<size_t>(ncols) * 8, st), "init")) return -1;
    if (chk(cudaMemsetAsync(rch.p, 0, ncols, st), "init")) return -1;
    return chk(cudaMemsetAsync(status.p, 0, 4, st), "init");
  }
  int rowmin_(int64_t* out, int32_t* hstatus) {
    if (ncols == 0) {
      for (int32_t i = 0; i < n; ++i) out[i] = kmb::kShardInf;
      *hstatus = 0;
      return 0;
    }
    kmb::k_sh_rowmin<<<std::min<int>(1024, (n + 7) / 8), 256, 0, st>>>(C.p, lds, n, ncols, drowmin.p,
                                                                       status.p);
    if (chk(cudaGetLastError(), "k_sh_rowmin")) return -1;
    if (chk(cudaMemcpyAsync(out, drowmin.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, st), "d2h"))
      return -1;
    if (chk(cudaMemcpyAsync(hstatus, status.p, 4, cudaMemcpyDeviceToHost, st), "d2h")) return -1;
    return chk(cudaStreamSynchronize(st), "sync");
  }
  int rowmin(int64_t* out, int32_t* hstatus) { return rowmin_(out, hstatus); }
  int relax(const int32_t* hrows, const int64_t* hws, int32_t c, bool set_v, int64_t* lmin) {
    if (c) {
      if (chk(cudaMemcpyAsync(rows.p, hrows, static_cast<size_t>(c) * 4, cudaMemcpyHostToDevice, st), "h2d") ||
          chk(cudaMemcpyAsync(ws.p, hws, static_cast<size_t>(c) * 8, cudaMemcpyHostToDevice, st), "h2d"))
        return -1;
    }
    if (chk(cudaMemsetAsync(mn.p, 0xff, 8, st), "memset")) return -1;
    if (ncols > 0)
      kmb::k_sh_relax<<<GB, 256, 0, st>>>(C.p, lds, ncols, rows.p, ws.p, c, key.p, v.p, rch.p,
                                           set_v ? 1 : 0, v.p, mn.p);
    if (chk(cudaGetLastError(), "k_sh_relax")) return -1;
    unsigned long long h = ~0ull;
    if (chk(cudaMemcpyAsync(&h, mn.p, 8, cudaMemcpyDeviceToHost, st), "d2h") ||
        chk(cudaStreamSynchronize(st), "sync"))
      return -1;
    *lmin = h == ~0ull ? kmb::kShardInf : static_cast<int64_t>(h);
    return 0;
  }
  int absorb(int64_t D, int32_t* hcols, int32_t* hpars, int32_t* na) {
    *na = 0;
    if (ncols == 0) return 0;
    if (chk(cudaMemsetAsync(cnt.p, 0, 4, st), "memset")) return -1;
    kmb::k_sh_absorb<<<GB, 256, 0, st>>>(ncols, key.p, v.p, rch.p, dc.p, tree.p, D, cols.p, pars.p,
                                          cnt.p);
    if (chk(cudaGetLastError(), "k_sh_absorb")) return -1;
    if (chk(cudaMemcpyAsync(na, cnt.p, 4, cudaMemcpyDeviceToHost, st), "d2h") ||
        chk(cudaStreamSynchronize(st), "sync"))
      return -1;
    if (*na) {
      if (chk(cudaMemcpyAsync(hcols, cols.p, static_cast<size_t>(*na) * 4, cudaMemcpyDeviceToHost, st), "d2h") ||
          chk(cudaMemcpyAsync(hpars, pars.p, static_cast<size_t>(*na) * 4, cudaMemcpyDeviceToHost, st), "d2h") ||
          chk(cudaStreamSynchronize(st), "sync"))
        return -1;
    }
    return 0;
  }
  int reached(uint8_t* h) {
    if (ncols == 0) return 0;
    if (chk(cudaMemcpyAsync(h, rch.p, ncols, cudaMemcpyDeviceToHost, st), "d2h")) return -1;
    return chk(cudaStreamSynchronize(st), "sync");
  }
  int dissolve(const int32_t* hroot, const uint8_t* hcl, int64_t D) {
    if (ncols == 0) return 0;
    if (chk(cudaMemcpyAsync(root.p, hroot, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "h2d") ||
        chk(cudaMemcpyAsync(claimed.p, hcl, n, cudaMemcpyHostToDevice, st), "h2d"))
      return -1;
    kmb::k_sh_dissolve<<<GB, 256, 0, st>>>(ncols, key.p, v.p, rch.p, dc.p, tree.p, root.p,
                                            claimed.p, D);
    return chk(cudaGetLastError(), "k_sh_dissolve");
  }
  int finish(int64_t D, int64_t* v_out) {
    if (ncols == 0) return 0;
    kmb::k_sh_finish<<<GB, 256, 0, st>>>(ncols, v.p, rch.p, dc.p, D);
    if (chk(cudaGetLastError(), "k_sh_finish")) return -1;
    if (v_out && chk(cudaMemcpyAsync(v_out, v.p, static_cast<size_t>(ncols) * 8, cudaMemcpyDefault, st), "d2h"))
      return -1;
    return chk(cudaStreamSynchronize(st), "sync");
  }
  int cost(const int32_t* hr2c, int64_t* part) {
    *part = 0;
    if (ncols == 0) return 0;
    if (chk(cudaMemcpyAsync(r2c.p, hr2c, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "h2d") ||
        chk(cudaMemsetAsync(cost_acc.p, 0, 8, st), "memset"))
      return -1;
    kmb::k_sh_cost<<<std::max(1, std::min<int>(148, (n + 255) / 256)), 256, 0, st>>>(
        C.p, lds, n, col_begin_, ncols, r2c.p, cost_acc.p);
    if (chk(cudaGetLastError(), "k_sh_cost")) return -1;
    unsigned long long h = 0;
    if (chk(cudaMemcpyAsync(&h, cost_acc.p, 8, cudaMemcpyDeviceToHost, st), "d2h") ||
        chk(cudaStreamSynchronize(st), "sync"))
      return -1;
    *part = static_cast<int64_t>(h);
    return 0;
  }
  int32_t col_begin_ = 0;
};

}  // namespace

extern "C" {

int kmb_nccl_unique_id(uint8_t* out128) {
  std::string err;
  if (!g_nccl.load(&err)) return sfail(KMB_ECUDA, "kmb_nccl_unique_id: " + err);
  NcclId id;
  if (g_nccl.get_id(&id) != 0) return sfail(KMB_ECUDA, "kmb_nccl_unique_id: ncclGetUniqueId failed");
  std::memcpy(out128, id.internal, 128);
  return KMB_OK;
}

int kmb_shard_init_nccl(kmb_context* c, int32_t nranks, int32_t rank, const uint8_t* id128) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks || !id128)
    return sfail(KMB_EINVAL, "kmb_shard_init_nccl: bad arguments");
  std::string err;
  if (!g_nccl.load(&err)) return sfail(KMB_ECUDA, "kmb_shard_init_nccl: " + err);
  cudaSetDevice(kmb::context_device(c));
  auto ex = std::make_unique<NcclExchange>();
  ex->nranks = nranks;
  ex->rank = rank;
  ex->st = kmb::context_stream(c);
  NcclId id;
  std::memcpy(id.internal, id128, 128);
  const int rc = g_nccl.init_rank(&ex->comm, nranks, id, rank);
  if (rc != 0)
    return sfail(KMB_ECUDA, std::string("kmb_shard_init_nccl: ncclCommInitRank: ") +
                                (g_nccl.errstr ? g_nccl.errstr(rc) : "error"));
  kmb::context_exchange(c) = std::move(ex);
  return KMB_OK;
}

int kmb_shard_init_callbacks(kmb_context* c, int32_t nranks, int32_t rank,
                             kmb_allreduce_min_i64_fn allreduce_min, kmb_allgather_fn allgather,
                             void* user) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks || !allreduce_min || !allgather)
    return sfail(KMB_EINVAL, "kmb_shard_init_callbacks: bad arguments");
  auto ex = std::make_unique<kmb::CallbackExchange>();
  ex->nranks = nranks;
  ex->rank = rank;
  ex->ar = allreduce_min;
  ex->ag = allgather;
  ex->user = user;
  kmb::context_exchange(c) = std::move(ex);
  return KMB_OK;
}

int kmb_solve_sharded_i32(kmb_context* c, const int32_t* slab, int32_t n, int64_t ld,
                          int32_t col_begin, int32_t ncols, int32_t seed, int32_t* row_to_col,
                          int64_t* u_out, int64_t* v_slab, int64_t* total_cost, kmb_stats* stats) {
  const char* who = "kmb_solve_sharded_i32";
  if (!c) return sfail(KMB_EINVAL, "kmb_solve_sharded_i32: NULL context");
  auto& exp = kmb::context_exchange(c);
  if (!exp) return sfail(KMB_EINVAL, "kmb_solve_sharded_i32: call kmb_shard_init_* first");
  // A local failure before the protocol starts is still voted on in its first
  // collective (kmb_shard_proto.h), so the peer ranks return an error instead
  // of waiting forever in their next allreduce.
  if (n <= 0 || ncols < 0 || ld < ncols || !slab || col_begin < 0 || col_begin + ncols > n ||
      (seed != KMB_SEED_KM && seed != KMB_SEED_BATCHED)) {
    int64_t vote = kmb::kShardPeerFail;
    exp->allreduce_min(&vote, 1);
    return sfail(KMB_EINVAL, "kmb_solve_sharded_i32: bad arguments");
  }
  cudaSetDevice(kmb::context_device(c));
  CudaSlabOps ops(kmb::context_stream(c), n, ncols);
  ops.col_begin_ = col_begin;
  std::string pre;
  if (!ops.ok()) pre = std::string(who) + ": out of device memory";
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, ops.st);
  if (pre.empty() && ops.load(slab, ld) != 0) pre = std::string(who) + ": " + ops.err;
  kmb::ShardResult res;
  std::string err;
  const int rc = kmb::sharded_solve(ops, *exp, n, col_begin, ncols, seed, row_to_col, u_out, v_slab,
                                    &res, &err, pre);
  cudaEventRecord(e1, ops.st);
  cudaStreamSynchronize(ops.st);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc == KMB_ENEGATIVE) return sfail(rc, std::string(who) + ": costs must be nonnegative");
  if (rc == KMB_ERANGE) return sfail(rc, std::string(who) + ": cost exceeds the device range [0, 2^29)");
  if (rc == -2) return sfail(KMB_EINTERNAL, std::string(who) + ": " + err);
  if (rc != 0) return sfail(KMB_ECUDA, std::string(who) + ": " + err);
  if (total_cost) *total_cost = res.total_cost;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->phases = res.epochs;
    stats->dual_steps = res.dual_steps;
    stats->rows_scanned = res.rows_scanned;
    stats->rounds = res.rounds;
    stats->cost_bytes_read = 4ll * ncols * (res.rows_scanned + n);
    stats->seconds = ms * 1e-3;  // wall of the whole collective solve on this rank's stream
    stats->converged = 1;
    stats->engine = 7;
  }
  return KMB_OK;
}

}  // extern "C"
