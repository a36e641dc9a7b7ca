// TEST INFRASTRUCTURE ONLY — simulated shards.  Instantiates the product's
// column-sharded protocol (paper_2005_01182_b200/csrc/kmb_shard_proto.h) with
// plain CPU loops in place of the CUDA slab kernels, so tests/test_sharded.py
// can run the exact exchange protocol under torch.distributed gloo with
// world_size 2 on a machine without a GPU and compare with the oracle.
// Never linked into libkmb.so.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "kmb_shard_proto.h"

namespace {

constexpr int64_t BIAS = int64_t{1} << 30;

struct CpuSlabOps {
  const int32_t* C;
  int64_t ld;
  int32_t n, ncols, col_begin;
  std::string err;
  std::vector<uint64_t> key;
  std::vector<int64_t> v, dc;
  std::vector<uint8_t> rch;
  std::vector<int32_t> tree;
  // failure injection (tests of the failure vote): op 1 rowmin, 2 relax,
  // 3 absorb, 4 reached, 5 dissolve, 6 finish, 7 cost fails on its fail_at-th call
  int32_t fail_op = 0, fail_at = 0, calls[8] = {};
  bool inject(int op) {
    if (op != fail_op || ++calls[op] != fail_at) return false;
    err = "injected failure";
    return true;
  }
  static uint64_t pack(int64_t val, int32_t row) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(val + BIAS)) << 32) | static_cast<uint32_t>(row);
  }
  static int64_t kval(uint64_t k) { return static_cast<int64_t>(k >> 32) - BIAS; }
  static int32_t krow(uint64_t k) { return static_cast<int32_t>(k & 0xffffffffu); }
  int rowmin(int64_t* out, int32_t* status) {
    if (inject(1)) return -1;
    *status = 0;
    for (int32_t i = 0; i < n; ++i) {
      int64_t lo = kmb::kShardInf;
      for (int32_t j = 0; j < ncols; ++j) {
        const int32_t c = C[i * ld + j];
        if (c < 0) *status = 2;
        else if (c >= (1 << 29) && *status == 0) *status = 3;
        lo = std::min<int64_t>(lo, c);
      }
      out[i] = lo;
    }
    return 0;
  }
  int relax(const int32_t* rows, const int64_t* ws, int32_t cnt, bool set_v, int64_t* lmin) {
    if (inject(2)) return -1;
    int64_t m = kmb::kShardInf;
    for (int32_t j = 0; j < ncols; ++j) {
      for (int32_t r = 0; r < cnt; ++r) {
        const uint64_t k = pack(static_cast<int64_t>(C[rows[r] * ld + j]) - ws[r], rows[r]);
        if (k < key[j]) key[j] = k;
      }
      if (set_v) v[j] = kval(key[j]);
      if (!rch[j]) m = std::min(m, kval(key[j]) - v[j]);
    }
    *lmin = m;
    return 0;
  }
  int absorb(int64_t D, int32_t* cols, int32_t* pars, int32_t* na) {
    if (inject(3)) return -1;
    *na = 0;
    for (int32_t j = ncols - 1; j >= 0; --j) {  // reverse: the protocol must not rely on order
      if (rch[j] || kval(key[j]) - v[j] != D) continue;
      rch[j] = 1;
      dc[j] = D;
      tree[j] = krow(key[j]);
      cols[*na] = j;
      pars[*na] = tree[j];
      ++*na;
    }
    return 0;
  }
  int reached(uint8_t* out) {
    if (inject(4)) return -1;
    if (!rch.empty()) std::memcpy(out, rch.data(), rch.size());
    return 0;
  }
  int dissolve(const int32_t* root, const uint8_t* claimed, int64_t D) {
    if (inject(5)) return -1;
    for (int32_t j = 0; j < ncols; ++j) {
      if (rch[j]) {
        if (claimed[root[tree[j]]]) {
          v[j] -= D - dc[j];
          rch[j] = 0;
          key[j] = ~0ull;
        }
      } else if (key[j] != ~0ull && claimed[root[krow(key[j])]]) {
        key[j] = ~0ull;
      }
    }
    return 0;
  }
  int finish(int64_t D, int64_t* vout) {
    if (inject(6)) return -1;
    for (int32_t j = 0; j < ncols; ++j) {
      if (rch[j]) v[j] -= D - dc[j];
      if (vout) vout[j] = v[j];
    }
    return 0;
  }
  int cost(const int32_t* r2c, int64_t* part) {
    if (inject(7)) return -1;
    int64_t s = 0;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t j = r2c[i] - col_begin;
      if (j >= 0 && j < ncols) s += C[i * ld + j];
    }
    *part = s;
    return 0;
  }
};

typedef int (*ar_fn)(int64_t*, int32_t, void*);
typedef int (*ag_fn)(const void*, int64_t, void*, void*);

struct CbExchange : kmb::ShardExchange {
  ar_fn ar = nullptr;
  ag_fn ag = nullptr;
  int allreduce_min(int64_t* p, int32_t c) override { return ar(p, c, nullptr); }
  int allgather(const void* s, int64_t b, void* r) override { return ag(s, b, r, nullptr); }
};

}  // namespace

// fail_op 8: a failure before the protocol starts (the entry point's
// pre-protocol vote); 1..7: CpuSlabOps::inject.
extern "C" int shardsim_solve_fail(const int32_t* slab, int32_t n, int64_t ld, int32_t col_begin,
                                   int32_t ncols, int32_t seed, int32_t nranks, int32_t rank,
                                   ar_fn ar, ag_fn ag, int32_t* r2c, int64_t* u, int64_t* v,
                                   int64_t* out4, int32_t fail_op, int32_t fail_at) {
  CpuSlabOps ops{slab, ld, n, ncols, col_begin, {}, std::vector<uint64_t>(ncols, ~0ull),
                 std::vector<int64_t>(ncols, 0), std::vector<int64_t>(ncols, 0),
                 std::vector<uint8_t>(ncols, 0), std::vector<int32_t>(ncols, -1)};
  ops.fail_op = fail_op;
  ops.fail_at = fail_at;
  CbExchange ex;
  ex.nranks = nranks;
  ex.rank = rank;
  ex.ar = ar;
  ex.ag = ag;
  kmb::ShardResult res;
  std::string err;
  const int rc = kmb::sharded_solve(ops, ex, n, col_begin, ncols, seed, r2c, u, v, &res, &err,
                                    fail_op == 8 ? "injected pre-protocol failure" : "");
  out4[0] = res.total_cost;
  out4[1] = res.dual_steps;
  out4[2] = res.epochs;
  out4[3] = res.rounds;
  return rc;
}

extern "C" int shardsim_solve(const int32_t* slab, int32_t n, int64_t ld, int32_t col_begin,
                              int32_t ncols, int32_t seed, int32_t nranks, int32_t rank, ar_fn ar,
                              ag_fn ag, int32_t* r2c, int64_t* u, int64_t* v, int64_t* out4) {
  return shardsim_solve_fail(slab, n, ld, col_begin, ncols, seed, nranks, rank, ar, ag, r2c, u, v,
                             out4, 0, 0);
}
