// Host control loop of the column-sharded solve (kmb_shard.cu), templated on
// the slab operations so the exchange protocol is one piece of code:
//   * kmb_shard.cu instantiates it with CUDA slab kernels (the product);
//   * tests/cpp/shard_sim.cpp instantiates it with plain loops (TEST
//     INFRASTRUCTURE: simulated shards, run under torch.distributed gloo with
//     world_size 2 on CPU to check the protocol against the oracle).
//
// Rank r owns columns [col_begin, col_begin + ncols); the row side (u, w,
// root, match_row, reached-row list) is replicated and kept identical on every
// rank: every rank applies the same gathered entries in the same (rank-major,
// column-sorted) order.  The engine is the incremental-epoch search of
// kmb_solver.cu (hungarian.cpp:175-217 restated with lazy duals).
//
// Ops interface (all host-visible results):
//   int rowmin(int64_t* rowmin /*n*/, int32_t* status)
//   int relax(const int32_t* rows, const int64_t* ws, int32_t cnt, bool set_v,
//             int64_t* local_min /*INF if none*/)
//   int absorb(int64_t D, int32_t* cols, int32_t* pars, int32_t* na)
//   int reached(uint8_t* rch /*ncols*/)
//   int dissolve(const int32_t* root /*n*/, const uint8_t* claimed /*n*/, int64_t D)
//   int finish(int64_t D, int64_t* v_out /*ncols*/)
//   int cost(const int32_t* row_to_col /*n*/, int64_t* partial)
//   std::string err
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

namespace kmb {

struct ShardExchange {
  int nranks = 1, rank = 0;
  virtual ~ShardExchange() = default;
  virtual int allreduce_min(int64_t* host_inout, int32_t count) = 0;
  virtual int allgather(const void* host_send, int64_t bytes, void* host_recv) = 0;
};

struct ShardResult {
  int64_t epochs = 0, dual_steps = 0, rows_scanned = 0, rounds = 0, total_cost = 0;
};

constexpr int64_t kShardInf = 0x7FFFFFFFFFFFFFFFLL;

// Returns 0, a positive kmb_status (invalid input), or -1 (ops / exchange
// failure, message in *err), -2 (engine invariant).
template <class Ops>
int sharded_solve(Ops& ops, ShardExchange& ex, int32_t n, int32_t col_begin, int32_t ncols,
                  int32_t seed, int32_t* row_to_col, int64_t* u_out, int64_t* v_slab,
                  ShardResult* res, std::string* err) {
  const int NR = ex.nranks;
  const size_t nn = static_cast<size_t>(n), nc = static_cast<size_t>(ncols);
#define KMB_OK_OR(x, what)          \
  do {                              \
    if ((x) != 0) {                 \
      *err = std::string(what) + (ops.err.empty() ? "" : ": " + ops.err); \
      return -1;                    \
    }                               \
  } while (0)
  std::vector<int64_t> u(nn, 0), w(nn, 0), rowmin(nn, kShardInf);
  std::vector<int32_t> root(nn), match_row(nn, -1), match_col(nc, -1), tree_par(nc, -1);
  std::vector<int32_t> rows;
  int32_t status = 0;
  KMB_OK_OR(ops.rowmin(rowmin.data(), &status), "slab row minima");
  {  // validation is global: any rank's bad entry fails every rank
    int64_t bad = -static_cast<int64_t>(status);
    KMB_OK_OR(ex.allreduce_min(&bad, 1), "exchange (validation)");
    if (bad < 0) return static_cast<int>(-bad);
  }
  KMB_OK_OR(ex.allreduce_min(rowmin.data(), n), "exchange (row minima)");  // :323-327
  for (int32_t i = 0; i < n; ++i) {
    u[i] = seed == 1 ? rowmin[i] : 0;
    w[i] = u[i];
    root[i] = i;
    rows.push_back(i);
  }
  int64_t D = 0;
  int32_t matched = 0;
  size_t head = 0;
  std::vector<int32_t> cols(nc), pars(nc), order;
  std::vector<int64_t> ws, out, gathered, counts(NR);
  std::vector<int32_t> claim_col(nn, 0);
  std::vector<int64_t> claim_ep(nn, -1);
  bool first = true;
  while (matched < n) {
    ++res->rounds;
    // ---- relax the new rows over the slab, local min of unreached slack' ----
    const int32_t cnt = static_cast<int32_t>(rows.size() - head);
    ws.resize(cnt);
    for (int32_t r = 0; r < cnt; ++r) ws[r] = w[rows[head + r]];
    int64_t m = kShardInf;
    KMB_OK_OR(ops.relax(rows.data() + head, ws.data(), cnt, first && seed == 1, &m), "slab relax");
    first = false;
    res->rows_scanned += cnt;
    head = rows.size();
    KMB_OK_OR(ex.allreduce_min(&m, 1), "exchange (min slack)");  // :203-206
    if (m > D) {
      if (m == kShardInf) {
        *err = "no unreached column";
        return -2;
      }
      D = m;  // dual step (:207-215), lazy
      ++res->dual_steps;
    }
    // ---- absorb tight slab columns, entries for the replicated row side ----
    int32_t na = 0;
    KMB_OK_OR(ops.absorb(D, cols.data(), pars.data(), &na), "slab absorb");
    order.resize(na);
    for (int32_t k = 0; k < na; ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cols[a] < cols[b]; });
    out.clear();
    for (int32_t k : order) {
      const int32_t j = cols[k], par = pars[k];
      tree_par[j] = par;
      const int32_t rt = root[par];
      const int32_t i2 = match_col[j];
      if (i2 < 0) out.insert(out.end(), {1, col_begin + j, rt, 0});  // free column
      else out.insert(out.end(), {0, i2, u[i2] - D, rt});             // new row
    }
    int64_t mine = static_cast<int64_t>(out.size() / 4);
    KMB_OK_OR(ex.allgather(&mine, 8, counts.data()), "exchange (entry counts)");
    int64_t maxc = 0;
    for (int64_t x : counts) maxc = std::max(maxc, x);
    if (maxc == 0) continue;
    out.resize(static_cast<size_t>(maxc) * 4, 0);
    gathered.assign(static_cast<size_t>(maxc) * 4 * NR, 0);
    KMB_OK_OR(ex.allgather(out.data(), maxc * 32, gathered.data()), "exchange (entries)");
    std::vector<int32_t> free_cols, free_roots;
    for (int r = 0; r < NR; ++r)
      for (int64_t k = 0; k < counts[r]; ++k) {
        const int64_t* e = gathered.data() + (static_cast<size_t>(r) * maxc + k) * 4;
        if (e[0] == 0) {
          const int32_t i2 = static_cast<int32_t>(e[1]);
          w[i2] = e[2];
          root[i2] = static_cast<int32_t>(e[3]);
          rows.push_back(i2);
        } else {
          const int32_t col = static_cast<int32_t>(e[1]), rt = static_cast<int32_t>(e[2]);
          free_cols.push_back(col);
          free_roots.push_back(rt);
          if (claim_ep[rt] != res->epochs || col < claim_col[rt]) {
            claim_ep[rt] = res->epochs;
            claim_col[rt] = col;
          }
        }
      }
    if (free_cols.empty()) continue;

    // ---- epoch end: augment and dissolve the claimed trees ----
    const int64_t ep = res->epochs;
    auto claimed = [&](int32_t rt) { return claim_ep[rt] == ep; };
    std::vector<uint8_t> rch(nc, 0);
    KMB_OK_OR(ops.reached(rch.data()), "slab reached");
    std::vector<int64_t> tout;  // (global col, parent) of claimed trees' columns
    for (int32_t j = 0; j < ncols; ++j)
      if (rch[j] && claimed(root[tree_par[j]])) tout.insert(tout.end(), {col_begin + j, tree_par[j]});
    int64_t tc = static_cast<int64_t>(tout.size() / 2);
    KMB_OK_OR(ex.allgather(&tc, 8, counts.data()), "exchange (tree counts)");
    int64_t tmax = 0;
    for (int64_t x : counts) tmax = std::max(tmax, x);
    tout.resize(static_cast<size_t>(tmax) * 2, 0);
    std::vector<int64_t> tall(static_cast<size_t>(tmax) * 2 * NR);
    if (tmax) KMB_OK_OR(ex.allgather(tout.data(), tmax * 16, tall.data()), "exchange (trees)");
    std::vector<int32_t> tp_full(nn, -1);
    for (int r = 0; r < NR; ++r)
      for (int64_t k = 0; k < counts[r]; ++k) {
        const int64_t* e = tall.data() + (static_cast<size_t>(r) * tmax + k) * 2;
        tp_full[e[0]] = static_cast<int32_t>(e[1]);
      }
    std::vector<uint8_t> cl(nn, 0);
    for (int32_t i = 0; i < n; ++i) cl[i] = claimed(i) ? 1 : 0;
    KMB_OK_OR(ops.dissolve(root.data(), cl.data(), D), "slab dissolve");
    std::vector<int32_t> surv;
    for (int32_t i : rows) {
      if (claimed(root[i])) u[i] = w[i] + D;
      else surv.push_back(i);
    }
    for (size_t f = 0; f < free_cols.size(); ++f) {
      int32_t j = free_cols[f];
      if (claim_col[free_roots[f]] != j) continue;
      ++matched;
      for (;;) {
        const int32_t i = tp_full[j];
        const int32_t nx = match_row[i];
        match_row[i] = j;
        if (j >= col_begin && j < col_begin + ncols) match_col[j - col_begin] = i;
        if (nx < 0) break;
        j = nx;
      }
    }
    rows.swap(surv);
    head = 0;
    ++res->epochs;
  }
  KMB_OK_OR(ops.finish(D, v_slab), "slab finish");
  int64_t part = 0;
  KMB_OK_OR(ops.cost(match_row.data(), &part), "slab cost");
  std::vector<int64_t> parts(NR);
  KMB_OK_OR(ex.allgather(&part, 8, parts.data()), "exchange (cost)");
  res->total_cost = 0;
  for (int64_t x : parts) res->total_cost += x;
  if (row_to_col) std::copy(match_row.begin(), match_row.end(), row_to_col);
  if (u_out) std::copy(u.begin(), u.end(), u_out);
#undef KMB_OK_OR
  return 0;
}

}  // namespace kmb
