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

// Every rank must reach the same collectives, so a rank-local failure never
// returns on its own: it is remembered (lfail) and voted on at the next
// collective, which carries a failure flag (the min-slack allreduce a second
// word, the count allgathers a negative count), and then every rank returns
// -1 together.  A failure before the protocol starts (bad arguments, out of
// memory, slab load) enters as `pre_fail` and is voted on in the first
// collective.  Only a failing collective itself returns at once.
//
// Returns 0, a positive kmb_status (invalid input), -1 (ops / exchange
// failure on this or another rank, message in *err), -2 (engine invariant).
constexpr int64_t kShardPeerFail = -100;  // vote value of a rank-local failure

template <class Ops>
int sharded_solve(Ops& ops, ShardExchange& ex, int32_t n, int32_t col_begin, int32_t ncols,
                  int32_t seed, int32_t* row_to_col, int64_t* u_out, int64_t* v_slab,
                  ShardResult* res, std::string* err, const std::string& pre_fail = "") {
  const int NR = ex.nranks;
  const size_t nn = static_cast<size_t>(n > 0 ? n : 0), nc = static_cast<size_t>(ncols > 0 ? ncols : 0);
  std::string lfail = pre_fail;
  auto failed_everywhere = [&]() {
    *err = lfail.empty() ? std::string("another rank failed") : lfail;
    return -1;
  };
#define KMB_OK_OR(x, what)          \
  do {                              \
    if ((x) != 0) {                 \
      *err = std::string(what) + (ops.err.empty() ? "" : ": " + ops.err); \
      return -1;                    \
    }                               \
  } while (0)
#define KMB_TRY(x, what)                                                        \
  do {                                                                          \
    if ((x) != 0 && lfail.empty())                                              \
      lfail = std::string(what) + (ops.err.empty() ? "" : ": " + ops.err);      \
  } while (0)
  std::vector<int64_t> u(nn, 0), w(nn, 0), rowmin(nn, kShardInf);
  std::vector<int32_t> root(nn), match_row(nn, -1), match_col(nc, -1), tree_par(nc, -1);
  std::vector<int32_t> rows;
  int32_t status = 0;
  if (lfail.empty()) KMB_TRY(ops.rowmin(rowmin.data(), &status), "slab row minima");
  {  // validation is global: any rank's bad entry (or local failure) fails every rank
    int64_t bad = lfail.empty() ? -static_cast<int64_t>(status) : kShardPeerFail;
    KMB_OK_OR(ex.allreduce_min(&bad, 1), "exchange (validation)");
    if (bad == kShardPeerFail) return failed_everywhere();
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
    int64_t mv[2] = {kShardInf, 0};  // min slack', failure flag
    KMB_TRY(ops.relax(rows.data() + head, ws.data(), cnt, first && seed == 1, &mv[0]), "slab relax");
    first = false;
    res->rows_scanned += cnt;
    head = rows.size();
    if (!lfail.empty()) mv[1] = -1;
    KMB_OK_OR(ex.allreduce_min(mv, 2), "exchange (min slack)");  // :203-206
    if (mv[1] < 0) return failed_everywhere();
    const int64_t m = mv[0];
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
    KMB_TRY(ops.absorb(D, cols.data(), pars.data(), &na), "slab absorb");
    if (!lfail.empty()) na = 0;
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
    int64_t mine = lfail.empty() ? static_cast<int64_t>(out.size() / 4) : -1;
    KMB_OK_OR(ex.allgather(&mine, 8, counts.data()), "exchange (entry counts)");
    int64_t maxc = 0;
    for (int64_t x : counts) {
      if (x < 0) return failed_everywhere();
      maxc = std::max(maxc, x);
    }
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
    KMB_TRY(ops.reached(rch.data()), "slab reached");
    std::vector<int64_t> tout;  // (global col, parent) of claimed trees' columns
    for (int32_t j = 0; lfail.empty() && j < ncols; ++j)
      if (rch[j] && claimed(root[tree_par[j]])) tout.insert(tout.end(), {col_begin + j, tree_par[j]});
    int64_t tc = lfail.empty() ? static_cast<int64_t>(tout.size() / 2) : -1;
    KMB_OK_OR(ex.allgather(&tc, 8, counts.data()), "exchange (tree counts)");
    int64_t tmax = 0;
    for (int64_t x : counts) {
      if (x < 0) return failed_everywhere();
      tmax = std::max(tmax, x);
    }
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
    KMB_TRY(ops.dissolve(root.data(), cl.data(), D), "slab dissolve");  // voted next round
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
  KMB_TRY(ops.finish(D, v_slab), "slab finish");
  int64_t part[2] = {0, 0};  // partial cost, failure flag
  if (lfail.empty()) KMB_TRY(ops.cost(match_row.data(), &part[0]), "slab cost");
  if (!lfail.empty()) part[1] = -1;
  std::vector<int64_t> parts(2 * NR);
  KMB_OK_OR(ex.allgather(part, 16, parts.data()), "exchange (cost)");
  res->total_cost = 0;
  for (int r = 0; r < NR; ++r) {
    if (parts[2 * r + 1] < 0) return failed_everywhere();
    res->total_cost += parts[2 * r];
  }
  if (row_to_col) std::copy(match_row.begin(), match_row.end(), row_to_col);
  if (u_out) std::copy(u.begin(), u.end(), u_out);
#undef KMB_OK_OR
#undef KMB_TRY
  return 0;
}

}  // namespace kmb
