// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim around the UNMODIFIED reference solver, compiled directly from
// /root/reference/proj/src/{core,hungarian}.cpp by oracle/Makefile into
// oracle/_ref/libotref.so.  Only tests/, __graft_entry__.smoke() and the
// bench.py cpu_baseline / --impl reference legs load it, as the checker and
// as the CPU baseline.  The reference entry points wrapped here:
//   ot::solve_km           hungarian.hpp:39-40, hungarian.cpp:55-136
//   ot::solve_batched_km   hungarian.hpp:53-56, hungarian.cpp:313-381
//   ot::quantize_costs     hungarian.hpp:35,   hungarian.cpp:33-53
//   ot::solve_auction      auction.hpp:30-32,  auction.cpp:186-199
//   ot::solve_auction_scaled auction.hpp:48-50, auction.cpp:201-229
//   ot::build_instance     datasets.hpp,       datasets.cpp:184-214
// Errors: std::invalid_argument -> 1, std::logic_error -> 2, other -> 3;
// the message is kept in a thread-local buffer (otref_last_error).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include "ot/auction.hpp"
#include "ot/core.hpp"
#include "ot/datasets.hpp"
#include "ot/hungarian.hpp"

namespace {

thread_local std::string g_err;

ot::OTInstance make_unit(const int64_t* cost, int32_t n) {
  ot::OTInstance inst;
  inst.n = inst.m = n;
  inst.cost.assign(cost, cost + static_cast<size_t>(n) * (n > 0 ? n : 0));
  inst.supplies.assign(n > 0 ? n : 0, 1);
  inst.demands.assign(n > 0 ? n : 0, 1);
  inst.name = "otref";
  return inst;
}

struct ResultOut {
  int32_t* row_to_col;
  int64_t* total_cost;
  double* objective;
  int64_t* iterations;
  int32_t* exact_converged;  // [exact, converged]
  double* wall;
};

void fill(const ot::OTInstance& inst, const ot::SolveResult& res, const ResultOut& o) {
  if (o.row_to_col) {
    for (int32_t i = 0; i < inst.n; ++i) o.row_to_col[i] = -1;
    for (const auto& e : res.flow.entries()) o.row_to_col[e.i] = e.j;
  }
  if (o.total_cost) {
    int64_t t = 0;
    for (const auto& e : res.flow.entries()) t += inst.cost_at(e.i, e.j);
    *o.total_cost = t;
  }
  if (o.objective) *o.objective = res.objective;
  if (o.iterations) *o.iterations = res.iterations;
  if (o.exact_converged) {
    o.exact_converged[0] = res.exact ? 1 : 0;
    o.exact_converged[1] = res.converged ? 1 : 0;
  }
  if (o.wall) *o.wall = res.wall_seconds;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // namespace

extern "C" {

const char* otref_last_error(void) { return g_err.c_str(); }

// supplies/demands may be NULL (unit caps); otherwise n entries each, so the
// reference's own validation (core.cpp:30-55, hungarian.cpp:15-21) is exercised.
int otref_solve_km(const int64_t* cost, int32_t n, const int64_t* supplies,
                   const int64_t* demands, double time_budget_s, int64_t* u,
                   int64_t* v, int32_t* row_to_col, int64_t* total_cost,
                   double* objective, int64_t* iterations,
                   int32_t* exact_converged, double* wall) {
  return guarded([&] {
    ot::OTInstance inst = make_unit(cost, n);
    if (supplies) inst.supplies.assign(supplies, supplies + n);
    if (demands) inst.demands.assign(demands, demands + n);
    ot::DualPotentials d;
    ot::Matching m;
    const ot::SolveResult res = ot::solve_km(inst, &d, &m, time_budget_s);
    if (u && !d.u.empty()) std::memcpy(u, d.u.data(), sizeof(int64_t) * n);
    if (v && !d.v.empty()) std::memcpy(v, d.v.data(), sizeof(int64_t) * n);
    fill(inst, res, {row_to_col, total_cost, objective, iterations, exact_converged, wall});
  });
}

int otref_solve_batched_km(const int64_t* cost, int32_t n, const int64_t* supplies,
                           const int64_t* demands, int64_t B, double time_budget_s,
                           int64_t* u, int64_t* v, int64_t* chat,
                           int32_t* row_to_col, int64_t* total_cost,
                           double* objective, int64_t* iterations,
                           int32_t* exact_converged, double* wall) {
  return guarded([&] {
    ot::OTInstance inst = make_unit(cost, n);
    if (supplies) inst.supplies.assign(supplies, supplies + n);
    if (demands) inst.demands.assign(demands, demands + n);
    ot::BatchedKMConfig cfg;
    cfg.B = B;
    cfg.time_budget_s = time_budget_s;
    ot::DualPotentials d;
    ot::QuantizedCosts q;
    const ot::SolveResult res = ot::solve_batched_km(inst, cfg, &d, &q);
    if (u && !d.u.empty()) std::memcpy(u, d.u.data(), sizeof(int64_t) * n);
    if (v && !d.v.empty()) std::memcpy(v, d.v.data(), sizeof(int64_t) * n);
    if (chat && !q.chat.empty()) std::memcpy(chat, q.chat.data(), sizeof(int64_t) * q.chat.size());
    fill(inst, res, {row_to_col, total_cost, objective, iterations, exact_converged, wall});
  });
}

int otref_quantize_costs(const int64_t* cost, int64_t count, int64_t B,
                         int64_t* chat, int64_t* N, int32_t* lossless) {
  return guarded([&] {
    std::vector<int64_t> c(cost, cost + count);
    const ot::QuantizedCosts q = ot::quantize_costs(c, B);
    if (chat && !q.chat.empty()) std::memcpy(chat, q.chat.data(), sizeof(int64_t) * q.chat.size());
    if (N) *N = q.N;
    if (lossless) *lossless = q.lossless ? 1 : 0;
  });
}

// ot::build_instance (datasets.cpp:184-214): C_ij = llround(scale * ||a_i - b_j||)
// for unit-weight point clouds a (n x dim) and b (m x dim); the pin for the GPU
// cost construction (csrc/kmb_costs.cu).
int otref_build_instance(const double* a, int32_t n, const double* b, int32_t m, int32_t dim,
                         double scale, int64_t* cost) {
  return guarded([&] {
    ot::PointCloudDistribution sa, sb;
    sa.dim = sb.dim = dim;
    sa.coords.assign(a, a + static_cast<size_t>(n) * dim);
    sb.coords.assign(b, b + static_cast<size_t>(m) * dim);
    sa.weights.assign(n, 1);
    sb.weights.assign(m, 1);
    if (n != m) throw std::invalid_argument("otref_build_instance: unit weights need n == m");
    const ot::OTInstance inst = ot::build_instance(sa, sb, {scale}, "pts");
    std::memcpy(cost, inst.cost.data(), sizeof(int64_t) * inst.cost.size());
  });
}

// ot::solve_auction / ot::solve_auction_scaled (auction.cpp:186-229).
// scaled = 0: eps0 is AuctionConfig::epsilon (theta, eps_final unused);
// scaled = 1: AuctionScaledConfig{eps0, theta, eps_final}.  prices: n doubles.
int otref_solve_auction(const int64_t* cost, int32_t n, int32_t scaled, double eps0, double theta,
                        double eps_final, int64_t max_bids, double time_budget_s,
                        double* prices, int32_t* row_to_col, int64_t* total_cost,
                        double* objective, int64_t* iterations, int32_t* exact_converged,
                        double* wall) {
  return guarded([&] {
    ot::OTInstance inst = make_unit(cost, n);
    std::vector<double> p;
    ot::SolveResult res;
    if (scaled) {
      ot::AuctionScaledConfig cfg;
      cfg.epsilon0 = eps0;
      cfg.theta = theta;
      cfg.epsilon_final = eps_final;
      cfg.max_bids = max_bids;
      cfg.time_budget_s = time_budget_s;
      res = ot::solve_auction_scaled(inst, cfg, &p);
    } else {
      ot::AuctionConfig cfg;
      cfg.epsilon = eps0;
      cfg.max_bids = max_bids;
      cfg.time_budget_s = time_budget_s;
      res = ot::solve_auction(inst, cfg, &p);
    }
    if (prices && !p.empty()) std::memcpy(prices, p.data(), sizeof(double) * p.size());
    fill(inst, res, {row_to_col, total_cost, objective, iterations, exact_converged, wall});
  });
}

// CPU baseline helper: `batch` independent int32 instances (n x n each),
// solved with the reference solver (mode 0 = solve_km, 1 = solve_batched_km
// at the lossless B = max(N,1)) on `nthreads` threads (the reference is
// re-entrant: no mutable globals in core.cpp / hungarian.cpp).  Outputs (each
// optional): total cost per instance, and the duals u, v (batch x n each), so
// the caller can compare every instance bit for bit.  *wall_seconds is the
// wall time of the whole pool, and it INCLUDES each instance's int32 -> int64
// widening into an OTInstance (a 64 KiB copy for n = 128, well under 1% of a
// 3-4 ms solve); bench.cpp:95-121 times spec.run alone, so this rate is a
// slight underestimate of the reference's.
int otref_solve_many_i32(const int32_t* costs, int32_t batch, int32_t n,
                         int32_t mode, int32_t nthreads, int64_t* total_costs,
                         int64_t* u_out, int64_t* v_out, double* wall_seconds) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    std::atomic<int32_t> next{0};
    std::atomic<int> failed{0};
    std::string first_err;
    auto worker = [&] {
      std::vector<int64_t> buf(static_cast<size_t>(n) * n);
      for (;;) {
        const int32_t b = next.fetch_add(1);
        if (b >= batch) break;
        const int32_t* src = costs + static_cast<size_t>(b) * n * n;
        int64_t mx = 0;
        for (size_t k = 0; k < buf.size(); ++k) {
          buf[k] = src[k];
          if (buf[k] > mx) mx = buf[k];
        }
        try {
          ot::OTInstance inst = make_unit(buf.data(), n);
          ot::SolveResult res;
          ot::DualPotentials d;
          if (mode == 0) {
            res = ot::solve_km(inst, &d);
          } else {
            ot::BatchedKMConfig cfg;
            cfg.B = mx > 0 ? mx : 1;
            res = ot::solve_batched_km(inst, cfg, &d);
          }
          int64_t t = 0;
          for (const auto& e : res.flow.entries()) t += inst.cost_at(e.i, e.j);
          if (total_costs) total_costs[b] = t;
          const size_t o = static_cast<size_t>(b) * n;
          if (u_out && d.u.size() == static_cast<size_t>(n)) std::memcpy(u_out + o, d.u.data(), 8 * n);
          if (v_out && d.v.size() == static_cast<size_t>(n)) std::memcpy(v_out + o, d.v.data(), 8 * n);
        } catch (const std::exception&) {
          failed.store(1);
        }
      }
    };
    const int32_t nt = nthreads < 1 ? 1 : nthreads;
    std::vector<std::thread> pool;
    for (int32_t t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (wall_seconds)
      *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failed.load()) throw std::runtime_error("otref_solve_many_i32: a solve failed");
  });
}

}  // extern "C"
