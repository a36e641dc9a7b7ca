// kmb_ot.hpp — reference-side drop-in over the kmb C ABI (include/kmb.h).
//
// Include AFTER the reference's own headers ("ot/core.hpp", "ot/hungarian.hpp")
// and link libkmb.so.  It adds, in namespace ot, functions with the exact
// signatures and semantics of the reference solvers:
//
//   solve_km_b200          == ot::solve_km          (hungarian.hpp:39-40)
//   solve_batched_km_b200  == ot::solve_batched_km  (hungarian.hpp:53-56)
//   solve_auction_b200        == ot::solve_auction        (auction.hpp:30-32)
//   solve_auction_scaled_b200 == ot::solve_auction_scaled (auction.hpp:48-50)
//     (declared when "ot/auction.hpp" is included first; bit-identical prices,
//      bids and assignment; costs must fit int32)
//
// Same inputs (OTInstance), same outputs (SolveResult built with the
// reference's own make_result, optional DualPotentials / Matching /
// QuantizedCosts overwritten wholesale), same exceptions and messages
// (hungarian.cpp:15-21, :34, :44-45, :353-354).  The KM solvers take the
// reference's int64 costs over its whole admissible range (kmb_solve_i64,
// kmb_solve_batched_km_i64: validation and quantization run on the device; the
// one deviation is a quantized cost above 2^60, i.e. B > 2^60, which throws
// std::invalid_argument rather than risk the reference's own int64 overflow).
// A CUDA failure throws std::runtime_error (there is no CPU fallback).
//
// Registering them as bench plugins (bench.cpp:391-464) is one line each,
// see INTEGRATION.md.
#ifndef KMB_OT_HPP
#define KMB_OT_HPP

#include <chrono>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kmb.h"

namespace ot {

namespace kmb_detail {

inline kmb_context* context() {
  // one context per thread (the C ABI is re-entrant; a context is not)
  thread_local std::unique_ptr<kmb_context, void (*)(kmb_context*)> ctx(nullptr, kmb_destroy);
  if (!ctx) {
    kmb_context* c = nullptr;
    if (kmb_create(0, &c) != KMB_OK) throw std::runtime_error(kmb_last_error());
    ctx.reset(c);
  }
  return ctx.get();
}

inline void require_unit_square(const OTInstance& inst, const char* who) {
  if (auto err = validate_instance(inst))
    throw std::invalid_argument(std::string(who) + ": " + *err);
  if (!inst.unit_caps())
    throw std::invalid_argument(std::string(who) + ": requires a unit-capacity square instance");
}

inline void check(int rc, const char* who) {
  if (rc == KMB_OK) return;
  if (rc > 0) throw std::invalid_argument(std::string(who) + ": " + kmb_last_error());
  throw std::runtime_error(std::string(who) + ": " + kmb_last_error());
}

// the C ABI's message as is: kmb_solve_batched_km_i64 words its errors like
// the reference ("solve_batched_km: ...", "quantize_costs: ...")
inline void check_verbatim(int rc) {
  if (rc == KMB_OK) return;
  if (rc > 0) throw std::invalid_argument(kmb_last_error());
  throw std::runtime_error(kmb_last_error());
}

inline Flow matching_flow(int32_t n, const std::vector<int32_t>& row_to_col) {
  std::vector<Flow::Entry> entries;
  entries.reserve(n);
  for (int32_t i = 0; i < n; ++i)
    if (row_to_col[i] >= 0) entries.push_back({i, row_to_col[i], 1.0});
  return Flow(n, n, std::move(entries));
}

}  // namespace kmb_detail

inline SolveResult solve_km_b200(const OTInstance& inst, DualPotentials* duals = nullptr,
                                 Matching* matching = nullptr, double time_budget_s = 0.0) {
  kmb_detail::require_unit_square(inst, "solve_km");
  const auto t0 = std::chrono::steady_clock::now();
  const int32_t n = inst.n;
  std::vector<int32_t> r2c(n, -1);
  std::vector<int64_t> u(n), v(n);
  int64_t total = 0;
  kmb_stats st{};
  kmb_detail::check(kmb_solve_i64(kmb_detail::context(), inst.cost.data(), n, n, KMB_SEED_KM,
                                  time_budget_s, r2c.data(), u.data(), v.data(), &total, &st),
                    "solve_km");
  const bool done = st.converged != 0;
  if (done) {
    if (duals) {
      duals->u = u;
      duals->v = v;
    }
    if (matching) matching->row_to_col = r2c;
  }
  int32_t matched = 0;
  for (int32_t j : r2c) matched += j >= 0;
  // iterations: rows inserted (hungarian.cpp:113, :130).  On budget expiry the
  // reference reports the i + 1 rows it processed, each of which it matched;
  // the parallel engine's counterpart is the number of matched rows.
  SolveResult res = make_result(inst, kmb_detail::matching_flow(n, r2c), done ? n : matched,
                                /*exact=*/done, /*converged=*/done);
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

inline SolveResult solve_batched_km_b200(const OTInstance& inst, const BatchedKMConfig& config = {},
                                         DualPotentials* duals = nullptr,
                                         QuantizedCosts* quantized = nullptr) {
  kmb_detail::require_unit_square(inst, "solve_batched_km");
  const auto t0 = std::chrono::steady_clock::now();
  const int32_t n = inst.n;
  std::vector<int32_t> r2c(n, -1);
  std::vector<int64_t> u(n), v(n);
  int64_t total = 0;
  kmb_stats st{};
  QuantizedCosts q;
  q.B = config.B;
  if (quantized) q.chat.resize(inst.cost.size());
  int32_t lossless = 0;
  // validation, quantize_costs (:33-53, K11), reductions and search on the device
  kmb_detail::check_verbatim(kmb_solve_batched_km_i64(
      kmb_detail::context(), inst.cost.data(), n, config.B, config.time_budget_s, r2c.data(), u.data(),
      v.data(), &total, quantized ? q.chat.data() : nullptr, &q.N, &lossless, &st));
  q.lossless = lossless != 0;
  const bool budget_ok = st.converged != 0;
  if (duals) {
    duals->u = u;
    duals->v = v;
  }
  if (quantized) *quantized = std::move(q);
  // iterations = phases + dual adjustments (hungarian.cpp:375); the dual-step
  // count equals the reference's, the phase count is the engine's own.
  SolveResult res = make_result(inst, kmb_detail::matching_flow(n, r2c), st.phases + st.dual_steps,
                                /*exact=*/q.lossless && budget_ok, budget_ok);
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

#ifdef OT_AUCTION_HPP
namespace kmb_detail {
inline SolveResult auction(const OTInstance& inst, const kmb_auction_config& cfg, const char* who,
                           std::vector<double>* prices_out, Matching* matching_out) {
  require_unit_square(inst, who);  // require_auctionable (auction.cpp:181-188)
  const auto t0 = std::chrono::steady_clock::now();
  const int32_t n = inst.n;
  std::vector<int32_t> c(inst.cost.size());
  for (size_t k = 0; k < c.size(); ++k) {
    if (inst.cost[k] > std::numeric_limits<int32_t>::max())
      throw std::invalid_argument(std::string(who) + ": cost exceeds the device range [0, 2^31)");
    c[k] = static_cast<int32_t>(inst.cost[k]);
  }
  std::vector<double> prices(n);
  std::vector<int32_t> r2c(n, -1);
  int64_t total = 0, bids = 0;
  int32_t converged = 0;
  double eps = 0.0;
  check(kmb_auction_i32(context(), c.data(), 1, n, &cfg, prices.data(), r2c.data(), &total, &bids,
                        &converged, &eps, nullptr),
        who);
  const bool complete = converged != 0;
  // finish (auction.cpp:161-179)
  SolveResult res = make_result(inst, matching_flow(n, r2c), bids,
                                /*exact=*/complete && eps * n < 1.0, complete);
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (prices_out) *prices_out = std::move(prices);
  if (matching_out) matching_out->row_to_col = std::move(r2c);
  return res;
}
}  // namespace kmb_detail

inline SolveResult solve_auction_b200(const OTInstance& inst, const AuctionConfig& config,
                                      std::vector<double>* prices_out = nullptr,
                                      Matching* matching_out = nullptr) {
  kmb_detail::require_unit_square(inst, "solve_auction");
  if (!(config.epsilon > 0.0)) throw std::invalid_argument("solve_auction: epsilon must be positive");
  const kmb_auction_config cfg{0, config.epsilon, 4.0, 0.0, config.max_bids, config.time_budget_s};
  return kmb_detail::auction(inst, cfg, "solve_auction", prices_out, matching_out);
}

inline SolveResult solve_auction_scaled_b200(const OTInstance& inst,
                                             const AuctionScaledConfig& config = {},
                                             std::vector<double>* prices_out = nullptr) {
  kmb_detail::require_unit_square(inst, "solve_auction_scaled");
  if (!(config.theta > 1.0))
    throw std::invalid_argument("solve_auction_scaled: theta must exceed 1");
  const kmb_auction_config cfg{1, config.epsilon0, config.theta, config.epsilon_final,
                               config.max_bids, config.time_budget_s};
  return kmb_detail::auction(inst, cfg, "solve_auction_scaled", prices_out, nullptr);
}
#endif  // OT_AUCTION_HPP

}  // namespace ot

#endif  // KMB_OT_HPP
