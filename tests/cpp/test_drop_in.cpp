// C++ parity tests of the drop-in (include/kmb_ot.hpp) against the UNMODIFIED
// reference solvers, written like the reference's own tests/test_hungarian.cpp
// (same cases, same RNG seeds, same assertions) plus exact-equality checks of
// the duals.  Built by tests/cpp/build.sh (needs /root/reference headers), run
// on the GPU by tests/test_cpp_drop_in.py.
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

#include "ot/auction.hpp"
#include "ot/core.hpp"
#include "ot/hungarian.hpp"
#include "kmb_ot.hpp"
#include "testutil.hpp"  // the reference's own fixtures (proj/tests/testutil.hpp)

using namespace ot;
using ot::testing::color_style_pair;
using ot::testing::random_unit_instance;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                        \
  } while (0)

static OTInstance unit_2x2() {
  OTInstance inst;
  inst.n = inst.m = 2;
  inst.cost = {1, 3, 2, 1};
  inst.supplies = {1, 1};
  inst.demands = {1, 1};
  return inst;
}

static int64_t dual_total(const DualPotentials& d) {
  int64_t t = 0;
  for (int64_t x : d.u) t += x;
  for (int64_t x : d.v) t += x;
  return t;
}

int main() {
  {  // km: zero diagonal picks the identity matching (test_hungarian.cpp:61-70)
    OTInstance inst;
    inst.n = inst.m = 3;
    inst.cost = {0, 5, 5, 5, 0, 5, 5, 5, 0};
    inst.supplies = inst.demands = {1, 1, 1};
    Matching m;
    const SolveResult res = solve_km_b200(inst, nullptr, &m);
    CHECK(res.objective == 0.0);
    for (int32_t i = 0; i < 3; ++i) CHECK(m.row_to_col[i] == i);
  }
  {  // km: 2x2 with known optimum (:72-85)
    const OTInstance inst = unit_2x2();
    Matching m;
    DualPotentials d;
    const SolveResult res = solve_km_b200(inst, &d, &m);
    CHECK(res.objective == 2.0);
    CHECK((m.row_to_col == std::vector<int32_t>{0, 1}));
    CHECK(dual_total(d) == 2);
  }
  {  // km: requires a unit square (:87-94) — same exception, same message
    OTInstance inst = unit_2x2();
    inst.supplies = {2, 1};
    inst.demands = {1, 2};
    std::string a, b;
    try { solve_km_b200(inst); } catch (const std::invalid_argument& e) { a = e.what(); }
    try { solve_km(inst); } catch (const std::invalid_argument& e) { b = e.what(); }
    CHECK(!a.empty() && a == b);
  }
  {  // km: agreement with the reference on random unit instances (:96-105, seed 11)
    std::mt19937 rng(11);
    for (int t = 0; t < 100; ++t) {
      const OTInstance inst = random_unit_instance(rng, 2 + static_cast<int32_t>(rng() % 5), 9);
      DualPotentials d1, d2;
      const SolveResult a = solve_km_b200(inst, &d1);
      const SolveResult b = solve_km(inst, &d2);
      CHECK(objective_int(inst, a.flow) == objective_int(inst, b.flow));
      CHECK(d1.u == d2.u && d1.v == d2.v);
      CHECK(residue(inst, a.flow) == 0.0);
    }
  }
  {  // km: duals feasible and tight (:107-122, seed 13) and equal to the reference's
    std::mt19937 rng(13);
    const OTInstance inst = random_unit_instance(rng, 50, 100000);
    DualPotentials d, dr;
    Matching m;
    const SolveResult res = solve_km_b200(inst, &d, &m);
    solve_km(inst, &dr);
    for (int32_t i = 0; i < inst.n; ++i) {
      for (int32_t j = 0; j < inst.m; ++j) CHECK(d.u[i] + d.v[j] <= inst.cost_at(i, j));
      CHECK(d.u[i] + d.v[m.row_to_col[i]] == inst.cost_at(i, m.row_to_col[i]));
    }
    CHECK(static_cast<double>(dual_total(d)) == res.objective);
    CHECK(d.u == dr.u && d.v == dr.v);
  }
  {  // batched: lossless quantization reproduces km (:124-131)
    const OTInstance inst = unit_2x2();
    BatchedKMConfig cfg;
    cfg.B = inst.max_cost();
    const SolveResult res = solve_batched_km_b200(inst, cfg);
    CHECK(res.objective == 2.0);
    CHECK(res.exact);
  }
  {  // batched: constant costs (:133-142): objective 24; no dual step
    OTInstance inst;
    inst.n = inst.m = 6;
    inst.cost.assign(36, 4);
    inst.supplies.assign(6, 1);
    inst.demands.assign(6, 1);
    const SolveResult res = solve_batched_km_b200(inst);
    CHECK(res.objective == 24.0);
  }
  {  // batched: B = N*n matches km and the reference, duals bit-exact (:144-156, seed 17)
    std::mt19937 rng(17);
    for (int t = 0; t < 100; ++t) {
      const OTInstance inst = random_unit_instance(rng, 2 + static_cast<int32_t>(rng() % 7), 50);
      BatchedKMConfig cfg;
      cfg.B = std::max<int64_t>(inst.max_cost(), 1) * inst.n;
      DualPotentials d1, d2;
      const SolveResult a = solve_batched_km_b200(inst, cfg, &d1);
      const SolveResult b = solve_batched_km(inst, cfg, &d2);
      CHECK(a.objective == b.objective);
      CHECK(a.exact);
      CHECK(d1.u == d2.u && d1.v == d2.v);
    }
  }
  {  // batched: objective within the quantization error bound (:158-172, seed 19)
    std::mt19937 rng(19);
    for (int64_t B : {1, 2, 5, 10, 37}) {
      const OTInstance inst = random_unit_instance(rng, 40, 100000);
      BatchedKMConfig cfg;
      cfg.B = B;
      DualPotentials d1, d2;
      const SolveResult batched = solve_batched_km_b200(inst, cfg, &d1);
      const SolveResult ref = solve_batched_km(inst, cfg, &d2);
      const SolveResult km = solve_km(inst);
      const double bound = km.objective + static_cast<double>(inst.n) * inst.max_cost() / static_cast<double>(B);
      CHECK(batched.objective >= km.objective);
      CHECK(batched.objective <= bound);
      CHECK(!batched.exact == !ref.exact);
      CHECK(d1.u == d2.u && d1.v == d2.v);  // lossy mode: duals on chat still canonical
    }
  }
  {  // batched: certificate against the quantized costs (:174-189, seed 23)
    std::mt19937 rng(23);
    const OTInstance inst = random_unit_instance(rng, 60, 5000);
    BatchedKMConfig cfg;
    cfg.B = 64;
    DualPotentials d;
    QuantizedCosts q;
    const SolveResult res = solve_batched_km_b200(inst, cfg, &d, &q);
    CHECK(q.chat.size() == inst.cost.size());
    for (int32_t i = 0; i < inst.n; ++i)
      for (int32_t j = 0; j < inst.m; ++j)
        CHECK(d.u[i] + d.v[j] <= q.chat[static_cast<size_t>(i) * inst.m + j]);
    for (const Flow::Entry& e : res.flow.entries())
      CHECK(d.u[e.i] + d.v[e.j] == q.chat[static_cast<size_t>(e.i) * inst.m + e.j]);
  }
  {  // batched: rejects non-unit instances (:200-205)
    OTInstance inst = unit_2x2();
    inst.supplies = {2, 1};
    inst.demands = {1, 2};
    bool threw = false;
    try { solve_batched_km_b200(inst); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
  }
  {  // quantize_costs: B must be positive (:34) surfaces unchanged
    BatchedKMConfig cfg;
    cfg.B = 0;
    std::string a;
    try { solve_batched_km_b200(unit_2x2(), cfg); } catch (const std::invalid_argument& e) { a = e.what(); }
    CHECK(a == "quantize_costs: B must be positive");
  }
  {  // batched: iterations count phases plus dual adjustments (:191-198, seed 29)
    std::mt19937 rng(29);
    const OTInstance inst = random_unit_instance(rng, 30, 1000);
    const SolveResult res = solve_batched_km_b200(inst);
    CHECK(res.iterations >= 1);
    CHECK(res.iterations <= static_cast<int64_t>(inst.n) * (inst.n + 1));
  }
  {  // km on the color-style instance (:207-212): the reference's objective and duals
    const OTInstance inst = color_style_pair(9, "color_check");
    DualPotentials d1, d2;
    const SolveResult a = solve_km_b200(inst, &d1);
    const SolveResult b = solve_km(inst, &d2);
    CHECK(a.objective == b.objective);
    CHECK(d1.u == d2.u && d1.v == d2.v);
  }
  {  // the reference's whole int64 range: costs up to validate_instance's headroom
     // (core.cpp:47-53) through the wide engine; duals and objective identical
    std::mt19937_64 rng(97);
    for (int32_t n : {2, 17, 64}) {
      const int64_t head = ((int64_t{1} << 62) / n) / (2 * static_cast<int64_t>(n) + 2);
      OTInstance inst;
      inst.n = inst.m = n;
      inst.supplies.assign(n, 1);
      inst.demands.assign(n, 1);
      inst.cost.resize(static_cast<size_t>(n) * n);
      for (int64_t& x : inst.cost) x = static_cast<int64_t>(rng() % static_cast<uint64_t>(head));
      inst.cost[0] = head;
      DualPotentials d1, d2;
      const SolveResult a = solve_km_b200(inst, &d1);
      const SolveResult b = solve_km(inst, &d2);
      CHECK(a.objective == b.objective && d1.u == d2.u && d1.v == d2.v);
      // B = N: B * N overflows int64 for costs this wide, so quantize_costs
      // rejects it — the drop-in the same way, with the same message
      BatchedKMConfig c0;
      c0.B = head;
      std::string m1, m2;
      try { solve_batched_km_b200(inst, c0); } catch (const std::invalid_argument& e) { m1 = e.what(); }
      try { solve_batched_km(inst, c0); } catch (const std::invalid_argument& e) { m2 = e.what(); }
      CHECK(m1 == m2 && m1 == "quantize_costs: B * max cost overflows");
      // B = N with N = 2^31 (N * N fits): lossless, chat = C beyond the 32-bit
      // engines' range, solved on the wide engine
      for (int64_t& x : inst.cost) x = static_cast<int64_t>(rng() % (int64_t{1} << 31));
      inst.cost[1] = int64_t{1} << 31;
      c0.B = int64_t{1} << 31;
      DualPotentials e0, f0;
      const SolveResult g = solve_batched_km_b200(inst, c0, &e0);
      const SolveResult h = solve_batched_km(inst, c0, &f0);
      CHECK(g.exact && h.exact && g.objective == h.objective && e0.u == f0.u && e0.v == f0.v);
      for (int64_t& x : inst.cost) x = static_cast<int64_t>(rng() % 1000000);
      DualPotentials e1, e2;
      QuantizedCosts q1, q2;
      BatchedKMConfig cfg;
      cfg.B = 3000000007;  // lossy, chat beyond the 32-bit engines' range
      const SolveResult c = solve_batched_km_b200(inst, cfg, &e1, &q1);
      const SolveResult d = solve_batched_km(inst, cfg, &e2, &q2);
      CHECK(e1.u == e2.u && e1.v == e2.v && q1.chat == q2.chat && q1.N == q2.N);
      CHECK(q1.lossless == q2.lossless && c.exact == d.exact);
    }
    OTInstance big = unit_2x2();
    big.cost[0] = int64_t{1} << 61;  // beyond the headroom: the reference's message
    std::string a, b;
    try { solve_km_b200(big); } catch (const std::invalid_argument& e) { a = e.what(); }
    try { solve_km(big); } catch (const std::invalid_argument& e) { b = e.what(); }
    CHECK(!a.empty() && a == b);
  }
  // ---- auction (test_auction.cpp cases; bit-identical prices vs the reference)
  auto same_bits = [](const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return false;
    for (size_t k = 0; k < a.size(); ++k)
      if (std::memcmp(&a[k], &b[k], sizeof(double)) != 0) return false;
    return true;
  };
  {  // small epsilon is exact on the 2x2
    AuctionConfig cfg;
    cfg.epsilon = 0.4;
    const SolveResult res = solve_auction_b200(unit_2x2(), cfg);
    CHECK(res.objective == 2.0 && res.exact && res.converged);
  }
  {  // epsilon-CS instances (seed 41) and random eps: same prices, bids, matching
    std::mt19937 rng(41);
    for (double eps : {0.5, 2.5, 10.0}) {
      const OTInstance inst = random_unit_instance(rng, 30, 100);
      AuctionConfig cfg;
      cfg.epsilon = eps;
      std::vector<double> pa, pb;
      Matching ma, mb;
      const SolveResult a = solve_auction_b200(inst, cfg, &pa, &ma);
      const SolveResult b = solve_auction(inst, cfg, &pb, &mb);
      CHECK(same_bits(pa, pb));
      CHECK(ma.row_to_col == mb.row_to_col);
      CHECK(a.iterations == b.iterations && a.objective == b.objective);
      CHECK(a.exact == b.exact && a.converged == b.converged);
    }
  }
  {  // scaled auction: default schedule exact, matches the reference (seed 61)
    std::mt19937 rng(61);
    for (int t = 0; t < 20; ++t) {
      const OTInstance inst = random_unit_instance(rng, 25, 800);
      std::vector<double> pa, pb;
      const SolveResult a = solve_auction_scaled_b200(inst, {}, &pa);
      const SolveResult b = solve_auction_scaled(inst, {}, &pb);
      CHECK(a.converged && a.exact);
      CHECK(same_bits(pa, pb) && a.iterations == b.iterations && a.objective == b.objective);
    }
  }
  {  // bid budget produces a flagged result (seed 59)
    std::mt19937 rng(59);
    const OTInstance inst = random_unit_instance(rng, 40, 1000);
    AuctionConfig cfg;
    cfg.epsilon = 0.1;
    cfg.max_bids = 5;
    const SolveResult res = solve_auction_b200(inst, cfg);
    CHECK(!res.converged && !res.exact && res.iterations == 5);
  }
  {  // epsilon must be positive; theta must exceed 1 — same messages
    AuctionConfig cfg;
    cfg.epsilon = 0.0;
    std::string a, b;
    try { solve_auction_b200(unit_2x2(), cfg); } catch (const std::invalid_argument& e) { a = e.what(); }
    try { solve_auction(unit_2x2(), cfg); } catch (const std::invalid_argument& e) { b = e.what(); }
    CHECK(!a.empty() && a == b);
    AuctionScaledConfig sc;
    sc.theta = 1.0;
    a.clear();
    b.clear();
    try { solve_auction_scaled_b200(unit_2x2(), sc); } catch (const std::invalid_argument& e) { a = e.what(); }
    try { solve_auction_scaled(unit_2x2(), sc); } catch (const std::invalid_argument& e) { b = e.what(); }
    CHECK(!a.empty() && a == b);
  }
  std::printf("drop-in: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
