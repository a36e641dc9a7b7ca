/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the auction path.  Never
 * linked into the product library; only tests/ and bench.py's reference leg
 * load it (libkmoracle.so), as the checker.
 *
 * Plain-C restatement of the reference's Gauss-Seidel auction
 * (/root/reference/proj/src/auction.cpp), in the form the GPU engines use:
 *
 *  - the pending min-heap (auction.cpp:22-23, 162-164) always holds exactly
 *    the unassigned rows (a row is pushed when it is displaced, :67-69, and
 *    popped when it bids; try_complete only commits when the loop then
 *    breaks, :150), so "pop the top" is "the smallest unassigned row";
 *  - bid (:45-74): best = the largest value -C[i][j] - p[j] (first index on
 *    ties), second = the largest value over the other columns (the multiset
 *    second maximum), p[best_j] += (best - second) + eps, n == 1 -> second =
 *    best;
 *  - try_complete (:79-120) when at most two rows are free;
 *  - epsilon scaling (:201-229): prices persist, assignments reset,
 *    eps <- max(eps / theta, eps_final), per-round bid budget max_bids - total.
 *
 * Every double operation is the reference's, in the reference's order, so
 * prices are bit-identical (tests/test_auction.py pins this against
 * oracle/_ref).  Time budgets are not modelled (wall-clock dependent).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  const int64_t* C;
  int32_t n;
  double eps;
  double* p;
  int32_t* owner;    /* column -> row */
  int32_t* assigned; /* row -> column */
  int32_t unmatched;
  int64_t bids;
} ko_auction;

static double ko_value(const ko_auction* a, int32_t i, int32_t j) { /* :34-36 */
  return -(double)a->C[(int64_t)i * a->n + j] - a->p[j];
}

static double ko_best_value(const ko_auction* a, int32_t i) { /* :38-42 */
  double best = -INFINITY;
  for (int32_t j = 0; j < a->n; ++j) {
    const double v = ko_value(a, i, j);
    if (v > best) best = v; /* std::max(best, v) */
  }
  return best;
}

static void ko_bid(ko_auction* a, int32_t i) { /* :44-74 */
  int32_t best_j = 0;
  double best = -INFINITY, second = -INFINITY;
  for (int32_t j = 0; j < a->n; ++j) {
    const double v = ko_value(a, i, j);
    if (v > best) {
      second = best;
      best = v;
      best_j = j;
    } else if (v > second) {
      second = v;
    }
  }
  if (a->n == 1) second = best;
  a->p[best_j] += (best - second) + a->eps;
  const int32_t displaced = a->owner[best_j];
  if (displaced >= 0)
    a->assigned[displaced] = -1;
  else
    --a->unmatched;
  a->owner[best_j] = i;
  a->assigned[i] = best_j;
  ++a->bids;
}

static int ko_edge_ok(const ko_auction* a, int32_t i, int32_t j) { /* :90-92 */
  return ko_value(a, i, j) >= ko_best_value(a, i) - a->eps - 1e-9;
}

static int ko_try_complete(ko_auction* a) { /* :79-120 */
  int32_t rows[2], cols[2], nr = 0, nc = 0;
  for (int32_t i = 0; i < a->n; ++i)
    if (a->assigned[i] < 0 && nr < 2) rows[nr++] = i;
  for (int32_t j = 0; j < a->n; ++j)
    if (a->owner[j] < 0 && nc < 2) cols[nc++] = j;
  if (nr == 0) return 1;
  if (nr == 1) {
    if (!ko_edge_ok(a, rows[0], cols[0])) return 0;
    a->assigned[rows[0]] = cols[0];
    a->owner[cols[0]] = rows[0];
    --a->unmatched;
    return 1;
  }
  const int64_t n = a->n;
  const int64_t straight = a->C[rows[0] * n + cols[0]] + a->C[rows[1] * n + cols[1]];
  const int64_t crossed = a->C[rows[0] * n + cols[1]] + a->C[rows[1] * n + cols[0]];
  const int straight_first = straight <= crossed;
  for (int pass = 0; pass < 2; ++pass) {
    const int take_straight = (pass == 0) == straight_first;
    const int32_t j0 = take_straight ? cols[0] : cols[1];
    const int32_t j1 = take_straight ? cols[1] : cols[0];
    if (ko_edge_ok(a, rows[0], j0) && ko_edge_ok(a, rows[1], j1)) {
      a->assigned[rows[0]] = j0;
      a->owner[j0] = rows[0];
      a->assigned[rows[1]] = j1;
      a->owner[j1] = rows[1];
      a->unmatched -= 2;
      return 1;
    }
  }
  return 0;
}

/* AuctionCore::run without the time budget (:133-158): 1 = perfect matching. */
static int ko_run(ko_auction* a, int64_t max_bids) {
  while (a->unmatched > 0) {
    if (a->unmatched <= 2 && ko_try_complete(a)) break;
    if (a->bids >= max_bids) return 0;
    int32_t i = 0;
    while (a->assigned[i] >= 0) ++i; /* the heap's top: smallest unassigned row */
    ko_bid(a, i);
  }
  return 1;
}

/* solve_auction (scaled = 0, eps0 = AuctionConfig::epsilon > 0) or
 * solve_auction_scaled (scaled = 1; eps0/eps_final <= 0 pick the defaults,
 * theta > 1).  Returns 0, or 1 on invalid arguments.  Outputs: prices (n),
 * row_to_col (n, -1 when unassigned), total bids, complete flag, the
 * epsilon of the last round (exact = complete && eps * n < 1, :172). */
int kmo_auction(const int64_t* C, int32_t n, int32_t scaled, double eps0, double theta,
                double eps_final, int64_t max_bids, double* prices, int32_t* row_to_col,
                int64_t* bids_out, int32_t* complete_out, double* eps_out) {
  if (n <= 0) return 1;
  double eps = eps0;
  if (scaled) {
    if (!(theta > 1.0)) return 1;
    int64_t mx = 0;
    for (int64_t k = 0; k < (int64_t)n * n; ++k)
      if (C[k] > mx) mx = C[k];
    const double ef = eps_final > 0.0 ? eps_final : 1.0 / (n + 1); /* :209-211 */
    eps = eps0 > 0.0 ? eps0 : fmax((double)mx / 2.0, ef);         /* :212-215 */
    eps = fmax(eps, ef);
    eps_final = ef;
  } else if (!(eps > 0.0)) {
    return 1;
  }
  ko_auction a;
  a.C = C;
  a.n = n;
  a.p = prices;
  a.owner = malloc(sizeof(int32_t) * n);
  a.assigned = malloc(sizeof(int32_t) * n);
  for (int32_t j = 0; j < n; ++j) prices[j] = 0.0;
  int64_t total = 0;
  int complete = 0;
  for (;;) {
    a.eps = eps;
    a.unmatched = n;
    a.bids = 0;
    for (int32_t k = 0; k < n; ++k) a.owner[k] = a.assigned[k] = -1;
    complete = ko_run(&a, max_bids - total);
    total += a.bids;
    if (!scaled || !complete || eps <= eps_final) break;
    eps = fmax(eps / theta, eps_final); /* :226 */
  }
  for (int32_t i = 0; i < n; ++i) row_to_col[i] = a.assigned[i];
  *bids_out = total;
  *complete_out = complete;
  *eps_out = eps;
  free(a.owner);
  free(a.assigned);
  return 0;
}
