/*
 * TEST INFRASTRUCTURE ONLY — a step-by-step CPU mirror of the GPU engine in
 * paper_2005_01182_b200/csrc/ (same phases, same packed-key argmin parents,
 * same lazy dual bookkeeping, same forest augmentation), used to debug the
 * CUDA kernels and to check, on CPU and at scale, that the engine's duals
 * equal the reference's.  It is not the oracle: the
 * oracle is km_oracle.c / oracle/_ref.  Only tests/ load it.
 *
 * Engine (one phase = one multi-source search + one batch augmentation):
 *  - every free row is a root; D = dual shift accumulated in this phase;
 *  - row i reached at shift Dr stores w_i = u_i - Dr; column j keeps the
 *    packed key min_i ((C_ij - w_i + 2^30) << 32 | i) over reached rows, so
 *    slack'_j = val(key_j) - v_j is invariant under dual steps and a column
 *    is tight iff slack'_j == D;
 *  - a round = relax the rows reached last round, m = min unreached slack',
 *    if m > D it is a dual step (D = m; no tight unreached column and no
 *    pending row, exactly hungarian.cpp:201-215), then absorb every
 *    unreached column with slack' == D (hungarian.cpp:186-199);
 *  - absorbing a free column claims its tree root; the search ends after the
 *    round that found one (or, with continue_bfs, once the tight closure at
 *    the current D is exhausted — never with another dual step);
 *  - duals are finalised (u_i = w_i + D, v_j -= D - Dc_j), then every claimed
 *    tree flips its parent-pointer path (vertex-disjoint: one path per tree).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KM_BIAS (1LL << 30)

static inline uint64_t pack_key(int64_t val, int32_t row) {
  return ((uint64_t)(uint32_t)(val + KM_BIAS) << 32) | (uint32_t)row;
}
static inline int64_t key_val(uint64_t k) { return (int64_t)(k >> 32) - KM_BIAS; }
static inline int32_t key_row(uint64_t k) { return (int32_t)(k & 0xffffffffu); }

/* seed: 0 = u = v = 0 (solve_km start, hungarian.cpp:63),
 *       1 = row/column reductions (hungarian.cpp:323-333).
 * Costs must lie in [0, 2^30).  Returns 0 or a negative error. */
int kmm_solve(const int32_t* C, int32_t n, int32_t seed, int32_t continue_bfs,
              int64_t* u, int64_t* v, int32_t* match_row, int64_t* total_cost,
              int64_t* phases_out, int64_t* dual_steps_out, int64_t* rows_scanned_out,
              int64_t* trace, int64_t trace_cap) {
  int32_t* match_col = malloc(sizeof(int32_t) * (size_t)n);
  uint64_t* key = malloc(sizeof(uint64_t) * (size_t)n);
  int64_t* w = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* dc = malloc(sizeof(int64_t) * (size_t)n);
  char* rcol = malloc((size_t)n);
  int32_t* tree_par = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* root_row = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* claim = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* list = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* found = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* dead_round = malloc(sizeof(int32_t) * (size_t)n);
  if (!match_col || !key || !w || !dc || !rcol || !tree_par || !root_row ||
      !claim || !list || !found)
    return -1;
  int rc = 0;
  for (int32_t i = 0; i < n; ++i) {
    match_row[i] = match_col[i] = -1;
    claim[i] = -1;
    u[i] = 0;
    v[i] = 0;
  }
  if (seed == 1)
    for (int32_t i = 0; i < n; ++i) {
      const int32_t* row = C + (size_t)i * n;
      int32_t lo = row[0];
      for (int32_t j = 1; j < n; ++j) if (row[j] < lo) lo = row[j];
      u[i] = lo;
    }

  int64_t phases = 0, dual_steps = 0, rows_scanned = 0;
  for (int32_t phase = 0;; ++phase) {
    int32_t tail = 0;
    for (int32_t i = 0; i < n; ++i)
      if (match_row[i] < 0) {
        list[tail++] = i;
        w[i] = u[i];
        root_row[i] = i;
      }
    if (tail == 0) break;
    const int32_t nroots = tail;
    for (int32_t j = 0; j < n; ++j) { key[j] = UINT64_MAX; rcol[j] = 0; }
    int64_t D = 0;
    int32_t head = 0, nfound = 0;
    int first = (phase == 0 && seed == 1);
    for (int32_t round = 0;; ++round) {
      /* relax rows reached last round */
      for (int32_t r = head; r < tail; ++r) {
        const int32_t i = list[r];
        const int32_t* row = C + (size_t)i * n;
        for (int32_t j = 0; j < n; ++j) {
          const uint64_t k = pack_key((int64_t)row[j] - w[i], i);
          if (k < key[j]) key[j] = k;
        }
      }
      rows_scanned += tail - head;
      head = tail;
      if (first) { /* column reduction is the first relax (hungarian.cpp:328-333) */
        for (int32_t j = 0; j < n; ++j) v[j] = key_val(key[j]);
        first = 0;
      }
      int64_t m = INT64_MAX;
      for (int32_t j = 0; j < n; ++j)
        if (!rcol[j]) {
          const int64_t s = key_val(key[j]) - v[j];
          if (s < m) m = s;
        }
      if (m == INT64_MAX) {
        if (nfound) break; /* every column absorbed */
        rc = -2;
        goto done;
      }
      if (m > D) {
        if (nfound) break; /* closure exhausted at this D */
        if (trace && dual_steps < trace_cap) {
          trace[2 * dual_steps] = m - D;
          trace[2 * dual_steps + 1] = tail;
        }
        D = m;
        ++dual_steps;
      }
      for (int32_t j = 0; j < n; ++j) {
        if (rcol[j] || key_val(key[j]) - v[j] != D) continue;
        rcol[j] = 1;
        dc[j] = D;
        const int32_t p = key_row(key[j]);
        tree_par[j] = p;
        const int32_t root = root_row[p];
        const int32_t i2 = match_col[j];
        if (i2 < 0) {
          if (claim[root] != phase) {
            claim[root] = phase;
            dead_round[root] = round;
            found[nfound++] = j;
          }
        } else if (continue_bfs == 2 && claim[root] == phase && dead_round[root] < round) {
          /* harvest mode: a tree that already owns a free column stops growing */
        } else {
          w[i2] = u[i2] - D;
          root_row[i2] = root;
          list[tail++] = i2;
        }
      }
      if (nfound && (!continue_bfs || head == tail)) break;
    }
    /* finalise duals of this phase */
    for (int32_t r = 0; r < tail; ++r) u[list[r]] = w[list[r]] + D;
    for (int32_t j = 0; j < n; ++j)
      if (rcol[j]) v[j] -= D - dc[j];
    /* flip one parent-pointer path per claimed tree */
    for (int32_t f = 0; f < nfound; ++f) {
      int32_t j = found[f];
      for (;;) {
        const int32_t i = tree_par[j];
        const int32_t nxt = match_row[i];
        match_row[i] = j;
        match_col[j] = i;
        if (nxt < 0) break;
        j = nxt;
      }
    }
    (void)nroots;
    ++phases;
  }
  int64_t tot = 0;
  for (int32_t i = 0; i < n; ++i) tot += C[(size_t)i * n + match_row[i]];
  *total_cost = tot;
  *phases_out = phases;
  *dual_steps_out = dual_steps;
  if (rows_scanned_out) *rows_scanned_out = rows_scanned;
done:
  free(match_col); free(key); free(w); free(dc); free(rcol); free(tree_par);
  free(root_row); free(claim); free(list); free(found); free(dead_round);
  return rc;
}

/*
 * Incremental variant (the engine's "epoch" schedule): the multi-source search
 * is never restarted.  When a round absorbs free columns, the trees that own
 * one are augmented and dissolved — their rows and columns are finalised
 * (u = w + D, v -= D - Dc) and become unreached — while every other tree
 * stays reached with its lazy duals.  Columns whose argmin row belonged to a
 * dissolved tree are reset and all surviving rows are relaxed once more, which
 * restores key_j = min over the surviving reached rows for every unreached
 * column; the search then continues at the same D.  Surviving trees are tight
 * alternating trees from free roots, so the explored set is still exactly the
 * tight closure of the free rows and dual steps still happen only when it
 * holds no free column.
 */
int kmm_solve_incr(const int32_t* C, int32_t n, int32_t seed, int64_t* u, int64_t* v,
                   int32_t* match_row, int64_t* total_cost, int64_t* epochs_out,
                   int64_t* dual_steps_out, int64_t* rows_scanned_out, int64_t* rounds_out,
                   int64_t* trace, int64_t trace_cap) {
  int32_t* match_col = malloc(sizeof(int32_t) * (size_t)n);
  uint64_t* key = malloc(sizeof(uint64_t) * (size_t)n);
  int64_t* w = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* dc = malloc(sizeof(int64_t) * (size_t)n);
  char* rcol = malloc((size_t)n);
  char* rrow = malloc((size_t)n);
  int32_t* tree_par = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* root_row = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* claim = malloc(sizeof(int32_t) * (size_t)n); /* epoch stamp */
  int32_t* claim_col = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* rows = malloc(sizeof(int32_t) * (size_t)n);  /* reached rows */
  int32_t* nxt_rows = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* found = malloc(sizeof(int32_t) * (size_t)n);
  char* dmask = malloc((size_t)n);
  int dirty_only = 0;
  if (!match_col || !key || !w || !dc || !rcol || !rrow || !tree_par || !root_row || !claim ||
      !claim_col || !rows || !nxt_rows || !found || !dmask)
    return -1;
  for (int32_t i = 0; i < n; ++i) {
    match_row[i] = match_col[i] = -1;
    claim[i] = -1;
    u[i] = 0;
    v[i] = 0;
    key[i] = UINT64_MAX;
    rcol[i] = 0;
  }
  if (seed == 1)
    for (int32_t i = 0; i < n; ++i) {
      const int32_t* row = C + (size_t)i * n;
      int32_t lo = row[0];
      for (int32_t j = 1; j < n; ++j) if (row[j] < lo) lo = row[j];
      u[i] = lo;
    }
  /* every row starts free and reached */
  int32_t nrows = n;
  for (int32_t i = 0; i < n; ++i) {
    rows[i] = i;
    rrow[i] = 1;
    w[i] = u[i];
    root_row[i] = i;
  }
  int32_t head = 0; /* rows[head, nrows) still to relax */
  int64_t D = 0, dual_steps = 0, rows_scanned = 0, rounds = 0, epochs = 0;
  int first = (seed == 1);
  int32_t nfree = n;
  int rc = 0;
  while (nfree > 0) {
    ++rounds;
    /* epoch start: the survivors only over the dirty columns (keys reset at
     * the epoch end); every other unreached key is attained at a survivor */
    if (dirty_only)
      for (int32_t j = 0; j < n; ++j) dmask[j] = key[j] == UINT64_MAX && !rcol[j];
    for (int32_t r = head; r < nrows; ++r) {
      const int32_t i = rows[r];
      const int32_t* row = C + (size_t)i * n;
      for (int32_t j = 0; j < n; ++j) {
        if (dirty_only && !dmask[j]) continue;
        const uint64_t k = pack_key((int64_t)row[j] - w[i], i);
        if (k < key[j]) key[j] = k;
      }
    }
    if (!dirty_only) rows_scanned += nrows - head;
    dirty_only = 0;
    head = nrows;
    if (first) {
      for (int32_t j = 0; j < n; ++j) v[j] = key_val(key[j]);
      first = 0;
    }
    int64_t m = INT64_MAX;
    for (int32_t j = 0; j < n; ++j)
      if (!rcol[j]) {
        const int64_t s = key_val(key[j]) - v[j];
        if (s < m) m = s;
      }
    if (m == INT64_MAX) { rc = -2; goto done; }
    if (m > D) {
      if (trace && dual_steps < trace_cap) {
        trace[2 * dual_steps] = m - D;
        trace[2 * dual_steps + 1] = nrows;
      }
      D = m;
      ++dual_steps;
    }
    int32_t nfound = 0;
    const int32_t ep = (int32_t)epochs;
    for (int32_t j = 0; j < n; ++j) {
      if (rcol[j] || key_val(key[j]) - v[j] != D) continue;
      rcol[j] = 1;
      dc[j] = D;
      const int32_t p = key_row(key[j]);
      tree_par[j] = p;
      const int32_t root = root_row[p];
      const int32_t i2 = match_col[j];
      if (i2 < 0) {
        if (claim[root] != ep || j < claim_col[root]) {
          claim[root] = ep;
          claim_col[root] = j;
        }
        found[nfound++] = j;
      } else {
        w[i2] = u[i2] - D;
        root_row[i2] = root;
        rrow[i2] = 1;
        rows[nrows++] = i2;
      }
    }
    if (!nfound) continue;
    /* ---- epoch end: relax the rows appended this round over all columns
     * (the epoch-start re-relax covers dirty columns only), then dissolve ---- */
    for (int32_t r = head; r < nrows; ++r) {
      const int32_t i = rows[r];
      const int32_t* row = C + (size_t)i * n;
      for (int32_t j = 0; j < n; ++j) {
        const uint64_t k = pack_key((int64_t)row[j] - w[i], i);
        if (k < key[j]) key[j] = k;
      }
    }
    rows_scanned += nrows - head;
    /* ---- epoch end: dissolve claimed trees ---- */
    for (int32_t j = 0; j < n; ++j) {
      if (rcol[j]) {
        if (claim[root_row[tree_par[j]]] == ep) {
          v[j] -= D - dc[j];
          rcol[j] = 0;
          key[j] = UINT64_MAX;
        }
      } else if (key[j] != UINT64_MAX && claim[root_row[key_row(key[j])]] == ep) {
        key[j] = UINT64_MAX; /* dirty: argmin row leaves the search */
      }
    }
    int32_t ns = 0;
    for (int32_t r = 0; r < nrows; ++r) {
      const int32_t i = rows[r];
      if (claim[root_row[i]] == ep) {
        u[i] = w[i] + D;
        rrow[i] = 0;
      } else {
        nxt_rows[ns++] = i;
      }
    }
    for (int32_t f = 0; f < nfound; ++f) {
      int32_t j = found[f];
      const int32_t root = root_row[tree_par[j]];
      if (claim_col[root] != j) continue;
      --nfree;
      for (;;) {
        const int32_t i = tree_par[j];
        const int32_t nx = match_row[i];
        match_row[i] = j;
        match_col[j] = i;
        if (nx < 0) break;
        j = nx;
      }
    }
    memcpy(rows, nxt_rows, sizeof(int32_t) * (size_t)ns);
    nrows = ns;
    head = 0; /* survivors relax once more for the reset columns */
    dirty_only = 1;
    ++epochs;
  }
  {
    int64_t tot = 0;
    for (int32_t i = 0; i < n; ++i) tot += C[(size_t)i * n + match_row[i]];
    *total_cost = tot;
  }
  *epochs_out = epochs;
  *dual_steps_out = dual_steps;
  if (rows_scanned_out) *rows_scanned_out = rows_scanned;
  if (rounds_out) *rounds_out = rounds;
done:
  free(match_col); free(key); free(w); free(dc); free(rcol); free(rrow); free(tree_par);
  free(root_row); free(claim); free(claim_col); free(rows); free(nxt_rows); free(found);
  free(dmask);
  return rc;
}
