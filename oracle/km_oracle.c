/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into the product
 * library (paper_2005_01182_b200/); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg load it, as the checker.
 *
 * Plain-C restatement of the reference's exact assignment path
 * (/root/reference/proj/src/hungarian.cpp), int64 throughout like the
 * reference.  Each function names the lines it follows.  The restatement is
 * pinned against the reference compiled from its own sources
 * (oracle/_ref/libotref.so, see oracle/Makefile) and against the reference's
 * own known answers (tests/test_oracle.py).
 *
 * Extra over the reference: instrumentation (phase count, dual-step count and
 * the per-step (delta, |closure rows|) trace), which SURVEY.md fact 0.5 shows
 * to be independent of the augmentation order and is used as an intermediate
 * parity vector for the GPU engine.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KMO_INF (INT64_MAX / 4) /* hungarian.cpp:13 */

/* quantize_costs, hungarian.cpp:33-53.  Returns 0, or 1 for "B must be
 * positive", 2 for "B * max cost overflows". */
int kmo_quantize(const int64_t* cost, int64_t count, int64_t B, int64_t* chat,
                 int64_t* N_out, int32_t* lossless_out) {
  if (B <= 0) return 1;
  int64_t N = 0;
  for (int64_t a = 0; a < count; ++a)
    if (a == 0 || cost[a] > N) N = cost[a];
  if (count == 0) N = 0;
  if (N <= 0) { /* all-zero (or empty) matrix passes through, divisor 1 */
    if (count) memcpy(chat, cost, sizeof(int64_t) * (size_t)count);
    *N_out = 1;
    *lossless_out = 1;
    return 0;
  }
  if (B > INT64_MAX / N) return 2;
  int32_t lossless = 1;
  for (int64_t a = 0; a < count; ++a) {
    const int64_t scaled = cost[a] * B;
    chat[a] = scaled / N;
    if (chat[a] * N != scaled) lossless = 0;
  }
  *N_out = N;
  *lossless_out = lossless;
  return 0;
}

/* solve_km, hungarian.cpp:55-136: e-maxx O(n^3) potentials with a virtual
 * start column n; rows are inserted one at a time.  No time budget here (the
 * reference's budget exit, :106-118, is exercised through oracle/_ref). */
int kmo_solve_km(const int64_t* C, int32_t n, int64_t* u_out, int64_t* v_out,
                 int32_t* row_to_col, int64_t* total_cost) {
  int64_t* u = calloc((size_t)n, sizeof(int64_t));
  int64_t* v = calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* minv = malloc(sizeof(int64_t) * (size_t)n);
  int32_t* p = malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* way = malloc(sizeof(int32_t) * (size_t)n);
  char* used = malloc((size_t)n + 1);
  if (!u || !v || !minv || !p || !way || !used) return -1;
  for (int32_t j = 0; j <= n; ++j) p[j] = -1;

  for (int32_t r = 0; r < n; ++r) {
    p[n] = r;
    int32_t j0 = n;
    for (int32_t j = 0; j < n; ++j) minv[j] = KMO_INF;
    memset(used, 0, (size_t)n + 1);
    while (1) { /* :72-99 */
      used[j0] = 1;
      const int32_t i0 = p[j0];
      const int64_t* row = C + (size_t)i0 * n;
      int64_t delta = KMO_INF;
      int32_t j1 = -1;
      for (int32_t j = 0; j < n; ++j) {
        if (used[j]) continue;
        const int64_t cur = row[j] - u[i0] - v[j];
        if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
        if (minv[j] < delta) { delta = minv[j]; j1 = j; }
      }
      for (int32_t j = 0; j <= n; ++j) {
        if (used[j]) { u[p[j]] += delta; v[j] -= delta; }
        else minv[j] -= delta;
      }
      j0 = j1;
      if (p[j0] == -1) break;
    }
    while (j0 != n) { /* :100-104 path flip */
      const int32_t j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    }
  }
  int64_t tot = 0;
  for (int32_t j = 0; j < n; ++j) {
    row_to_col[p[j]] = j;
    tot += C[(size_t)p[j] * n + j];
  }
  memcpy(u_out, u, sizeof(int64_t) * (size_t)n);
  memcpy(v_out, v, sizeof(int64_t) * (size_t)n); /* drop virtual col, :124-127 */
  *total_cost = tot;
  free(u); free(v); free(minv); free(p); free(way); free(used);
  return 0;
}

/* ---- batched KM (hungarian.cpp:140-381) ---------------------------------- */

typedef struct {
  int32_t n;
  const int64_t* c;
  int64_t *u, *v;
  int32_t *mrow, *mcol;
  /* BatchedSearch scratch, :152-155 */
  char *rrow, *rcol;
  int64_t* slack;
  int32_t* queue;
  int32_t qlen;
  /* TightPhase scratch, :225-231 */
  int32_t *adj_start, *adj, *dist, *it;
  int32_t limit;
  int64_t adj_cap;
  /* instrumentation */
  int64_t dual_steps;
  int64_t* trace; /* pairs (delta, |reached rows|), may be NULL */
  int64_t trace_cap;
} kmo_state;

/* BatchedSearch::relax_from, :164-172 */
static void bs_relax(kmo_state* s, int32_t i) {
  const int64_t* row = s->c + (size_t)i * s->n;
  const int64_t ui = s->u[i];
  for (int32_t j = 0; j < s->n; ++j) {
    if (s->rcol[j]) continue;
    const int64_t d = row[j] - ui - s->v[j];
    if (d < s->slack[j]) s->slack[j] = d;
  }
}

/* BatchedSearch::run, :175-217: multi-source search from every free row,
 * dual step only when the tight closure has no free column. */
static int bs_run(kmo_state* s) {
  const int32_t n = s->n;
  memset(s->rrow, 0, (size_t)n);
  memset(s->rcol, 0, (size_t)n);
  for (int32_t j = 0; j < n; ++j) s->slack[j] = KMO_INF;
  s->qlen = 0;
  for (int32_t i = 0; i < n; ++i)
    if (s->mrow[i] < 0) { s->rrow[i] = 1; s->queue[s->qlen++] = i; }
  int32_t head = 0;
  for (;;) {
    while (head < s->qlen) bs_relax(s, s->queue[head++]);
    int found = 0, progressed = 0;
    for (int32_t j = 0; j < n; ++j) { /* absorb, :188-199 */
      if (s->rcol[j] || s->slack[j] != 0) continue;
      s->rcol[j] = 1;
      progressed = 1;
      const int32_t i2 = s->mcol[j];
      if (i2 < 0) found = 1;
      else if (!s->rrow[i2]) { s->rrow[i2] = 1; s->queue[s->qlen++] = i2; }
    }
    if (found) return 0;
    if (progressed || head < s->qlen) continue;
    int64_t delta = KMO_INF; /* :203-215 */
    for (int32_t j = 0; j < n; ++j)
      if (!s->rcol[j] && s->slack[j] < delta) delta = s->slack[j];
    if (!(delta > 0 && delta < KMO_INF)) return -2;
    if (s->trace && s->dual_steps < s->trace_cap) {
      int64_t nr = 0;
      for (int32_t i = 0; i < n; ++i) nr += s->rrow[i];
      s->trace[2 * s->dual_steps] = delta;
      s->trace[2 * s->dual_steps + 1] = nr;
    }
    ++s->dual_steps;
    for (int32_t i = 0; i < n; ++i)
      if (s->rrow[i]) s->u[i] += delta;
    for (int32_t j = 0; j < n; ++j) {
      if (s->rcol[j]) s->v[j] -= delta;
      else s->slack[j] -= delta;
    }
  }
}

/* TightPhase constructor, :233-252: CSR of the equality subgraph. */
static int tp_build(kmo_state* s) {
  const int32_t n = s->n;
  s->adj_start[0] = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t* row = s->c + (size_t)i * n;
    int32_t deg = 0;
    for (int32_t j = 0; j < n; ++j)
      if (row[j] - s->u[i] - s->v[j] == 0) ++deg;
    s->adj_start[i + 1] = s->adj_start[i] + deg;
  }
  const int64_t m = s->adj_start[n];
  if (m > s->adj_cap) {
    int32_t* na = realloc(s->adj, sizeof(int32_t) * (size_t)(m ? m : 1));
    if (!na) return -1;
    s->adj = na;
    s->adj_cap = m;
  }
  for (int32_t i = 0; i < n; ++i) {
    const int64_t* row = s->c + (size_t)i * n;
    int32_t k = s->adj_start[i];
    for (int32_t j = 0; j < n; ++j)
      if (row[j] - s->u[i] - s->v[j] == 0) s->adj[k++] = j;
  }
  return 0;
}

/* TightPhase::bfs, :254-278: layered BFS from free rows; limit = length of
 * the shortest augmenting path. */
static int tp_bfs(kmo_state* s) {
  const int32_t n = s->n;
  int32_t qh = 0, qt = 0;
  int32_t* q = s->queue;
  for (int32_t i = 0; i < n; ++i) {
    s->dist[i] = -1;
    if (s->mrow[i] < 0) { s->dist[i] = 0; q[qt++] = i; }
  }
  s->limit = INT32_MAX;
  while (qh < qt) {
    const int32_t i = q[qh++];
    if (s->dist[i] >= s->limit) continue;
    for (int32_t a = s->adj_start[i]; a < s->adj_start[i + 1]; ++a) {
      const int32_t i2 = s->mcol[s->adj[a]];
      if (i2 < 0) {
        if (s->dist[i] + 1 < s->limit) s->limit = s->dist[i] + 1;
      } else if (s->dist[i2] < 0) {
        s->dist[i2] = s->dist[i] + 1;
        q[qt++] = i2;
      }
    }
  }
  return s->limit != INT32_MAX;
}

/* TightPhase::dfs, :280-298 (recursive, adjacency order). */
static int tp_dfs(kmo_state* s, int32_t i) {
  for (; s->it[i] < s->adj_start[i + 1]; ++s->it[i]) {
    const int32_t j = s->adj[s->it[i]];
    const int32_t i2 = s->mcol[j];
    int ok = 0;
    if (i2 < 0) ok = (s->dist[i] + 1 == s->limit);
    else ok = (s->dist[i2] == s->dist[i] + 1) && tp_dfs(s, i2);
    if (ok) { s->mcol[j] = i; s->mrow[i] = j; return 1; }
  }
  s->dist[i] = -1;
  return 0;
}

/* TightPhase::augment_all, :301-308 */
static int32_t tp_augment(kmo_state* s) {
  if (!tp_bfs(s)) return 0;
  memcpy(s->it, s->adj_start, sizeof(int32_t) * (size_t)s->n);
  int32_t paths = 0;
  for (int32_t i = 0; i < s->n; ++i)
    if (s->mrow[i] < 0 && s->dist[i] == 0 && tp_dfs(s, i)) ++paths;
  return paths;
}

/* solve_batched_km, :313-381, on an already-quantized matrix chat (the
 * caller applies kmo_quantize; at B = N it is the identity, test :44-52).
 * Returns 0, -1 (alloc), -2 (no positive finite delta), -3 ("batched km: no
 * augmenting path after search", :353-354). */
int kmo_solve_batched(const int64_t* chat, int32_t n, int64_t* u_out,
                      int64_t* v_out, int32_t* row_to_col, int64_t* total_cost,
                      int64_t* phases_out, int64_t* dual_steps_out,
                      int64_t* trace, int64_t trace_cap) {
  kmo_state s;
  memset(&s, 0, sizeof(s));
  s.n = n;
  s.c = chat;
  s.u = u_out;
  s.v = v_out;
  s.mrow = row_to_col;
  s.mcol = malloc(sizeof(int32_t) * (size_t)n);
  s.rrow = malloc((size_t)n);
  s.rcol = malloc((size_t)n);
  s.slack = malloc(sizeof(int64_t) * (size_t)n);
  s.queue = malloc(sizeof(int32_t) * (size_t)n);
  s.adj_start = malloc(sizeof(int32_t) * ((size_t)n + 1));
  s.dist = malloc(sizeof(int32_t) * (size_t)n);
  s.it = malloc(sizeof(int32_t) * (size_t)n);
  s.trace = trace;
  s.trace_cap = trace_cap;
  int rc = 0;
  if (!s.mcol || !s.rrow || !s.rcol || !s.slack || !s.queue || !s.adj_start ||
      !s.dist || !s.it) { rc = -1; goto done; }

  /* initial reductions, :323-333 */
  for (int32_t i = 0; i < n; ++i) {
    const int64_t* row = chat + (size_t)i * n;
    int64_t lo = row[0];
    for (int32_t j = 1; j < n; ++j) if (row[j] < lo) lo = row[j];
    s.u[i] = lo;
  }
  for (int32_t j = 0; j < n; ++j) {
    int64_t lo = KMO_INF;
    for (int32_t i = 0; i < n; ++i) {
      const int64_t d = chat[(size_t)i * n + j] - s.u[i];
      if (d < lo) lo = d;
    }
    s.v[j] = lo;
  }
  for (int32_t i = 0; i < n; ++i) { s.mrow[i] = -1; s.mcol[i] = -1; }

  int32_t matched = 0;
  int64_t phases = 0;
  while (matched < n) { /* :340-366 */
    rc = bs_run(&s);
    if (rc) goto done;
    if (tp_build(&s)) { rc = -1; goto done; }
    const int32_t paths = tp_augment(&s);
    if (paths <= 0) { rc = -3; goto done; }
    matched += paths;
    ++phases;
  }
  int64_t tot = 0;
  for (int32_t i = 0; i < n; ++i) tot += chat[(size_t)i * n + s.mrow[i]];
  *total_cost = tot;
  *phases_out = phases;
  *dual_steps_out = s.dual_steps;
done:
  free(s.mcol); free(s.rrow); free(s.rcol); free(s.slack); free(s.queue);
  free(s.adj_start); free(s.adj); free(s.dist); free(s.it);
  return rc;
}

/* Seeded e-maxx KM (SURVEY.md fact 0.5, 4th bullet): the solve_km loop of
 * hungarian.cpp:67-119 started from the batched reductions of :323-333
 * instead of u = v = 0.  Much cheaper than the batched restatement at
 * n = 16384 (no per-phase n^2 tight-graph rebuild); it is cross-validated
 * against kmo_solve_batched / oracle/_ref on every smaller config before it is
 * trusted for config 5 (tests/test_oracle.py). */
int kmo_solve_km_seeded(const int32_t* C, int32_t n, int64_t* u_out,
                        int64_t* v_out, int32_t* row_to_col,
                        int64_t* total_cost) {
  int64_t* u = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* v = malloc(sizeof(int64_t) * ((size_t)n + 1));
  int64_t* minv = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* entry = malloc(sizeof(int64_t) * ((size_t)n + 1));
  int32_t* p = malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* way = malloc(sizeof(int32_t) * (size_t)n);
  char* used = calloc((size_t)n + 1, 1);
  int32_t* usedlist = malloc(sizeof(int32_t) * ((size_t)n + 1));
  if (!u || !v || !minv || !entry || !p || !way || !used || !usedlist) return -1;
  /* seed: the reductions of hungarian.cpp:323-333 */
  for (int32_t i = 0; i < n; ++i) {
    const int32_t* row = C + (size_t)i * n;
    int64_t lo = row[0];
    for (int32_t j = 1; j < n; ++j) if (row[j] < lo) lo = row[j];
    u[i] = lo;
  }
  for (int32_t j = 0; j < n; ++j) v[j] = KMO_INF;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t* row = C + (size_t)i * n;
    for (int32_t j = 0; j < n; ++j) {
      const int64_t d = (int64_t)row[j] - u[i];
      if (d < v[j]) v[j] = d;
    }
  }
  v[n] = 0;
  for (int32_t j = 0; j <= n; ++j) p[j] = -1;
  for (int32_t r = 0; r < n; ++r) {
    /* One row search of hungarian.cpp:67-104 with the O(n) per-step dual
     * update deferred: `shift` is the running sum of deltas, minv holds
     * (true minv + shift), and a row entering the used set at shift s is
     * stored as u - s, so every relaxation reads C - u - v unchanged.  The
     * deferred updates are applied once when the free column is reached. */
    p[n] = r;
    int32_t j0 = n, nused = 0;
    int64_t shift = 0;
    entry[n] = 0;
    for (int32_t j = 0; j < n; ++j) minv[j] = KMO_INF;
    for (;;) {
      used[j0] = 1;
      usedlist[nused++] = j0;
      const int32_t i0 = p[j0];
      const int32_t* row = C + (size_t)i0 * n;
      const int64_t ui = u[i0];
      int64_t best = KMO_INF;
      int32_t j1 = -1;
      for (int32_t j = 0; j < n; ++j) {
        if (used[j]) continue;
        const int64_t cur = (int64_t)row[j] - ui - v[j];
        if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
        if (minv[j] < best) { best = minv[j]; j1 = j; }
      }
      shift = best; /* true delta of this step = best - previous shift */
      j0 = j1;
      if (p[j0] == -1) break;
      entry[j0] = shift;
      u[p[j0]] -= shift;
    }
    for (int32_t k = 0; k < nused; ++k) {
      const int32_t j = usedlist[k];
      v[j] -= shift - entry[j];
      u[p[j]] += shift;
      used[j] = 0;
    }
    while (j0 != n) {
      const int32_t j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    }
  }
  int64_t tot = 0;
  for (int32_t j = 0; j < n; ++j) {
    row_to_col[p[j]] = j;
    tot += C[(size_t)p[j] * n + j];
  }
  memcpy(u_out, u, sizeof(int64_t) * (size_t)n);
  memcpy(v_out, v, sizeof(int64_t) * (size_t)n);
  *total_cost = tot;
  free(u); free(v); free(minv); free(entry); free(p); free(way); free(used);
  free(usedlist);
  return 0;
}
