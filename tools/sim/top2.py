"""CPU model of the warp engine's incremental epochs (oracle/kmb_mirror.c
kmm_solve_incr, restated with numpy) with a second-best key per column, to
count how many epoch-start re-relaxes a top-2 cache would avoid.  Not product
code.  Usage: python tools/sim/top2.py [instances]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2005_01182_b200 import workloads as W

INF = np.iinfo(np.int64).max


def solve(C, seed=1, continue_bfs=False):
    n = C.shape[0]
    C = C.astype(np.int64)
    u = C.min(1) if seed == 1 else np.zeros(n, np.int64)
    v = np.zeros(n, np.int64)
    k1v = np.full(n, INF); k1r = np.full(n, -1)
    k2v = np.full(n, INF); k2r = np.full(n, -1); k2ok = np.ones(n, bool)
    match_row = np.full(n, -1); match_col = np.full(n, -1)
    rcol = np.zeros(n, bool); dc = np.zeros(n, np.int64)
    w = u.copy(); root = np.arange(n); tree_par = np.full(n, -1)
    rows = list(range(n)); head = 0; D = 0; first = seed == 1; nfree = n; ep = 0
    stats = dict(epochs=0, relaxed=0, rerelax_full=0, dirty=0, resolved=0, epochs_all_resolved=0,
                 rerelax_rows_needed=0, rounds=0)
    pending = []  # continue_bfs: free columns found earlier in this epoch
    claim_ep = np.full(n, -1); claim_col = np.zeros(n, np.int64)
    dirty_cols = None

    def relax(rs, cols=None):
        for i in rs:
            x = C[i] - w[i]
            idx = np.arange(n) if cols is None else cols
            xv = x[idx]
            # insert (xv, i) into top-2 (keys ordered by (value, row))
            better1 = (xv < k1v[idx]) | ((xv == k1v[idx]) & (i < k1r[idx]))
            better2 = ~better1 & ((xv < k2v[idx]) | ((xv == k2v[idx]) & (i < k2r[idx])))
            j1 = idx[better1]
            k2v[j1] = k1v[j1]; k2r[j1] = k1r[j1]
            k1v[j1] = xv[better1]; k1r[j1] = i
            j2 = idx[better2]
            k2v[j2] = xv[better2]; k2r[j2] = i

    while nfree > 0:
        stats["rounds"] += 1
        if dirty_cols is not None:
            # epoch start: survivors over the dirty columns only (key1 and key2 from scratch)
            if len(dirty_cols):
                k1v[dirty_cols] = INF; k1r[dirty_cols] = -1; k2v[dirty_cols] = INF; k2r[dirty_cols] = -1
                k2ok[dirty_cols] = True
                relax(rows[:head], dirty_cols)
            dirty_cols = None
        relax(rows[head:])
        stats["relaxed"] += len(rows) - head
        head = len(rows)
        if first:
            v = k1v.copy(); first = False
        s = np.where(rcol, INF, k1v - v)
        m = s.min()
        if m > D and not pending:
            D = m
        tight = np.nonzero(~rcol & (k1v - v == D))[0]
        found = []
        for j in tight:
            rcol[j] = True; dc[j] = D; p = k1r[j]; tree_par[j] = p; rt = root[p]
            i2 = match_col[j]
            if i2 < 0:
                if claim_ep[rt] != ep or j < claim_col[rt]:
                    claim_ep[rt] = ep; claim_col[rt] = j
                found.append(j)
            else:
                w[i2] = u[i2] - D; root[i2] = rt; rows.append(i2)
        if continue_bfs:
            nrow_before = head
            pending += found
            # keep growing while the tight closure still adds rows
            if len(rows) > head or (found and m <= D):
                if len(rows) > head:
                    continue
            found = pending
            pending = []
            if not found:
                continue
        if not found:
            continue
        relax(rows[head:]); stats["relaxed"] += len(rows) - head; head = len(rows)
        claimed = lambda r: claim_ep[root[r]] == ep
        dirty = []
        for j in range(n):
            if rcol[j]:
                if claimed(tree_par[j]):
                    v[j] -= D - dc[j]; rcol[j] = False
                    dirty.append(j)  # reached column of a dissolved tree
            elif k1r[j] >= 0 and claimed(k1r[j]):
                dirty.append(j)
        # a top-2 cache resolves a dirty column whose key1 row left if key2 is a
        # valid second-min over the reached rows and its row survived
        res = 0
        need = []
        for j in dirty:
            if k1r[j] >= 0 and not claimed(k1r[j]):
                # reached column of a dissolved tree whose argmin row survived? (cannot be:
                # the argmin is its tree parent) -- treat as needing recompute
                need.append(j); continue
            if k2ok[j] and k2r[j] >= 0 and not claimed(k2r[j]):
                k1v[j], k1r[j] = k2v[j], k2r[j]; k2v[j] = INF; k2r[j] = -1; k2ok[j] = False
                res += 1
            else:
                need.append(j)
        # key2 rows that dissolve invalidate key2 (a new second is unknown)
        for j in range(n):
            if k2r[j] >= 0 and claimed(k2r[j]):
                k2ok[j] = False; k2v[j] = INF; k2r[j] = -1
        surv = [i for i in rows if not claimed(i)]
        for i in rows:
            if claimed(i):
                u[i] = w[i] + D
        for j in found:
            if claim_col[root[tree_par[j]]] != j:
                continue
            nfree -= 1
            while True:
                i = tree_par[j]; nx = match_row[i]; match_row[i] = j; match_col[j] = i
                if nx < 0: break
                j = nx
        stats["epochs"] += 1; stats["dirty"] += len(dirty); stats["resolved"] += res
        stats["rerelax_full"] += len(surv)
        if need:
            stats["rerelax_rows_needed"] += len(surv)
        else:
            stats["epochs_all_resolved"] += 1
        rows = surv; head = len(surv); dirty_cols = np.array(need, np.int64)
        ep += 1
    tot = int(C[np.arange(n), match_row].sum())
    return tot, u, v, stats


if __name__ == "__main__" and os.environ.get("CFG"):
    import oracle as O
    c = W.CONFIGS[os.environ["CFG"]].make()
    for cb in (False, True):
        tot, u, v, st = solve(c, 1, cb)
        ref = O.ref_solve_batched_km(c) if c.shape[0] <= 1024 else None
        ok = ref is None or (tot == ref.total_cost and np.array_equal(u, ref.u))
        print("continue_bfs", cb, "ok", ok, {k: st[k] for k in ("rounds", "epochs", "relaxed", "rerelax_full")})
    sys.exit(0)

if __name__ == "__main__":
    import oracle as O
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    c = W.CONFIGS["c3"].make(batch=k)
    agg = {}
    for t in range(k):
        tot, u, v, st = solve(c[t])
        ref = O.ref_solve_batched_km(c[t])
        assert tot == ref.total_cost and np.array_equal(u, ref.u) and np.array_equal(v, ref.v), t
        for a, b in st.items():
            agg[a] = agg.get(a, 0) + b
    print({a: b / k for a, b in agg.items()})
