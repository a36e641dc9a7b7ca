/*
 * kmb.h — C ABI of the B200-native exact assignment solver (KM / batched KM).
 *
 * Drop-in boundary for the reference's solver entry points
 *   ot::solve_km          /root/reference/proj/include/ot/hungarian.hpp:39-40
 *                         (impl. proj/src/hungarian.cpp:55-136)
 *   ot::solve_batched_km  hungarian.hpp:53-56 (impl. hungarian.cpp:313-381)
 * and of their plugin registration  ot::bench::make_solver("km" /
 * "batched_km")  (proj/src/bench.cpp:404-422, SolverSpec bench.hpp:24-29).
 * The reference interface is C++ (OTInstance in, SolveResult + optional
 * DualPotentials / Matching out, exceptions on bad input); this ABI carries the
 * same data as plain pointers and sizes so any FFI can bind it, and
 * include/kmb_ot.hpp rebuilds the reference's C++ signatures on top of it.
 *
 * Semantics (identical to the reference on the same inputs):
 *   cost         n x n int32, row-major with leading dimension ld (>= n),
 *                entries in [0, 2^29) (the reference only requires >= 0; the
 *                device engine keeps reduced costs in 32 bits).
 *   seed         KMB_SEED_KM      = u = v = 0, the start of solve_km (:63)
 *                KMB_SEED_BATCHED = row/column reductions (:323-333), the start
 *                                   of solve_batched_km.
 *                Final duals are bit-identical to the reference solver with the
 *                same start; the total cost is the optimum.
 *   row_to_col   assignment, n entries (Matching::row_to_col, hungarian.hpp:12-14)
 *   u, v         row / column duals, n entries each, int64
 *                (DualPotentials, hungarian.hpp:19-22)
 *   total_cost   sum_i cost[i][row_to_col[i]], int64 (objective_int, core.cpp:76-90)
 *   time_budget_s  0 = none; checked once per phase on the device
 *                (hungarian.cpp:341-346); on expiry stats->converged = 0 and the
 *                partial matching is returned (row_to_col = -1 for free rows).
 * Pointers may be host or device memory (detected per call).  Work runs on the
 * context's stream (kmb_set_stream); every call returns after the results
 * reached the caller's buffers and the device status was checked, like the
 * reference's synchronous functions.
 *
 * Return value: 0 ok; > 0 invalid input (message via kmb_last_error(), the
 * reference's std::invalid_argument cases); < 0 CUDA / internal error.
 * There is no CPU fallback: without a usable B200 every solve returns < 0.
 */
#ifndef KMB_H
#define KMB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMB_ABI_VERSION 1

enum kmb_seed { KMB_SEED_KM = 0, KMB_SEED_BATCHED = 1 };

enum kmb_status {
  KMB_OK = 0,
  KMB_EINVAL = 1,        /* bad argument (n <= 0, null pointer, ld < n) */
  KMB_ENEGATIVE = 2,     /* "costs must be nonnegative" (core.cpp:144-145) */
  KMB_ERANGE = 3,        /* _i32 calls: a cost >= 2^29 (32-bit engines' range);
                            _i64 calls: validate_instance's headroom
                            (core.cpp:47-53) exceeded                        */
  KMB_ECUDA = -1,        /* CUDA runtime error                             */
  KMB_EINTERNAL = -2,    /* engine invariant violated                      */
  KMB_ENODEVICE = -3     /* no sm_100 device                               */
};

enum kmb_option {
  KMB_OPT_MAX_CTAS = 1,     /* grid engine: upper bound on CTAs (0 = #SMs)      */
  /* 2 (continue the BFS past a free column, ABI 1) was removed: the
     incremental-epoch engines never read it, and a CPU model of them measured
     more rounds with it (config 1: 185 -> 236; config 3: 368 -> 379) */
  KMB_OPT_ENGINE = 3,       /* 0 auto: single instances CTA n<=256, single-CTA
                               n<=1792, replicated cluster n<=4608, grid beyond;
                               batches warp or CTA (n<=256, by residency),
                               single-CTA (n<=4096);
                               1 grid (persistent), 4 warp (n <= 256),
                               5 cluster (grid engine on one <=16-CTA cluster),
                               6 CTA (n <= 256),
                               8 single-CTA (one 512-thread CTA, n <= 4096),
                               11 replicated cluster (one <=16-CTA cluster per
                               instance, row state replicated per CTA,
                               n <= 5120; KMB_OPT_MAX_CTAS = cluster size);
                               stats->engine 7 = column-sharded (host
                               exchange), 9 = wide (int64 costs,
                               kmb_solve_i64), 10 = column-sharded (device
                               exchange)                                       */
  KMB_OPT_WARPS_PER_SM = 4, /* warp engine: resident instances per SM (0 = max);
                               bounds the L2 working set of streamed matrices   */
  /* 5 (the 16-bit warp-engine mode of ABI 1) was removed: slower */
  KMB_OPT_PIPELINE = 6      /* host-input batches (>= 256 instances): chunks the
                               H2D copy is split into so solves overlap it.
                               0 = auto (tapered: min(8, batch/128) equal
                               chunks, the last one split by halving so the
                               solve after the final copy is short; measured
                               on config 3, tools/e2e_probe.py);
                               k > 0: k equal chunks (<= 64);
                               k < 0: tapered from |k| equal chunks            */
  ,
  KMB_OPT_RESIDENT16 = 7    /* warp engine, 64 < n <= 256: keep a 16-bit copy of
                               every row (offsets from the row minimum) in a
                               workspace and relax from it - half the L2
                               footprint and bytes per row; rows, and past
                               ~n/16 of them whole instances, that do not fit
                               16 bits stay int32.  0 = auto (by size: n > 128
                               from 128 MiB of matrices, n <= 128 between
                               192 and 448 MiB), 1 = always, -1 = never.
                               Results are identical either way.               */
};

typedef struct kmb_stats {
  int64_t phases;          /* augmentation phases (not a parity target)      */
  int64_t dual_steps;      /* dual adjustments: equals the reference's count */
  int64_t rows_scanned;    /* cost rows streamed by the reduced-cost scan    */
  int64_t cost_bytes_read; /* 4*n*(rows_scanned + n) + 16*segment_rows       */
  double seconds;          /* device time of the solve (CUDA events)         */
  int32_t converged;       /* 0 when the time budget expired                 */
  int32_t engine;          /* the engine that ran (KMB_OPT_ENGINE numbering) */
  int64_t rounds;          /* search rounds (relax | min | absorb)           */
  int64_t stage_ns[6];     /* grid engine, CTA 0's clock (ns): relax, barrier 1,
                              absorb, barrier 2, epoch end, barrier 3;
                              warp engine: SM cycles summed over instances in
                              relax, min, absorb, epoch end (0 unless built
                              with -DKMB_WARP_STAGE_CLOCKS=1)                */
  int64_t max_instance_cycles; /* batch engines: slowest instance (SM clocks) */
  int64_t sum_instance_cycles; /* batch engines: sum over instances          */
  int64_t segment_rows;    /* grid/cluster engines: (row, 4-column segment)
                              pairs of the epoch-start dirty-segment relaxes
                              (16 B each; rows_scanned counts full rows)     */
} kmb_stats;

typedef struct kmb_context kmb_context;

int kmb_create(int device, kmb_context** out);
void kmb_destroy(kmb_context* ctx);
/* cudaStream_t passed as void* (NULL = the legacy default stream). */
int kmb_set_stream(kmb_context* ctx, void* cuda_stream);
int kmb_set_option(kmb_context* ctx, int option, int64_t value);

/* One n x n instance (configs 1, 2, 4, 5). */
int kmb_solve_i32(kmb_context* ctx, const int32_t* cost, int32_t n, int64_t ld, int32_t seed,
                  double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                  int64_t* total_cost, kmb_stats* stats);

/* `batch` independent n x n instances stored back to back (config 3); n <= 4096
 * (one warp or one CTA per instance for n <= 256, one 512-thread CTA above).
 * row_to_col, u, v: batch*n entries; total_cost: batch entries; stats (optional)
 * receives the sums over the batch. */
int kmb_solve_batch_i32(kmb_context* ctx, const int32_t* costs, int32_t batch, int32_t n,
                        int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
                        int64_t* total_cost, kmb_stats* stats);

/* Stream-ordered variant of kmb_solve_batch_i32 for device-resident batches:
 * enqueues the solve on the context's stream and returns at once (no host
 * synchronisation, so back-to-back batches pipeline and the call can be
 * captured in a CUDA graph once a first call has sized the workspace; capture
 * in cudaStreamCaptureModeRelaxed, since the call queries pointer attributes).  All
 * six buffers must be device memory; status[b] (batch int32) receives instance
 * b's outcome when the stream reaches it: 0 ok, KMB_ENEGATIVE, KMB_ERANGE, or
 * another nonzero code for an engine fault.  The return value reports argument
 * and launch errors only. */
int kmb_solve_batch_async_i32(kmb_context* ctx, const int32_t* costs, int32_t batch, int32_t n,
                              int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
                              int64_t* total_cost, int32_t* status);

/* ---- 64-bit costs: the reference's own cost type (OTInstance::cost) --------
 * kmb_solve_i64 / kmb_solve_batch_i64: kmb_solve_i32 / kmb_solve_batch_i32 on
 * int64 costs over the reference's whole admissible range — any nonnegative
 * cost within validate_instance's headroom n * maxC * (2n + 2) <= 2^62
 * (core.cpp:47-53; KMB_ERANGE "supply * cost magnitude too large for 64-bit
 * arithmetic" beyond it).  Validation runs on the device; costs < 2^29 are
 * narrowed on the device and solved by the 32-bit engines, larger costs by the
 * wide engine (64-bit keys and duals, stats->engine 9).  Same duals as the
 * reference. */
int kmb_solve_i64(kmb_context* ctx, const int64_t* cost, int32_t n, int64_t ld, int32_t seed,
                  double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                  int64_t* total_cost, kmb_stats* stats);
int kmb_solve_batch_i64(kmb_context* ctx, const int64_t* costs, int32_t batch, int32_t n,
                        int32_t seed, int32_t* row_to_col, int64_t* u, int64_t* v,
                        int64_t* total_cost, kmb_stats* stats);

/* quantize_costs (hungarian.cpp:33-53) on the device: N = max cost (1 when
 * every cost is 0), chat[k] = floor(cost[k] * B / N), lossless = every product
 * divisible.  chat (count entries) may be NULL; host or device pointers.
 * KMB_EINVAL with the reference's messages "quantize_costs: B must be
 * positive" / "quantize_costs: B * max cost overflows". */
int kmb_quantize_i64(kmb_context* ctx, const int64_t* cost, int64_t count, int64_t B, int64_t* chat,
                     int64_t* N, int32_t* lossless);

/* ot::solve_batched_km (hungarian.cpp:313-381) end to end on the device:
 * validation, quantization to chat = floor(C * B / N), the reductions and the
 * search on chat.  u, v: the duals of chat (DualPotentials); row_to_col; total_cost
 * = the objective on the caller's costs C; chat (n*n, optional) / N / lossless:
 * QuantizedCosts.  B = N * n reproduces solve_km's optimum (lossless).  Error
 * messages are the reference's ("solve_batched_km: costs must be nonnegative",
 * "quantize_costs: ..."). */
int kmb_solve_batched_km_i64(kmb_context* ctx, const int64_t* cost, int32_t n, int64_t B,
                             double time_budget_s, int32_t* row_to_col, int64_t* u, int64_t* v,
                             int64_t* total_cost, int64_t* chat, int64_t* N, int32_t* lossless,
                             kmb_stats* stats);

/* One process, several GPUs (BASELINE config 3 "instances sharded across
 * GPUs" without one process per GPU): the batch is split into nctx contiguous
 * slices of equal size (+-1) and slice k is solved by kmb_solve_batch_i32 on
 * ctxs[k] (normally one context per device), all slices concurrently, one host
 * thread per extra context.  When the contexts span several devices the five
 * buffers must be host memory (pinned for copy/solve overlap).  stats: sums
 * over the slices, seconds = the slowest slice.  Errors name the slice. */
int kmb_solve_batch_multi_i32(kmb_context* const* ctxs, int32_t nctx, const int32_t* costs,
                              int32_t batch, int32_t n, int32_t seed, int32_t* row_to_col,
                              int64_t* u, int64_t* v, int64_t* total_cost, kmb_stats* stats);

/* ---- column-sharded single instance across ranks/GPUs (config 5) ----------
 * Rank r owns columns [col_begin, col_begin + ncols) of the n x n matrix
 * (`slab`: n rows x ncols, leading dimension ld).  Every rank calls
 * kmb_solve_sharded_i32 collectively; each returns the full assignment and u
 * (replicated) and the v of its own columns.  The per-round min-slack combine
 * and the entry exchanges go through NCCL (kmb_shard_init_nccl; rank 0 makes
 * the id with kmb_nccl_unique_id and the caller broadcasts it) or through
 * caller callbacks (kmb_shard_init_callbacks; e.g. torch.distributed gloo). */
typedef int (*kmb_allreduce_min_i64_fn)(int64_t* inout, int32_t count, void* user);
typedef int (*kmb_allgather_fn)(const void* send, int64_t bytes, void* recv, void* user);
int kmb_nccl_unique_id(uint8_t* out128);
int kmb_shard_init_nccl(kmb_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id128);
int kmb_shard_init_callbacks(kmb_context* ctx, int32_t nranks, int32_t rank,
                             kmb_allreduce_min_i64_fn allreduce_min, kmb_allgather_fn allgather,
                             void* user);
int kmb_solve_sharded_i32(kmb_context* ctx, const int32_t* slab, int32_t n, int64_t ld,
                          int32_t col_begin, int32_t ncols, int32_t seed, int32_t* row_to_col,
                          int64_t* u, int64_t* v_slab, int64_t* total_cost, kmb_stats* stats);

/* ---- column-sharded single instance, exchange on the device ---------------
 * The same column sharding with no host round trip per round: one persistent
 * kernel per rank (the grid engine with its row-side state replicated on every
 * rank); per round each rank stores its min-slack partial and its appended
 * rows / free columns into every rank's replica (peer stores over NVLink) and
 * the ranks meet at a system-scope counting barrier in rank 0's memory.
 * Collective setup: every rank calls kmb_shard_dev_open (allocates its window
 * and returns its 64-byte CUDA IPC handle and the slab width: rank r holds
 * columns [r * slab_cols, min(n, (r + 1) * slab_cols))), the caller allgathers
 * the handles, every rank calls kmb_shard_dev_connect, then
 * kmb_solve_sharded_dev_i32 collectively (kmb_shard_init_* must be set up too:
 * two host barriers per solve order rank 0's reset of its control block).
 * Outputs as kmb_solve_sharded_i32; stats->engine 10.
 * kmb_solve_sharded_local_i32 runs the same kernel with `nranks` ranks as CTA
 * groups of one launch on this context's GPU (replicas side by side; checked
 * equal after the solve): the protocol on a one-GPU box, whole matrix in. */
int kmb_shard_dev_open(kmb_context* ctx, int32_t n, int32_t nranks, int32_t rank, int32_t* slab_cols,
                       uint8_t* handle64);
int kmb_shard_dev_connect(kmb_context* ctx, const uint8_t* handles64);
int kmb_solve_sharded_dev_i32(kmb_context* ctx, const int32_t* slab, int32_t n, int64_t ld,
                              int32_t col_begin, int32_t ncols, int32_t seed, int32_t* row_to_col,
                              int64_t* u, int64_t* v_slab, int64_t* total_cost, kmb_stats* stats);
int kmb_solve_sharded_local_i32(kmb_context* ctx, const int32_t* cost, int32_t n, int64_t ld,
                                int32_t nranks, int32_t seed, int32_t* row_to_col, int64_t* u,
                                int64_t* v, int64_t* total_cost, kmb_stats* stats);

/* ---- auction (the reference's other unit-capacity solver, auction.hpp) ---
 * Gauss-Seidel auction, bit-identical to ot::solve_auction (scaled = 0,
 * epsilon = AuctionConfig::epsilon) and ot::solve_auction_scaled (scaled = 1,
 * epsilon = epsilon0, theta, epsilon_final; <= 0 picks the reference's
 * defaults): same bids, same double prices, same assignment.  `batch`
 * independent n x n instances back to back (n <= 18000); host or device
 * pointers; every output optional.  Per instance: prices (n doubles),
 * row_to_col (n; -1 for rows a budget left unassigned), total_cost of the
 * assigned pairs, bids (SolveResult::iterations), converged, and the epsilon
 * of the last round (exact = converged && epsilon * n < 1, auction.cpp:172).
 * seconds (optional): device time.  Errors: KMB_EINVAL with the reference's
 * messages for epsilon <= 0 / theta <= 1, KMB_ENEGATIVE for negative costs. */
typedef struct {
  int32_t scaled;
  double epsilon;
  double theta;
  double epsilon_final;
  int64_t max_bids;
  double time_budget_s;
} kmb_auction_config;
int kmb_auction_i32(kmb_context* ctx, const int32_t* costs, int32_t batch, int32_t n,
                    const kmb_auction_config* cfg, double* prices, int32_t* row_to_col,
                    int64_t* total_cost, int64_t* bids, int32_t* converged,
                    double* epsilon_last, double* seconds);

/* ---- cost construction (the caller before the path) -----------------------
 * The reference's build_instance (datasets.cpp:184-214) on the GPU:
 * out[b][i][j] = llround(scale * d(a_b[i], b_b[j])) with d the Euclidean
 * distance accumulated in double over the dimensions in order (squared = 1:
 * the squared distance, BASELINE configs 2 and 4).  a: batch x n x dim,
 * b: batch x m x dim, as double (dtype KMB_F64) or float promoted to double
 * (KMB_F32); out: batch x n x m int32.  Pointers may be host or device memory;
 * bit-identical to the reference on the same points.  KMB_ERANGE when a cost
 * does not fit int32 (the output is then undefined). */
enum { KMB_F64 = 0, KMB_F32 = 1 };
int kmb_costs_from_points(kmb_context* ctx, const void* a, const void* b, int32_t dtype,
                          int32_t batch, int32_t n, int32_t m, int32_t dim, double scale,
                          int32_t squared, int32_t* out);

/* Diagnostics: the grid engine's reduced-cost scan with every row in the
 * frontier (one full pass over the matrix per iteration), averaged over
 * `iters` passes; bytes counted = 4*n*n per pass. */
int kmb_bench_scan(kmb_context* ctx, const int32_t* cost, int32_t n, int64_t ld, int32_t iters,
                   double* seconds_per_pass, double* gbytes_per_s);

/* Diagnostics: per-instance counters of the last batch solve, KMB_ISTATS = 11
 * int64 per instance (epochs, dual steps, rows scanned, rounds, SM cycles,
 * cycles in relax / min / absorb / epoch end, %globaltimer start / end). */
int kmb_last_instance_stats(kmb_context* ctx, int64_t* out, int64_t capacity, int64_t* count);

/* Thread-local message of the last failing call on this thread. */
const char* kmb_last_error(void);
int kmb_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KMB_H */
