// Internal (non-ABI) declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>

#include "kmb.h"
#include "kmb_shard_proto.h"

namespace kmb {

// per-instance stats of the batch engines: phases/epochs, dual steps, rows
// scanned, rounds, SM cycles, cycles in relax / min / absorb / epoch end, then
// %globaltimer at the instance's start and end (ns)
constexpr int KMB_ISTATS = 11;

// Device control block of one single-instance solve.  Counters that are
// recycled between phases are double-buffered by phase parity (see k_solve).
struct Ctrl {
  unsigned long long bar_counter;  // grid barrier (monotone)
  int32_t tail[2];                 // row-list lengths
  int32_t nfound[2];               // free columns absorbed this phase
  int32_t status;                  // 0 ok, <0 internal error
  int32_t stop;                    // time budget expired
  int32_t free_rows;               // unmatched rows when the engine stopped
  int32_t matched;                 // rows matched so far
  int32_t rcnt[3];                 // row appends per barrier interval (k % 3)
  int32_t fcnt[3];                 // free-column appends per barrier interval
  int32_t pad2_[2];
  int64_t phases;
  int64_t dual_steps;
  int64_t rows_scanned;
  int64_t rounds;
  int64_t stage_ns[6];
  int64_t seg_rows;  // (row, 4-column segment) pairs of the dirty-only epoch-start relaxes
  // counting grid barrier (grid engine): per barrier k % 3, arrivals in bits
  // 0-15, row appends in 16-39, free-column appends in 40-63
  unsigned long long cbar[3];
  unsigned long long obj;  // column-sharded engine: the objective, summed over the slabs
};

// ---- column-sharded engine with device-side exchange (k_solve_sharded) --------
// R ranks (GPUs, or CTA groups of one launch when emulated on one GPU), Gr
// CTAs each; rank r holds the columns [r*Gr*W, (r+1)*Gr*W) as an n x Gr*W slab
// and a replica of the row-side state; claims, counters, the barrier word and
// the cross-rank row minima live in rank 0's home block.  Lives in device
// memory (the kernel reads it through a pointer).
constexpr int KMB_MAX_RANKS = 8;
struct ShardDevArgs {
  int32_t R, rank_base, Gr;
  int32_t sys;                         // 1: ranks on several GPUs (system-scope barrier)
  int64_t slab_pitch;
  const int32_t* slab[KMB_MAX_RANKS];  // rank r's cost slab (its own HBM)
  unsigned char* rep[KMB_MAX_RANKS];   // replica bases (peer-mapped for other GPUs)
  int64_t* vout[KMB_MAX_RANKS];        // rank r's v, slab-local columns
  int32_t* rowmin;                     // home: R x n slab row minima
};

struct SolverArgs {
  const int32_t* C;  // n x pitch, row-major, 16 B aligned, pitch % 4 == 0
  int64_t pitch;
  int32_t n;
  int32_t W;          // column slab per CTA (power of two >= 4); G*W >= n
  int32_t seed;       // 0: u = v = 0 (solve_km), 1: reductions (solve_batched_km)
  int32_t prefetch_rows;  // L2 bulk prefetch of appended rows (matrix larger than L2)
  int32_t slab_cache;     // grid / sharded engines: row roots + slab matches in shared memory
  unsigned long long deadline_ns;  // %globaltimer deadline, 0 = none
  int64_t* u;
  int64_t* v;
  int32_t* match_row;
  int32_t* match_col;
  int32_t* tree_par;   // per column
  int32_t* root_row;   // per row
  uint64_t* claim;     // per row, claim_key(phase, col)
  int32_t* list_row[2];
  int64_t* list_w[2];  // the dual shift D at which each listed row was reached (w = u - D)
  int32_t* found;
  int64_t* partial;    // per CTA
  Ctrl* ctrl;
};

cudaError_t launch_solver(const SolverArgs& a, int G, bool cluster, cudaStream_t st);
cudaError_t launch_solver_init(const SolverArgs& a, cudaStream_t st);
cudaError_t launch_objective(const int32_t* C, int64_t pitch, int n, const int32_t* match_row,
                             unsigned long long* out, cudaStream_t st);
size_t solver_smem_bytes(int W);
cudaError_t launch_scan_all(const SolverArgs& a, int G, uint64_t* keys_out, cudaStream_t st);
int solver_threads();
size_t shard_rep_bytes(int n, int G);  // one replica of the row side (G = CTAs over all ranks)
cudaError_t launch_solver_sharded(const SolverArgs& a, const ShardDevArgs* sh_dev, int grid, cudaStream_t st);

// ---- batched small instances (one CTA per instance, costs from L2) ----
struct BatchArgs {
  const int32_t* C;      // batch x n x n (contiguous instances)
  int32_t batch;
  int32_t n;
  int32_t seed;
  int32_t* row_to_col;   // batch x n
  int64_t* u;            // batch x n
  int64_t* v;            // batch x n
  int64_t* total_cost;   // batch
  int64_t* stats;        // batch x KMB_ISTATS (may be null)
  int32_t* status;       // batch (0 ok)
  int32_t carve_batch;   // launch hint: size the carveout for this many (0: batch)
};

int batch_max_n();
cudaError_t launch_batch(const BatchArgs& a, int sm_count, int warps_per_sm, cudaStream_t st,
                         int* grid_out);

}  // namespace kmb

namespace kmb {
// ---- warp engine (one warp per instance, n <= 256) -----------------------------
struct WarpArgs {
  const int32_t* C;      // batch x n x pitch (pitch == warp_pitch(n)), instances back to back
  int32_t batch;
  int32_t n;
  int32_t pitch;
  int32_t seed;
  int32_t* row_to_col;   // batch x n
  int64_t* u;            // batch x n
  int64_t* v;            // batch x n
  int64_t* total_cost;   // batch
  int64_t* stats;        // batch x KMB_ISTATS (may be null)
  int32_t* status;       // batch
  // optional workspace, batch x n x pitch uint16 (n > 64 only): the kernel keeps
  // a 16-bit copy of every row (offsets from the row minimum) and relaxes from it
  uint16_t* C16;
};
int warp_max_n();
int cta_batch_capacity(int n, int sm_count);  // CTA/L2 engine: instances resident at once
// folds per-instance stats + status into 11 int64 (kmb_batch.cu)
cudaError_t launch_batch_summary(const int64_t* stats, const int32_t* status, int32_t batch,
                                 int64_t* out, cudaStream_t st);
int warp_pitch(int n);  // padded row pitch the warp engine requires (32 * columns per lane)
cudaError_t launch_warp_batch(const WarpArgs& a, int sm_count, int warps_per_sm, cudaStream_t st,
                              int* grid_out);
// single-CTA engine for 256 < n <= 4096 (kmb_big.cu)
struct BigArgs {
  const int32_t* C;     // batch instances, row stride ld, instance stride inst_stride
  int64_t ld, inst_stride;
  int32_t batch, n, seed;
  int64_t deadline_ns;  // per-instance time budget (0: none)
  int32_t* row_to_col;  // batch x n
  int64_t* u;           // batch x n
  int64_t* v;           // batch x n
  int64_t* total_cost;  // batch
  int64_t* stats;       // batch x KMB_ISTATS (may be null)
  int32_t* status;      // batch
  int32_t* converged;   // batch (may be null)
  int32_t carve_batch;  // launch hint: size the carveout for this many (0: batch)
};
size_t big_smem_bytes(int n);
int big_max_n();
cudaError_t launch_big(const BigArgs& a, int sm_count, cudaStream_t st);
// replicated cluster engine (kmb_cluster.cu): one <=16-CTA cluster per instance
size_t cluster_smem_bytes(int n, int G);
int cluster_max_n();
cudaError_t launch_cluster(const BigArgs& a, int G, int sm_count, cudaStream_t st);
// Gauss-Seidel auction (kmb_auction.cu)
struct AuctionArgs {
  const int32_t* C;     // batch instances, row stride ld, instance stride inst_stride
  int64_t ld, inst_stride;
  int32_t batch, n;
  int32_t scaled;       // 0: solve_auction (eps0 = epsilon); 1: solve_auction_scaled
  double eps0, theta, eps_final;
  int64_t max_bids;
  int64_t budget_ns;    // 0: no time budget
  long long *cmin, *cmax;  // batch: workspace (validation, max_cost)
  double* prices;       // batch x n (may be null)
  int32_t* row_to_col;  // batch x n (may be null)
  int64_t* total_cost;  // batch (may be null)
  int64_t* bids;        // batch (may be null)
  int32_t* complete;    // batch (may be null)
  double* eps_last;     // batch (may be null)
  int32_t* status;      // batch
};
size_t auction_smem_bytes(int n);
int auction_max_n();
cudaError_t launch_auction(const AuctionArgs& a, int sm_count, cudaStream_t st);
// cost construction (kmb_costs.cu)
template <typename P>
cudaError_t launch_costs(const P* a, const P* b, int32_t batch, int32_t n, int32_t m, int32_t dim,
                         double scale, int32_t squared, int32_t* out, int32_t* bad, cudaStream_t st);
}  // namespace kmb

namespace kmb {
// ---- column-sharded solve (kmb_shard.cu): the collective interface ------------
using Exchange = ShardExchange;  // kmb_shard_proto.h
struct CallbackExchange : Exchange {
  kmb_allreduce_min_i64_fn ar = nullptr;
  kmb_allgather_fn ag = nullptr;
  void* user = nullptr;
  int allreduce_min(int64_t* p, int32_t count) override { return ar(p, count, user); }
  int allgather(const void* s, int64_t bytes, void* r) override { return ag(s, bytes, r, user); }
};
// device-resident column-sharded solve (kmb_shard_dev.cu): per-context state
struct ShardDevState;
void destroy_shard_dev(ShardDevState* p);
struct ShardDevDeleter {
  void operator()(ShardDevState* p) const { destroy_shard_dev(p); }
};
using ShardDevPtr = std::unique_ptr<ShardDevState, ShardDevDeleter>;
// context accessors (the context struct lives in kmb_capi.cu)
std::unique_ptr<Exchange>& context_exchange(kmb_context* c);
ShardDevPtr& context_shard_dev(kmb_context* c);
int context_sm_count(kmb_context* c);
cudaStream_t context_stream(kmb_context* c);
int context_device(kmb_context* c);
void set_last_error(const std::string& msg);
}  // namespace kmb

namespace kmb {
// ---- 64-bit cost path (kmb_wide.cu) ------------------------------------------
struct WideArgs {
  const int64_t* C;     // batch instances, row stride ld, instance stride inst_stride
  int64_t ld, inst_stride;
  int32_t batch, n, seed;
  int64_t deadline_ns;  // per-instance time budget (0: none)
  int32_t* row_to_col;  // batch x n
  int64_t* u;           // batch x n
  int64_t* v;           // batch x n
  int64_t* total_cost;  // batch
  int64_t* stats;       // batch x KMB_ISTATS (may be null)
  int32_t* status;      // batch
  int32_t* converged;   // batch (may be null)
  int64_t* ws64;        // wide_ws64_bytes(n, slots)
  int32_t* ws32;        // wide_ws32_bytes(n, slots)
  int64_t max_cost;     // an instance with a larger cost fails with status 3
};
int wide_slots(int batch, int sm_count);
size_t wide_ws64_bytes(int n, int slots);
size_t wide_ws32_bytes(int n, int slots);
cudaError_t launch_wide(const WideArgs& a, int slots, cudaStream_t st);
cudaError_t launch_minmax_i64(const int64_t* C, int64_t ld, int64_t rows, int32_t cols, long long* out,
                              int sm_count, cudaStream_t st);
cudaError_t launch_convert_i64(const int64_t* C, int64_t ld, int64_t rows, int32_t cols, bool quantize,
                               int64_t B, int64_t N, int64_t* chat, int32_t* narrow, int32_t* lossy,
                               int sm_count, cudaStream_t st);
cudaError_t launch_scale_i64(int64_t* x, int64_t count, int64_t k, int sm_count, cudaStream_t st);
cudaError_t launch_total_i64(const int64_t* C, int64_t ld, int64_t inst_stride, int32_t batch, int32_t n,
                             const int32_t* r2c, int64_t* total, int sm_count, cudaStream_t st);
}  // namespace kmb
