"""B200-native exact assignment solver (Kuhn-Munkres and batched KM, arXiv
2005.01182) behind the reference's solver entry point.

Layers:
  include/kmb.h               C ABI (the drop-in boundary)
  csrc/kmb_solver.cu          persistent grid / cluster engines (one instance, any n)
  csrc/kmb_warp.cu            warp engine (one warp per small instance, batches)
  csrc/kmb_batch.cu           CTA engines (one CTA per small instance)
  csrc/kmb_shard.cu           column-sharded single instance over ranks (NCCL)
  csrc/kmb_auction.cu         Gauss-Seidel auction (ot::solve_auction[_scaled])
  csrc/kmb_costs.cu           cost construction (ot::build_instance)
  csrc/kmb_capi.cu            context, workspace, staging
  api.py                      Python mirror of ot::solve_km / solve_batched_km /
                              solve_auction / solve_auction_scaled
  workloads.py                seeded inputs for the BASELINE configs
"""
from .api import (KMB_SEED_BATCHED, KMB_SEED_KM, KmbError, KmbUnavailable, Result, Solver,
                  calibrate_auction_eps, calibrate_batch_level, default_solver, load_library,
                  quantize_costs, solve_auction, solve_auction_scaled, solve_batch_multi,
                  solve_batched_km, solve_km)

__all__ = ["KMB_SEED_BATCHED", "KMB_SEED_KM", "KmbError", "KmbUnavailable", "Result", "Solver",
           "calibrate_auction_eps", "calibrate_batch_level", "default_solver", "load_library",
           "quantize_costs", "solve_auction", "solve_auction_scaled", "solve_batch_multi",
           "solve_batched_km",
           "solve_km"]
