"""B200-native exact assignment solver (Kuhn-Munkres and batched KM, arXiv
2005.01182) behind the reference's solver entry point.

Layers:
  include/kmb.h               C ABI (the drop-in boundary)
  csrc/kmb_solver.cu          persistent grid engine (one instance, any n)
  csrc/kmb_batch.cu           SMEM engine (one CTA per small instance)
  csrc/kmb_capi.cu            context, workspace, staging
  api.py                      Python mirror of ot::solve_km / ot::solve_batched_km
  workloads.py                seeded inputs for the BASELINE configs
"""
from .api import (KMB_SEED_BATCHED, KMB_SEED_KM, KmbError, KmbUnavailable, Result, Solver,
                  calibrate_batch_level, default_solver, load_library, quantize_costs,
                  solve_batched_km, solve_km)

__all__ = ["KMB_SEED_BATCHED", "KMB_SEED_KM", "KmbError", "KmbUnavailable", "Result", "Solver",
           "calibrate_batch_level", "default_solver", "load_library", "quantize_costs",
           "solve_batched_km", "solve_km"]
