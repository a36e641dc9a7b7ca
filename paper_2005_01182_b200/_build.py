"""In-tree builds of the native libraries (no JIT cache: the built .so files
travel to the GPU box with the repo snapshot).

* ``libkmb.so``      — the product: CUDA kernels for sm_100a + the C ABI of
  ``include/kmb.h`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``).
* ``libkmb_gen.so``  — seeded workload generators (C, OpenMP).
"""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB_SO = os.path.join(PKG, "libkmb.so")
GEN_SO = os.path.join(PKG, "libkmb_gen.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["kmb_solver.cu", "kmb_batch.cu", "kmb_warp.cu", "kmb_shard.cu", "kmb_costs.cu",
              "kmb_auction.cu", "kmb_big.cu", "kmb_cluster.cu", "kmb_wide.cu", "kmb_shard_dev.cu", "kmb_capi.cu"]
CU_HEADERS = ["kmb_common.cuh", "kmb_internal.h", "kmb_launch.h", "kmb_shard_proto.h", "kmb_stage.h"]


def _run(cmd: list[str]) -> None:
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out.stdout + out.stderr)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_gen(force: bool = False) -> str:
    src = os.path.join(CSRC, "kmb_gen.c")
    if force or _stale(GEN_SO, [src]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              src, "-o", GEN_SO, "-lm"])
    return GEN_SO


def build_lib(force: bool = False, extra: list[str] | None = None) -> str:
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in CU_HEADERS] + [os.path.join(INCLUDE, "kmb.h")]
    if force or _stale(LIB_SO, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC, *srcs, "-o", LIB_SO + ".tmp",
               "-lcudart", "-ldl"]
        cmd += extra or []
        _run(cmd)
        os.replace(LIB_SO + ".tmp", LIB_SO)
    return LIB_SO


def build_all(force: bool = False) -> None:
    build_gen(force)
    build_lib(force)
