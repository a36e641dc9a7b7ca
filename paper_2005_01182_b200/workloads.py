"""Seeded synthetic inputs for the five BASELINE.json configs.

The generators are C (``csrc/kmb_gen.c``, counter-based splitmix64 streams,
OpenMP over elements / instances — results do not depend on the thread
count).  Config k uses seed k.  Each returns a C-contiguous int32 array: the
same buffer feeds the oracle (widened to int64) and the GPU.

The paper's own datasets (MNIST/CIFAR/GloVe, PAPER.md) are not available
here; these seeded inputs with BASELINE.json's shapes, sizes and value
distributions stand in for them.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _build

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lib = None


def _load():
    global _lib
    if _lib is None:
        path = _build.GEN_SO
        if not os.path.exists(path):
            _build.build_gen()
        lib = C.CDLL(path)
        lib.kmb_gen_uniform.argtypes = [_i32p, C.c_int32, C.c_int32, C.c_int32, C.c_uint64]
        lib.kmb_gen_geometric.argtypes = [_i32p, C.c_int32, C.c_double, C.c_uint64]
        lib.kmb_gen_embedding_batch.argtypes = [_i32p, C.c_int32, C.c_int32, C.c_int32,
                                                C.c_int32, C.c_double, C.c_uint64]
        lib.kmb_gen_gmm.argtypes = [_i32p, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64]
        _f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        _f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
        lib.kmb_gen_geometric_points.argtypes = [_f64p, _f64p, C.c_int32, C.c_uint64]
        lib.kmb_gen_gmm_points.argtypes = [_f64p, _f64p, C.c_int32, C.c_int32, C.c_double,
                                           C.c_double, C.c_uint64]
        lib.kmb_gen_embedding_vectors.argtypes = [_f32p, _f32p, C.c_int32, C.c_int32, C.c_int32,
                                                  C.c_int32, C.c_uint64]
        lib.kmb_fnv1a64.argtypes = [C.c_void_p, C.c_int64]
        lib.kmb_fnv1a64.restype = C.c_uint64
        _lib = lib
    return _lib


def uniform(n: int, lo: int, hi: int, seed: int) -> np.ndarray:
    """n x n, i.i.d. uniform integers in [lo, hi], row-major."""
    out = np.empty((n, n), np.int32)
    _load().kmb_gen_uniform(out, n, lo, hi, seed)
    return out


def geometric(n: int, scale: float = 1e6, seed: int = 2) -> np.ndarray:
    """Two sets of n points U[0,1)^2 (fp64); llround(scale * squared distance)."""
    out = np.empty((n, n), np.int32)
    _load().kmb_gen_geometric(out, n, scale, seed)
    return out


def embedding_batch(batch: int, n: int = 128, dim: int = 300, scale: float = 1e4,
                    seed: int = 3, first: int = 0) -> np.ndarray:
    """Instances first..first+batch-1, each two n-sets of dim-D N(0,1) fp32
    vectors; llround(scale * Euclidean distance).  Shape (batch, n, n)."""
    out = np.empty((batch, n, n), np.int32)
    _load().kmb_gen_embedding_batch(out, first, batch, n, dim, scale, seed)
    return out


def gmm(n: int, comps: int = 16, box: float = 100.0, sigma: float = 1.0,
        scale: float = 1e3, seed: int = 4) -> np.ndarray:
    """Two sets of n 3-D points from a comps-component GMM; llround(scale * sq dist)."""
    out = np.empty((n, n), np.int32)
    _load().kmb_gen_gmm(out, n, comps, box, sigma, scale, seed)
    return out


def points(key: str, batch: int | None = None, first: int = 0):
    """The point sets behind configs 2-4 (same seeded streams as their cost
    matrices): (a, b, dim, scale, squared).  Config 3 returns float32
    (batch, n, 300) arrays, configs 2 and 4 float64 (n, dim)."""
    lib = _load()
    if key == "c2":
        a = np.empty((1024, 2)); b = np.empty((1024, 2))
        lib.kmb_gen_geometric_points(a, b, 1024, 2)
        return a, b, 2, 1e6, True
    if key == "c4":
        a = np.empty((4096, 3)); b = np.empty((4096, 3))
        lib.kmb_gen_gmm_points(a, b, 4096, 16, 100.0, 1.0, 4)
        return a, b, 3, 1e3, True
    if key == "c3":
        bt = 4096 if batch is None else batch
        a = np.empty((bt, 128, 300), np.float32); b = np.empty((bt, 128, 300), np.float32)
        lib.kmb_gen_embedding_vectors(a, b, first, bt, 128, 300, 3)
        return a, b, 300, 1e4, False
    raise KeyError(key)


def fnv1a64(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(_load().kmb_fnv1a64(a.ctypes.data, a.nbytes))


@dataclass(frozen=True)
class Config:
    key: str
    n: int
    batch: int
    description: str

    def make(self, batch: int | None = None, first: int = 0) -> np.ndarray:
        """The config's cost matrix (n, n), or (batch, n, n) for config 3.
        ``batch``/``first`` select instances first..first+batch-1 of config 3."""
        if self.key == "c1":
            return uniform(256, 0, 1000, seed=1)
        if self.key == "c2":
            return geometric(1024, 1e6, seed=2)
        if self.key == "c3":
            return embedding_batch(self.batch if batch is None else batch, 128, 300, 1e4, seed=3,
                                   first=first)
        if self.key == "c4":
            return gmm(4096, 16, 100.0, 1.0, 1e3, seed=4)
        if self.key == "c5":
            return uniform(16384, 0, 10**6, seed=5)
        raise KeyError(self.key)


CONFIGS = {
    "c1": Config("c1", 256, 1, "n=256, i.i.d. U{0..1000}"),
    "c2": Config("c2", 1024, 1, "n=1024, U[0,1)^2 points, llround(1e6*sq dist)"),
    "c3": Config("c3", 128, 4096, "4096 x n=128, 300-D N(0,1) fp32, llround(1e4*dist)"),
    "c4": Config("c4", 4096, 1, "n=4096, 16-comp 3-D GMM, llround(1e3*sq dist)"),
    "c5": Config("c5", 16384, 1, "n=16384, i.i.d. U{0..1e6} (1 GiB int32)"),
}
