"""CPU: the C-ABI library builds for sm_100a, loads, and exports exactly what
include/kmb.h declares; host-side logic (validation, sharding)
behaves like the reference.  No kernel is launched here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2005_01182_b200 import _build, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kmb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(kmb_\w+)\s*\(", src, re.M)))


def test_header_matches_python_binding():
    assert declared_symbols() == sorted(api.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol():
    path = _build.build_lib()
    lib = C.CDLL(path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True)
    exported = set(re.findall(r" T (kmb_\w+)", out.stdout))
    assert exported == set(declared_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB_SO], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_abi_version():
    assert api.load_library().kmb_abi_version() == 1


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(api.KmbUnavailable, match="kmb_create"):
        api.Solver(0)


def test_null_context_errors():
    lib = api.load_library()
    assert lib.kmb_solve_i32(None, None, 4, 4, 1, 0.0, None, None, None, None, None) == 1
    assert b"NULL context" in lib.kmb_last_error()
    assert lib.kmb_set_option(None, 1, 0) == 1


def test_validation_messages():
    with pytest.raises(ValueError, match="requires a unit-capacity square instance"):
        api._validate(np.ones((2, 3)), None, None, "solve_km")
    with pytest.raises(ValueError, match="requires a unit-capacity square instance"):
        api._validate(np.ones((2, 2)), [2, 1], [1, 2], "solve_batched_km")
    with pytest.raises(ValueError, match="dimensions must be positive"):
        api._validate(np.ones((0, 0)), None, None, "solve_km")


def test_bench_sharding_covers_batch():
    import bench
    for world in (1, 2, 3, 4, 8):
        spans = [bench.shard(world, r) for r in range(world)]
        assert spans[0][0] == 0
        assert sum(c for _, c in spans) == bench.BATCH
        for (f0, c0), (f1, _) in zip(spans, spans[1:]):
            assert f0 + c0 == f1


def test_multi_null_contexts_error():
    lib = api.load_library()
    assert lib.kmb_solve_batch_multi_i32(None, 0, None, 1, 4, 1, None, None, None, None, None) == 1
    assert b"no contexts" in lib.kmb_last_error()
    hs = (C.c_void_p * 2)(None, None)
    assert lib.kmb_solve_batch_multi_i32(hs, 2, None, 1, 4, 1, None, None, None, None, None) == 1
    assert b"NULL context" in lib.kmb_last_error()
