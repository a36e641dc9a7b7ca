"""GPU: the C++ drop-in (include/kmb_ot.hpp) against the unmodified reference,
written like the reference's test_hungarian.cpp (tests/cpp/test_drop_in.cpp)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "build", "test_drop_in")


@pytest.mark.gpu
def test_cpp_drop_in():
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: run tests/cpp/build.sh where /root/reference exists")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout


@pytest.mark.gpu
def test_cpp_reference_harness():
    """The B200 solvers as SolverSpec plugins inside the reference's run_suite."""
    b = os.path.join(HERE, "cpp", "build", "test_harness")
    if not os.path.exists(b):
        pytest.fail(f"{b} missing: run tests/cpp/build.sh where /root/reference exists")
    out = subprocess.run([b], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "harness: 0 failed" in out.stdout


@pytest.mark.gpu
def test_cpp_stream_ordered_and_graph():
    """C++ host through the C ABI: the stream-ordered call, its CUDA-graph
    capture/replay, the multi-context split and per-instance statuses."""
    b = os.path.join(HERE, "cpp", "build", "test_stream")
    if not os.path.exists(b):
        pytest.fail(f"{b} missing: run tests/cpp/build.sh")
    out = subprocess.run([b], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "test_stream: ok" in out.stdout
