#!/bin/sh
# Build the C++ drop-in tests against the reference headers (needs
# /root/reference, i.e. this container) and the in-tree libraries; the binary
# travels to the GPU box with the snapshot.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF=${OT_REF_DIR:-/root/reference/proj}
mkdir -p "$HERE/build"
# simulated-shard protocol library (no reference needed)
g++ -O2 -std=c++17 -fPIC -shared -I"$ROOT/paper_2005_01182_b200/csrc" "$HERE/shard_sim.cpp" \
  -o "$HERE/build/libshardsim.so"
# C ABI + CUDA runtime host test (stream-ordered call, CUDA graph, multi-context)
CUDA_HOME=${CUDA_HOME:-/usr/local/cuda}
g++ -O2 -std=c++17 -I"$ROOT/include" -I"$CUDA_HOME/include" "$HERE/test_stream.cpp" \
  -L"$ROOT/paper_2005_01182_b200" -lkmb -L"$CUDA_HOME/lib64" -lcudart \
  -Wl,-rpath,'$ORIGIN/../../../paper_2005_01182_b200' -o "$HERE/build/test_stream"
if [ ! -f "$REF/include/ot/hungarian.hpp" ]; then
  echo "reference headers absent; keeping prebuilt binary" ; exit 0
fi
mkdir -p "$HERE/build"
g++ -O2 -std=c++20 -I"$REF/include" -I"$REF/tests" -I"$ROOT/include" "$HERE/test_drop_in.cpp" \
  -L"$ROOT/oracle/_ref" -lotref -L"$ROOT/paper_2005_01182_b200" -lkmb \
  -Wl,-rpath,'$ORIGIN/../../../oracle/_ref' -Wl,-rpath,'$ORIGIN/../../../paper_2005_01182_b200' \
  -o "$HERE/build/test_drop_in"
# the reference harness (run_suite, make_solver, calibration rule) with the B200
# solvers registered as SolverSpecs: the reference library is compiled from its
# own sources for this test
g++ -O2 -std=c++20 -I"$REF/include" -I"$REF/tests" -I"$ROOT/include" "$HERE/test_harness.cpp" \
  "$REF/src/bench.cpp" "$REF/src/core.cpp" "$REF/src/hungarian.cpp" "$REF/src/netsimplex.cpp" \
  "$REF/src/auction.cpp" "$REF/src/scaling.cpp" "$REF/src/datasets.cpp" "$REF/src/io.cpp" \
  -L"$ROOT/paper_2005_01182_b200" -lkmb \
  -Wl,-rpath,'$ORIGIN/../../../paper_2005_01182_b200' -o "$HERE/build/test_harness"

