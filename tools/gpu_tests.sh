#!/bin/bash
# GPU test pass with per-test durations.  Usage: bash tools/gpu_tests.sh tag [pytest args...]
tag=${1:-rXX}; shift
O=gpurun_out; mkdir -p $O
timeout ${KMB_TEST_TIMEOUT:-2700} python -m pytest -m gpu -x -q -p no:cacheprovider --timeout=900 \
  --durations=60 "$@" > $O/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" | tee -a $O/${tag}_pytest_gpu.log; tail -3 $O/${tag}_pytest_gpu.log
