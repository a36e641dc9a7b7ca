#!/bin/bash
# One GPU-box session: GPU parity suite, bench line, launch list, then ncu
# full captures of each config's dominant kernel.  Usage (from the repo root):
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tag] [stages]'
# stages: any of t (tests) b (bench) l (launch list) n (ncu full); default "tbln"
tag=${1:-rXX}; stages=${2:-tbln}
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${tag}_gpu.txt 2>&1
if [[ $stages == *t* ]]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${tag}_pytest_gpu.log 2>&1
  echo "pytest exit $?" | tee -a $O/${tag}_pytest_gpu.log; tail -3 $O/${tag}_pytest_gpu.log
fi
if [[ $stages == *b* ]]; then
  timeout 900 python bench.py > $O/${tag}_bench.json 2> $O/${tag}_bench.err; echo "bench exit $?"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${tag}_bench_ref.json 2>> $O/${tag}_bench.err; echo "ref exit $?"
fi
if [[ $stages == *l* ]]; then
  B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-configs"
  timeout 600 $B > $O/${tag}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/${tag}_launches.csv $B > $O/${tag}_ncu_launches.log 2>&1; echo "launches exit $?"
fi
if [[ $stages == *n* ]]; then
  for spec in "c3 k_warp_batch 0" "c5 k_solve 0" "c4 k_cluster 0" "c2 k_big 0" "c1 k_cta_batch 0"; do
    set -- $spec; cfg=$1; k=$2; eng=$3
    P="python tools/prof_run.py --config $cfg --iters 2 --engine $eng"
    timeout 600 $P > $O/${tag}_prof_${cfg}_plain.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
        -o $O/${tag}_ncu_${cfg}_${k} -f $P > $O/${tag}_ncu_${cfg}.log 2>&1; echo "ncu $cfg $k exit $?"
  done
fi
