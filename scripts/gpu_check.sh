#!/bin/bash
# One gpurun call: GPU tests, default bench, config-5 launch list.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh <tag> [pytest selection]'
set -u
T=${1:-chk}
SEL=${2:-tests}
mkdir -p gpurun_out
timeout 1200 python -m pytest $SEL -m gpu -q -x --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/${T}_bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -s 2500 -c 1500 --csv \
  --log-file gpurun_out/${T}_fact_tensor_launches.csv python bench.py --estimator factorized_sqrt_r \
  --rank 128 --dense-update tensor --profile --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_fact.log 2>&1; echo fact_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -s 1200 -c 500 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --profile --no-graph --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1; echo launches_rc=$?
