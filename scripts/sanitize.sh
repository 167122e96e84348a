#!/bin/bash
# compute-sanitizer evidence on the final code (one gpurun call):
#   gpurun --timeout 3000 -- 'bash scripts/sanitize.sh <tag>'
# memcheck over the GPU tests that drive every kernel family and over the 13B-schedule shape
# (CTA pairs, stream-K tail, half-width tails, fp32-master update); racecheck + synccheck over
# the d = 1024 shape (CTA pairs, half tails) -- both tools serialise and instrument every
# shared-memory access, so the full 13B shape does not fit their time budget.
set -u
T=${1:-san}
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() { echo "== $*" >> gpurun_out/${T}_sanitizer.txt; timeout 1500 "$@" >> gpurun_out/${T}_sanitizer.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_sanitizer.txt; }
: > gpurun_out/${T}_sanitizer.txt
run $CS --tool memcheck python scripts/sanitize_shapes.py
run $CS --tool memcheck python -m pytest tests/test_gpu_kernels.py tests/test_gpu_scorer.py tests/test_gpu_abort.py tests/test_gpu_split_graph.py tests/test_gpu_fast_update.py tests/test_gpu_api.py -m gpu -q -x -p no:cacheprovider
run $CS --tool racecheck --racecheck-report hazard python scripts/sanitize_shapes.py --small
run $CS --tool synccheck python scripts/sanitize_shapes.py --small
grep -E "^==|rc=|ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|sanitize shapes ok" gpurun_out/${T}_sanitizer.txt
