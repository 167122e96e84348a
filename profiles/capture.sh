#!/bin/bash
# Profile capture recipe (run under gpurun on ONE B200; never multi-rank):
#   gpurun --timeout 1800 -- 'bash profiles/capture.sh <tag> [model]'
# Produces in gpurun_out/:
#   <tag>_launches.csv   every launch of 2 eager steps with its device time
#                        (cold-cache, serialised: compare SHARES, not absolutes)
#   <tag>_gemm.ncu-rep   --set full of the 4 GEMMs of decoder layer 1
#   <tag>_aux.ncu-rep    --set full of the LN / attention / ext-finalize / loss kernels
set -u
TAG=${1:-prof}
MODEL=${2:-opt-13b}
mkdir -p gpurun_out
B="python bench.py --model $MODEL --profile --no-graph --steps 2 --warmup 3 --no-cpu-baseline"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 500 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
# layer GEMMs: 161 k_gemm launches per step (4 per layer + LM head); skip step 0 + layer 0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 165 -c 5 \
  -o gpurun_out/${TAG}_gemm -f $B > gpurun_out/${TAG}_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_ln_ext|k_attn|k_ext_finalize|k_loss|k_final_ln|k_embed|k_update' -s 330 -c 8 \
  -o gpurun_out/${TAG}_aux -f $B > gpurun_out/${TAG}_aux.log 2>&1
echo done
