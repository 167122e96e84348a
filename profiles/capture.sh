#!/bin/bash
# Profile capture recipe (run under gpurun on ONE B200; never multi-rank):
#   gpurun --timeout 2400 -- 'bash profiles/capture.sh <tag> [model]'
# Produces in gpurun_out/:
#   <tag>_bench.json         the default bench line (no profiler attached)
#   <tag>_launches.csv       every launch of 2 eager steps with its device time
#                            (--cache-control none: L2 state as in the real step;
#                            serialised, so compare SHARES, not absolutes)
#   <tag>_gemm.ncu-rep       --set full of the 4 GEMMs of decoder layer 1
#   <tag>_aux.ncu-rep        --set full of the LN / attention / ext-finalize / loss kernels
#   <tag>_fact_launches.csv  launch list of one config-5 step (factorized r=128)
set -u
TAG=${1:-prof}
MODEL=${2:-opt-13b}
mkdir -p gpurun_out
B="python bench.py --model $MODEL --profile --no-graph --steps 2 --warmup 3 --no-cpu-baseline"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 600 python bench.py --model $MODEL > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 1200 -c 500 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
# layer GEMMs: 161 k_gemm launches per step (4 per layer + LM head); skip step 0 + layer 0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 165 -c 5 \
  -o gpurun_out/${TAG}_gemm -f $B > gpurun_out/${TAG}_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_ln_row|k_attn|k_ext_finalize|k_loss|k_final_ln|k_embed|k_update' -s 330 -c 8 \
  -o gpurun_out/${TAG}_aux -f $B > gpurun_out/${TAG}_aux.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 2500 -c 1500 --csv \
  --log-file gpurun_out/${TAG}_fact_launches.csv python bench.py --model $MODEL --estimator factorized_sqrt_r \
  --rank 128 --profile --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_fact.log 2>&1
# summaries on the box (the .ncu-rep files are large; gpurun brings back <= 64 MiB)
python profiles/extract_ncu.py gpurun_out/${TAG}_gemm.ncu-rep gpurun_out/${TAG}_ncu_gemm.csv
python profiles/extract_ncu.py gpurun_out/${TAG}_aux.ncu-rep gpurun_out/${TAG}_ncu_aux.csv
ncu -i gpurun_out/${TAG}_gemm.ncu-rep --page source --csv --print-source sass -k regex:k_gemm --launch-count 1 \
  > gpurun_out/${TAG}_gemm_qkv_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_aux.ncu-rep --page source --csv --print-source sass -k regex:k_attn --launch-count 1 \
  > gpurun_out/${TAG}_attn_source.csv 2>/dev/null
gzip -9 -f gpurun_out/${TAG}_gemm.ncu-rep gpurun_out/${TAG}_aux.ncu-rep
# keep the bundle under gpurun's 64 MiB: drop the aux report first, then the GEMM report
for f in gpurun_out/${TAG}_aux.ncu-rep.gz gpurun_out/${TAG}_gemm.ncu-rep.gz; do
  [ "$(du -sm gpurun_out | cut -f1)" -gt 58 ] && rm -f "$f"
done
du -sh gpurun_out
echo done
