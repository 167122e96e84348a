#!/bin/bash
# Profile capture recipe (run under gpurun on ONE B200; never multi-rank):
#   gpurun --timeout 3000 -- 'bash profiles/capture.sh <tag> [model]'
# Produces in gpurun_out/:
#   <tag>_bench.json          the default bench line (no profiler attached)
#   <tag>_launches.csv        every launch of 2 eager steps with its device time + DRAM bytes
#                             (--cache-control none: L2 state as in the real step;
#                             serialised, so compare SHARES, not absolutes)
#   <tag>_ncu_gemm.csv        --set full of the 4 GEMMs of decoder layer 1 (+ one repeat)
#   <tag>_ncu_aux.csv         --set full of LN / attention / ext-finalize / final LN / loss / update
#   <tag>_ncu_lmhead.csv      --set full of the LM-head GEMM (K6)
#   <tag>_fact_launches.csv   launch list of one config-5 step (factorized r=128, tensor update)
#   <tag>_ncu_update.csv      --set full of two config-5 tensor-update launches (EPI_UPDATE32)
set -u
TAG=${1:-prof}
MODEL=${2:-opt-13b}
mkdir -p gpurun_out
B="python bench.py --model $MODEL --profile --no-graph --steps 2 --warmup 3 --no-cpu-baseline"
F="python bench.py --model $MODEL --estimator factorized_sqrt_r --rank 128 --dense-update tensor --profile --no-graph --steps 1 --warmup 1 --no-cpu-baseline"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python bench.py --model $MODEL > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --model $MODEL --estimator factorized_sqrt_r --rank 128 --dense-update tensor --no-cpu-baseline \
  --no-materialising > gpurun_out/${TAG}_bench_fact.log 2>&1
tail -1 gpurun_out/${TAG}_bench_fact.log > gpurun_out/${TAG}_bench_fact_tensor.json
timeout 900 ncu $M -s 1200 -c 500 --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
# layer GEMMs: skip step 0 + layer 0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 165 -c 5 \
  -o gpurun_out/${TAG}_gemm -f $B > gpurun_out/${TAG}_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_ln_row|k_attn|k_ext_finalize|k_loss|k_final_ln|k_embed|k_update' -s 330 -c 9 \
  -o gpurun_out/${TAG}_aux -f $B > gpurun_out/${TAG}_aux.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:256, \(int\)3, \(int\)0, \(int\)0, \(int\)1' \
  -s 2 -c 1 -o gpurun_out/${TAG}_lmhead -f $B > gpurun_out/${TAG}_lmhead.log 2>&1
timeout 900 ncu $M -s 2500 -c 1500 --log-file gpurun_out/${TAG}_fact_launches.csv $F > gpurun_out/${TAG}_fact.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:256, \(int\)6,' -s 20 -c 2 \
  -o gpurun_out/${TAG}_update -f $F > gpurun_out/${TAG}_update.log 2>&1
# summaries on the box (the .ncu-rep files are large; gpurun brings back <= 64 MiB)
for r in gemm aux lmhead update; do
  python profiles/extract_ncu.py gpurun_out/${TAG}_${r}.ncu-rep gpurun_out/${TAG}_ncu_${r}.csv
done
ncu -i gpurun_out/${TAG}_gemm.ncu-rep --page source --csv --print-source sass -k regex:k_gemm --launch-count 1 \
  > gpurun_out/${TAG}_gemm_qkv_source.csv 2>/dev/null
python profiles/launch_table.py gpurun_out/${TAG}_launches.csv 30 > gpurun_out/${TAG}_launches_summary.txt
python profiles/launch_table.py gpurun_out/${TAG}_fact_launches.csv 30 > gpurun_out/${TAG}_fact_launches_summary.txt
gzip -9 -f gpurun_out/${TAG}_*.ncu-rep
# keep the bundle under gpurun's 64 MiB: drop the reports, largest first
for f in gpurun_out/${TAG}_aux.ncu-rep.gz gpurun_out/${TAG}_update.ncu-rep.gz gpurun_out/${TAG}_lmhead.ncu-rep.gz gpurun_out/${TAG}_gemm.ncu-rep.gz; do
  [ "$(du -sm gpurun_out | cut -f1)" -gt 58 ] && rm -f "$f"
done
du -sh gpurun_out
echo done
