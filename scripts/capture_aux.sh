set -u
mkdir -p gpurun_out
T=${1:-r02f}
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_baseline_shapes.py tests/test_gpu_api.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$?
B="python bench.py --profile --no-graph --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_loss|k_update|k_final_ln' -s 3 -c 6 -o gpurun_out/${T}_loss -f $B > gpurun_out/${T}_loss.log 2>&1; echo ncu_loss_rc=$?
python profiles/extract_ncu.py gpurun_out/${T}_loss.ncu-rep gpurun_out/${T}_ncu_loss.csv
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -s 2500 -c 1500 --csv \
  --log-file gpurun_out/${T}_fact_tensor_launches.csv python bench.py --estimator factorized_sqrt_r \
  --rank 128 --dense-update tensor --profile --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_fact.log 2>&1; echo fact_rc=$?
rm -f gpurun_out/*.ncu-rep
