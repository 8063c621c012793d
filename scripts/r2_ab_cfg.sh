# BERT-L, config 1 (n=1, sim 4), BERT-Base sim 4 with the current build; parity suite.
mkdir -p gpurun_out; out=gpurun_out/r2_cfg_runs.txt; : > $out
for args in "--workload bert-large" "--workload config1" "--workload config1 --sim-workers 4" "--workload bert-base --sim-workers 4"; do
  echo "$args|$(python bench.py $args --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)" >> $out
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/r2_parity_b.txt 2>&1
