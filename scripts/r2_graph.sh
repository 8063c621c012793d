# CUDA-graph step replay: parity suite (graphs on by default), and BL_GRAPH=0 vs 1 timings.
mkdir -p gpurun_out; out=gpurun_out/r2_graph_ab.txt; : > $out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_boundary.py tests/test_gpu_acceptance.py -q -x -p no:cacheprovider > gpurun_out/r2_graph_tests.txt 2>&1
for g in 0 1; do
  for args in "--workload config1" "--workload config1 --sim-workers 4" "--workload bert-large"; do
    echo "graph=$g $args|$(BL_GRAPH=$g python bench.py $args --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)" >> $out
  done
done
