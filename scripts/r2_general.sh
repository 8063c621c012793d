# k5/k6_general (general-path tiles in their own kernels) vs inline: parity + A/B timing.
mkdir -p gpurun_out
out=gpurun_out/r2_general.txt; : > $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_boundary.py -m gpu -x -q > gpurun_out/r2_general_tests.txt 2>&1; echo "tests rc=$?" >> $out
tail -n 2 gpurun_out/r2_general_tests.txt >> $out
for i in 1 2; do
for w in "config1" "config1 --sim-workers 4" "bert-base --sim-workers 4" "bert-large"; do
  for v in split inline; do
    if [ $v = inline ]; then export BL_GENERAL_SPLIT_MAX_TILES=0; else unset BL_GENERAL_SPLIT_MAX_TILES; fi
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$v [$w] $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"]*1e3,1), "us; k5", round(k["k5_update_a"]["ms_per_launch"]*1e3,1), "k6", round(k["k6_update_b"]["ms_per_launch"]*1e3,1))')" >> $out
  done
done
done
