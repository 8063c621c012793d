mkdir -p gpurun_out
out=gpurun_out/r2_k3t_ab.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/r2_k3t_tests.txt 2>&1; echo "tests rc=$?" >> $out; tail -n 1 gpurun_out/r2_k3t_tests.txt >> $out
for i in 1 2; do
for w in "bert-large --sim-workers 4" "bert-base --sim-workers 4"; do
  for v in new prev; do
    if [ $v = prev ]; then export BL_LIB_PATH=$PWD/build/lib_prev.so; else unset BL_LIB_PATH; fi
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$v [$w] $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"]*1e3,1), "us k3", round(k["k3_server_reduce"]["ms_per_launch"]*1e3,1))')" >> $out
  done
done
done
