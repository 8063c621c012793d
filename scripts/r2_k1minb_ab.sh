mkdir -p gpurun_out
out=gpurun_out/r2_k1minb_ab.txt; : > $out
for i in 1 2; do
for w in "config1 --sim-workers 4" "config1" "bert-large"; do
  for v in cur k1m3 k1m4; do
    export BL_LIB_PATH=$PWD/build/lib_$v.so
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$v [$w] $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"]*1e3,1), "us k1", round(k["k1_worker_compress"]["ms_per_launch"]*1e3,1))')" >> $out
  done
done
done
