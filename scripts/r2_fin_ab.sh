mkdir -p gpurun_out
out=gpurun_out/r2_fin16_ab.txt; : > $out
for i in 1 2 3; do
  for v in new prev; do
    if [ $v = prev ]; then export BL_LIB_PATH=$PWD/build/lib_prev.so; else unset BL_LIB_PATH; fi
    timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$v $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"]*1e3,1), {a: round(b["ms_per_launch"]*1e3,1) for a,b in k.items()})')" >> $out
  done
done
