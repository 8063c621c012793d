# config 0 (8M params, 4 simulated ranks): K1 path variants.
mkdir -p gpurun_out
out=gpurun_out/r2_cfg0_k1.txt; : > $out
for i in 1 2; do
for v in default none r8; do
  case $v in default) E="";; none) E="BL_K1_BULK=none";; r8) E="BL_K1_BULK_R=8";; esac
  env $E timeout 300 python bench.py --workload config1 --sim-workers 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "$v $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"]*1e3,1), {a: round(b["ms_per_launch"]*1e3,1) for a,b in k.items()})')" >> $out
done
done
