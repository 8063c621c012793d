# A/B of the in-tree library against build/lib_prev.so on several workloads (alternating), + parity.
mkdir -p gpurun_out
out=gpurun_out/r2_ab_${TAG:-x}.txt; : > $out
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -m gpu -q -x > gpurun_out/r2_ab_${TAG:-x}_tests.txt 2>&1; echo "tests rc=$?" >> $out; tail -n 1 gpurun_out/r2_ab_${TAG:-x}_tests.txt >> $out; fi
for i in 1 2; do
for w in "config1" "config1 --sim-workers 4" "bert-large --sim-workers 4" "bert-large"; do
  for v in new prev; do
    if [ $v = prev ]; then export BL_LIB_PATH=$PWD/build/lib_prev.so; else unset BL_LIB_PATH; fi
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$v [$w] $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"]*1e3,1), "us", {a: round(b["ms_per_launch"]*1e3,1) for a,b in k.items() if a.startswith("k")})')" >> $out
  done
done
done
