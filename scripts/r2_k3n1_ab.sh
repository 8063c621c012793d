# K3<1> variants at BERT-L N=1 (alternating).
mkdir -p gpurun_out
out=gpurun_out/r2_k3n1_ab.txt; : > $out
for i in 1 2; do
  for v in base k3a k3b k3c; do
    if [ $v = base ]; then unset BL_LIB_PATH; else export BL_LIB_PATH=$PWD/build/lib_$v.so; fi
    timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$v $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"],4), round(k["k3_server_reduce"]["ms_per_launch"],4))')" >> $out
  done
done
