# Sharded-warmup reduce load variants at N=4 (alternating).
mkdir -p gpurun_out
out=gpurun_out/r2_lossless_ab.txt; : > $out
for i in 1 2; do
  for v in base ld256 u4; do
    if [ $v = base ]; then unset BL_LIB_PATH; else export BL_LIB_PATH=$PWD/build/lib_$v.so; fi
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 2972$i bench.py --gpus 4 --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
    echo "$v $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"],4), "reduce", round(k["average"]["ms_per_launch"],4), "w2", round(k["w2_warmup_b"]["ms_per_launch"],4))')" >> $out
  done
done
