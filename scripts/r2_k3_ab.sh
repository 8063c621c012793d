# K3 (NT=4) variants at N=4, compression-stage bench, alternating.
mkdir -p gpurun_out
out=gpurun_out/r2_k3_ab.txt; : > $out
for i in 1 2; do
  for v in base k3a k3b k3c; do
    if [ $v = base ]; then unset BL_LIB_PATH; else export BL_LIB_PATH=$PWD/build/lib_$v.so; fi
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 2962$i bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e > /tmp/b.json 2>&1
    echo "$v $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"],4), round(k["k3_server_reduce"]["ms_per_launch"],4), round(k["k1_worker_compress"]["ms_per_launch"],4))')" >> $out
  done
done
