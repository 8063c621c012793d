# Push-based sharded-warmup exchange (BL_SHARD_PUSH=1) vs pull: parity + timing at N=4 and N=2.
mkdir -p gpurun_out
out=gpurun_out/r2_push_ab.txt; : > $out
for N in ${NS:-4 2}; do
  BL_SHARD_PUSH=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2961$N tests/multigpu_check.py > gpurun_out/r2_push_multi_n$N.txt 2>&1; echo "N=$N push multigpu_check rc=$? $(grep -c PASS gpurun_out/r2_push_multi_n$N.txt)" >> $out
  for i in ${IS:-1 2}; do
    for v in pull push; do
      if [ $v = push ]; then export BL_SHARD_PUSH=1; else unset BL_SHARD_PUSH; fi
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2973$i bench.py --gpus $N --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
      echo "N=$N $v $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"],4), {a: round(b["ms_per_launch"]*b["launches"]/d["steps"],3) for a,b in k.items()})')" >> $out
    done
  done
done
