# Owner-sharded warmup at N=2 and N=4: multi-GPU parity (bit-exact vs a
# simulated cluster) and the warmup-stage step time, sharded vs replicated.
mkdir -p gpurun_out
N=${N:-2}
out=gpurun_out/r2_shard_n$N.txt; : > $out
[ -z "$NOCHECK" ] && timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29611 tests/multigpu_check.py > gpurun_out/r2_shard_multi_n$N.txt 2>&1; echo "multigpu_check rc=$?" >> $out
tail -2 gpurun_out/r2_shard_multi_n$N.txt >> $out
run() {  # label env...
  label=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus $N --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
  echo "$label $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k: round(v["ms_per_launch"]*v["launches"]/10,3) for k,v in d["kernels"].items()})')" >> $out
}
run replicated BL_WARMUP_SHARD=0
for cfg in ${CFGS:-4:2:0:256 4:2:1:256}; do  # pieces:ctas_per_sm:shape:block
  IFS=: read k c sh b <<< "$cfg"
  run shard_k${k}_c${c}_s${sh}_b$b BL_SHARD_PIECES=$k BL_SHARD_CTAS_PER_SM=$c BL_SHARD_SHAPE=$sh BL_LOSSLESS_BLOCK=$b
done
