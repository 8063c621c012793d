# Owner-sharded warmup at N=2 and N=4: multi-GPU parity (bit-exact vs a
# simulated cluster) and the warmup-stage step time, sharded vs replicated.
mkdir -p gpurun_out
N=${N:-2}
out=gpurun_out/r2_shard_n$N.txt; : > $out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29611 tests/multigpu_check.py > gpurun_out/r2_shard_multi_n$N.txt 2>&1; echo "multigpu_check rc=$?" >> $out
tail -5 gpurun_out/r2_shard_multi_n$N.txt >> $out
run() {  # label env...
  label=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus $N --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
  echo "$label $(tail -1 /tmp/b.json)" >> $out
}
run shard BL_WARMUP_SHARD=1
run replicated BL_WARMUP_SHARD=0
run shard_b128 BL_WARMUP_SHARD=1 BL_LOSSLESS_BLOCK=128
