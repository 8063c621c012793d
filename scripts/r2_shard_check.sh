# Sharded warmup: multi-GPU parity (incl. the mid-warmup collective m/v read) + default warmup timing.
mkdir -p gpurun_out
N=${N:-2}
out=gpurun_out/r2_shard_check_n$N.txt; : > $out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29611 tests/multigpu_check.py > gpurun_out/r2_shard_multi_n$N.txt 2>&1; echo "multigpu_check rc=$?" >> $out
tail -2 gpurun_out/r2_shard_multi_n$N.txt >> $out
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus $N --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
tail -1 /tmp/b.json >> $out
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus $N --steps 10 --warmup 3 --no-e2e > /tmp/b.json 2>&1
tail -1 /tmp/b.json >> $out
