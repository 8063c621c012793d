# Round-2 scale run on a 4-GPU box: bench (compression + warmup stage) at N=1,2,4 and the
# message-size sweep at N=2,4 (fused LL small collective up to 2048 tiles, split kernels above).
mkdir -p gpurun_out
out=gpurun_out/r2_scale.jsonl; : > $out
for st in compression warmup; do
  python bench.py --steps 20 --warmup 5 --stage $st --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $out
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2966$n bench.py --gpus $n --steps 20 --warmup 5 --stage $st --no-e2e 2>/dev/null | tail -1 >> $out
  done
done
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2967$n bench_sweep.py --sizes-mb 1,2,4,8,16,32,64,256,1024 > gpurun_out/r2_sweep_n$n.jsonl 2>&1
  BL_SMALL_MAX_TILES=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2968$n bench_sweep.py --sizes-mb 8,16,32 > gpurun_out/r2_sweep_n${n}_split.jsonl 2>&1
done
