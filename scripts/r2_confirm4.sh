# Confirmation on 4 GPUs: full GPU suite, sweep at N=2/4, BERT-L N=1.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputests_4gpu_b.txt 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2967$n bench_sweep.py --sizes-mb 1,2,4,8,16,32,64 > gpurun_out/r2_sweep_n${n}_b.jsonl 2>&1
done
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_b.json 2>&1
