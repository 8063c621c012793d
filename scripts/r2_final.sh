# End-of-round confirmation on one 4-GPU box: full GPU suite, default bench (N=1),
# reference arm, multi-GPU benches (N=2, 4), sharded warmup, small-collective sweep.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/final_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/final_gputests.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/final_smoke.txt 2>&1; echo rc=$? >> gpurun_out/final_smoke.txt
timeout 900 python bench.py > gpurun_out/final_bench_n1.json 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/final_bench_n$n.json 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n --steps 10 --warmup 3 --stage warmup --no-e2e > gpurun_out/final_warmup_n$n.json 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2965$n bench_sweep.py --sizes-mb 1,2,4,8,16,32,64,256,1024 > gpurun_out/final_sweep_n$n.jsonl 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2>&1
