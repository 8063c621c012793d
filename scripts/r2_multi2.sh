mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 tests/multigpu_check.py > gpurun_out/r2_multi2b.txt 2>&1; echo rc=$? >> gpurun_out/r2_multi2b.txt
for st in warmup compression; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --stage $st --no-e2e > gpurun_out/r2_bench_n2_$st.json 2>&1
  BL_WARMUP_PIECES=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 --stage $st --no-e2e > gpurun_out/r2_bench_n2_${st}_nopieces.json 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench5.json 2>&1
