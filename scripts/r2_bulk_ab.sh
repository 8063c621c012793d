# k1_bulk producer change: parity (sim n=4 paths) + sim-4 BERT-L timing + N=4 step.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider > gpurun_out/r2_bulk_tests.txt 2>&1
python bench.py --workload bert-large --sim-workers 4 --no-cpu-baseline --no-e2e > gpurun_out/r2_bulk_sim4.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29664 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2_bulk_n4.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29665 tests/multigpu_check.py p2p > gpurun_out/r2_bulk_multi4.txt 2>&1; echo rc=$? >> gpurun_out/r2_bulk_multi4.txt
