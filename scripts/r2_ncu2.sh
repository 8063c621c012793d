# Round-2 ncu evidence, steady-state compression-stage kernels (GPU 0), plus the
# NVLink hardware counters of the fused multi-GPU kernels (torchrun, all GPUs).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r2_ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k1_worker_compress<2|k3_server_reduce|k5_update_a<1|k6_update_b" -c 6 \
    -o gpurun_out/r2_prof_ss $CMD > gpurun_out/r2_ncu_full2.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_full2.log
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port 29650 scripts/nvlink_counters.py > gpurun_out/r2_nvlink_n$NG.jsonl 2>&1
