# Round-2 ncu: steady-state K1 (mode 2) and K5 (MPREV 1) of the BERT-Large step (GPU 0).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r2_ncu_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_worker_compress|k5_update_a" -s 2 -c 2 \
    -o gpurun_out/r2_prof_k1k5 $CMD > gpurun_out/r2_ncu_full3.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_full3.log
