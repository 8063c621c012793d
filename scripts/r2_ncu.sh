# Round-2 ncu evidence (one GPU): launch list + one --set full capture of the final kernels.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r2_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_worker|k3_server|k5_update|k6_update|kw1_warmup|kw2_warmup" -c 8 -o gpurun_out/r2_prof $CMD > gpurun_out/r2_ncu_full.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_full.log
