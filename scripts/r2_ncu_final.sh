# End-of-round ncu: launch list + full capture of the steady-state K1/K3/K5/K6 (BERT-Large, one GPU).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r2f_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv $CMD > gpurun_out/r2f_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_worker_compress|k3_server_reduce|k5_update_a|k6_update_b" -s 4 -c 4 \
    -o gpurun_out/r2f_prof $CMD > gpurun_out/r2f_full.log 2>&1
echo rc=$? >> gpurun_out/r2f_full.log
