# ncu source-level capture of k1_bulk (sim n=4: odd chunk length -> bulk path), GPU 0.
mkdir -p gpurun_out
CMD="python bench.py --workload bert-large --sim-workers 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r2_bulk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_bulk -s 1 -c 1 -o gpurun_out/r2_prof_bulk $CMD > gpurun_out/r2_ncu_bulk.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_bulk.log
