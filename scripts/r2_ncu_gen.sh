mkdir -p gpurun_out
CMD="python bench.py --workload config1 --sim-workers 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
BL_GRAPH=0 $CMD > gpurun_out/r2_gen_plain.log 2>&1 && \
BL_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:general -s 4 -c 2 -o gpurun_out/r2_prof_gen $CMD > gpurun_out/r2_ncu_gen.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_gen.log
