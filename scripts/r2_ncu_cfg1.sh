# ncu of the config-1 step (8M params, one GPU): launch list + full capture of every kernel of one step.
mkdir -p gpurun_out
CMD="python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
BL_GRAPH=0 $CMD > gpurun_out/r2_cfg1_plain.log 2>&1 && \
BL_GRAPH=0 ncu --set full --clock-control none --import-source on -s 60 -c 8 -o gpurun_out/r2_prof_cfg1 $CMD > gpurun_out/r2_ncu_cfg1.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_cfg1.log
