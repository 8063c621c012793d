# ncu source-level capture of K3 at sim n=4 (k3_server_reduce<4>), GPU 0.
mkdir -p gpurun_out
CMD="python bench.py --workload bert-large --sim-workers 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r2_k3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k3_server -s 2 -c 1 -o gpurun_out/r2_prof_k3 $CMD > gpurun_out/r2_ncu_k3.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu_k3.log
