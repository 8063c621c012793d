# Warmup-stage overlap sweep at N=2 (bench.py --stage warmup): lossless pieces x CTAs/SM.
mkdir -p gpurun_out
out=gpurun_out/r2_warm_sweep.txt; : > $out
run() {  # env... label
  label=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus 2 --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
  echo "$label $(tail -1 /tmp/b.json)" >> $out
}
run base BL_WARMUP_PIECES=0
run p16c1 BL_WARMUP_PIECES=16 BL_LOSSLESS_CTAS_PER_SM=1
run p16c2 BL_WARMUP_PIECES=16 BL_LOSSLESS_CTAS_PER_SM=2
run p16c4 BL_WARMUP_PIECES=16 BL_LOSSLESS_CTAS_PER_SM=4
run p16c8 BL_WARMUP_PIECES=16 BL_LOSSLESS_CTAS_PER_SM=8
run p4c2 BL_WARMUP_PIECES=4 BL_LOSSLESS_CTAS_PER_SM=2
run p16c2_alone BL_WARMUP_PIECES=16 BL_LOSSLESS_CTAS_PER_SM=2 BL_WARMUP_NO_CONSUMERS=1
run p16c8_alone BL_WARMUP_PIECES=16 BL_LOSSLESS_CTAS_PER_SM=8 BL_WARMUP_NO_CONSUMERS=1
run p1c8_alone BL_WARMUP_PIECES=1 BL_LOSSLESS_CTAS_PER_SM=8 BL_WARMUP_NO_CONSUMERS=1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench6.json 2>&1
