# Warmup-stage overlap sweep at N=2 with the final kernels.
mkdir -p gpurun_out
out=gpurun_out/r2_warm_sweep2c.txt; : > $out
run() {  # label env...
  label=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus 2 --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
  echo "$label $(tail -1 /tmp/b.json)" >> $out
}
run base BL_WARMUP_PIECES=0
run p4c2b256e2 BL_WARMUP_PIECES=4 BL_LOSSLESS_CTAS_PER_SM=2 BL_LOSSLESS_BLOCK=256 BL_WARMUP_W2_EVERY=2
run p4c2b256e4 BL_WARMUP_PIECES=4 BL_LOSSLESS_CTAS_PER_SM=2 BL_LOSSLESS_BLOCK=256 BL_WARMUP_W2_EVERY=4
run p4c1b256e4 BL_WARMUP_PIECES=4 BL_LOSSLESS_CTAS_PER_SM=1 BL_LOSSLESS_BLOCK=256 BL_WARMUP_W2_EVERY=4
run p8c2b256e4 BL_WARMUP_PIECES=8 BL_LOSSLESS_CTAS_PER_SM=2 BL_LOSSLESS_BLOCK=256 BL_WARMUP_W2_EVERY=4
run p4c2b128e4 BL_WARMUP_PIECES=4 BL_LOSSLESS_CTAS_PER_SM=2 BL_LOSSLESS_BLOCK=128 BL_WARMUP_W2_EVERY=4
run p2c2b256e2 BL_WARMUP_PIECES=2 BL_LOSSLESS_CTAS_PER_SM=2 BL_LOSSLESS_BLOCK=256 BL_WARMUP_W2_EVERY=2
