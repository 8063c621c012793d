# Warmup overlap at N=4: exchange unroll (LOSSLESS_U) x CTA shape.
mkdir -p gpurun_out; out=gpurun_out/r2_warm_u4.txt; : > $out
run() {  # label lib env...
  label=$1; lib=$2; shift 2
  env BL_LIB_PATH=$PWD/$lib "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus 4 --steps 10 --warmup 3 --stage warmup --no-e2e > /tmp/b.json 2>&1
  echo "$label $(tail -1 /tmp/b.json)" >> $out
}
run u2_default paper_2104_06069_b200/libbitlamb_b200.so
run u4_b128 build/lib_u4.so
run u4_b256 build/lib_u4.so BL_LOSSLESS_BLOCK=256
run u1_b256 build/lib_u1.so BL_LOSSLESS_BLOCK=256
run u4_b64 build/lib_u4.so BL_LOSSLESS_BLOCK=64
run u4_b128_p16 build/lib_u4.so BL_WARMUP_PIECES=16
