# A/B of the k1_bulk producer change at N=4 and N=2 (same box, alternating).
mkdir -p gpurun_out; out=gpurun_out/r2_bulk_ab2.txt; : > $out
for rep in 1 2; do
for lib in build/lib_oldbulk.so paper_2104_06069_b200/libbitlamb_b200.so; do
  for n in 4 2; do
    echo "$lib n=$n $(BL_LIB_PATH=$PWD/$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2969$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1)" >> $out
  done
done
done
