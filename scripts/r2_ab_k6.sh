# A/B: K6 at 72 registers (3 CTAs/SM) vs 64 registers with spills (4 CTAs/SM); BERT-L and config 1.
mkdir -p gpurun_out; out=gpurun_out/r2_ab_k6.txt; : > $out
for lib in paper_2104_06069_b200/libbitlamb_b200.so build/lib_k6m4.so; do
  for w in bert-large config1; do
    echo "$lib $w $(BL_LIB_PATH=$PWD/$lib python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)" >> $out
  done
done
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r2_parity_partial.txt 2>&1
