# compute-sanitizer memcheck (one tool per call) over small GPU parity cases.
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
  -k "compressed_allreduce_bitexact and (1-6 or 2-5 or 3-10 or 4-4096 or 8-37) or optimizer_onebit_lamb_bitexact or other_variants or misaligned or identity_compressor_bitexact or weight_decay" \
  > gpurun_out/r2_memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_memcheck.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/r2_memcheck_boundary.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_memcheck_boundary.txt
