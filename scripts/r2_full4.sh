# Round-2 confirmation on a 4-GPU box: GPU suite (incl. world 2/4 multi-GPU), bench arms.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputests_4gpu.txt 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_full.json 2>&1
