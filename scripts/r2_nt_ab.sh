# A/B: small-collective K3 worker words specialised per n (NT) vs one n<=8 instantiation.
mkdir -p gpurun_out
N=${N:-2}
out=gpurun_out/r2_${TAG:-nt}_ab_n$N.txt; : > $out
for i in 1 2 3; do
  for v in new prev; do
    if [ $v = prev ]; then export BL_LIB_PATH=$PWD/build/${ALT:-lib_prev.so}; else unset BL_LIB_PATH; fi
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2961$i bench_sweep.py --sizes-mb ${SIZES:-1,2,4,8,16} --iters 50 > /tmp/s.txt 2>&1
    python - $v <<'PY' >> $out
import json, sys
for l in open('/tmp/s.txt'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], d['size_mb'], round(d['compressed_ms']*1e3, 1), round(d['nccl_fp32_ms']*1e3, 1))
PY
  done
done
