mkdir -p gpurun_out
run() { n=$1; tag=$2; shift 2; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 20 --warmup 3 --no-e2e > gpurun_out/sw_$tag.log 2>&1; python - "$tag" <<'P'
import json,sys
t=sys.argv[1]
for l in open(f"gpurun_out/sw_{t}.log"):
    if l.startswith("{"):
        d=json.loads(l); print(t, round(d["value"],4), {k:round(v["ms_per_launch"],4) for k,v in d["kernels"].items() if k.startswith("k1")})
P
}
run 4 n4_default X=1
run 4 n4_r8 BL_K1_BULK_R=8
run 4 n4_none BL_K1_BULK=none
run 4 n4_default2 X=1
run 2 n2_default X=1
run 2 n2_all BL_K1_BULK=all
run 2 n2_default2 X=1
