# BERT-L step at N = 1, 2, 4 (torchrun, one process per GPU) -> gpurun_out/scale_N*.json
# usage: bash scripts/scale_bench.sh "1 2 4" [extra bench.py args]
NS=${1:-"1 2 4"}; shift
mkdir -p gpurun_out
for n in $NS; do
  if [ "$n" = 1 ]; then
    python bench.py "$@" > gpurun_out/scale_N1.json 2> gpurun_out/scale_N1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n "$@" > gpurun_out/scale_N$n.json 2> gpurun_out/scale_N$n.err
  fi
  tail -1 gpurun_out/scale_N$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n', round(d['ms_per_step'],3), 'e2e', d.get('e2e') and round(d['e2e']['value'],2), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done
