# A/B the BERT-L step under environment settings (one bench run each).
# usage: bash scripts/env_sweep.sh [workers] [ENV=v,ENV2=w ...]   (X=1 = defaults)
# BL_LIB_PATH=<other .so> times another build of the library.
w=${1:-1}; shift
V=${@:-"X=1"}
for e in $V; do
  env $(echo $e | tr ',' ' ') python bench.py --sim-workers $w --no-cpu-baseline --no-e2e 2>/tmp/err.log | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', $w, round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/err.log
done
