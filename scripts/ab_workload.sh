# A/B library builds on a workload: bash scripts/ab_workload.sh <workload> name1 name2 ...
wl=$1; shift
for rep in 1 2; do for v in "$@"; do
  BL_LIB_PATH=$PWD/scripts/ab/libbitlamb_$v.so timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl', '$v', round(d['ms_per_step'],4), {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()})"
done; done
