# Compare tile-scheduling / K1 staging knobs on the BERT-L step (sim workers).
# usage: bash scripts/cmp_tiles.sh [workers...]
W=${@:-2 4}
for e in "X=1" "BL_STATIC_TILES=1" "BL_K1_BULK=none"; do for w in $W; do
  env $e python bench.py --sim-workers $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', $w, round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done; done
