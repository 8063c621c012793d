# e2e (host gradients through the C-ABI) with and without the H2D/K1 overlap.
for rep in 1 2; do for e in BL_OVERLAP_H2D=0 X=1; do
  env $e python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))"
done; done
