# A/B library builds (scripts/ab/libbitlamb_<name>.so) on the BERT-L step.
# usage: bash scripts/ab_sweep.sh <workers> name1 name2 ...
w=$1; shift
for rep in 1 2; do for v in "$@"; do
  BL_LIB_PATH=$PWD/scripts/ab/libbitlamb_$v.so timeout 300 bash scripts/env_sweep.sh $w LIB=$v
done; done
