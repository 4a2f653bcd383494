# A/B the top-k variants: tools/ab_topk.sh v0 v2 v3 ...
for v in "$@"; do
  if [ "$v" = "main" ]; then unset BINSKETCH_LIB_VARIANT; else export BINSKETCH_LIB_VARIANT=$PWD/variants/libbinsketch_$v.so; fi
  echo "== $v"; timeout 300 python tools/tc_prof.py 50000 1 2>&1 | tail -3; timeout 300 python tools/tc_prof.py 50000 4 2>&1 | tail -3
done
