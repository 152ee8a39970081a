# quick A/B of library variants on cfg3 (and optionally other configs): VARIANTS="a b", RUNS, CFGS="3:100000 2:1000000"
for rep in 1 2; do
for v in $VARIANTS; do
  lib=paper_2208_09985_b200/_lib/variants/$v.so; [ "$v" = default ] && lib=""
  for c in ${CFGS:-3:100000}; do
    cfg=${c%%:*}; pairs=${c##*:}
    echo "== $v cfg$cfg rep $rep: $(SG_LIB_OVERRIDE=$lib timeout 150 python scripts/profile_k1.py --cfg $cfg --pairs $pairs --runs ${RUNS:-4} 2>&1 | grep K1-K3 | awk '{print $7}' | sort -n | head -2 | tr '\n' ' ')"
  done
done
done
