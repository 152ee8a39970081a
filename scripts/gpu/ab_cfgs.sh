# A/B of library variants over several configs: VARIANTS="a b", RUNS; prints the two best K1 times per (variant, config)
for v in $VARIANTS; do
  lib=paper_2208_09985_b200/_lib/variants/$v.so; [ "$v" = default ] && lib=""
  for spec in "2 1000000 64 24" "1 10000 64 24" "4 20000 32 12" "4 20000 64 24" "3 100000 64 24"; do
    set -- $spec
    echo "== $v cfg$1 W$3 O$4: $(SG_LIB_OVERRIDE=$lib timeout 150 python scripts/profile_k1.py --cfg $1 --pairs $2 --W $3 --O $4 --runs ${RUNS:-4} 2>&1 | grep K1-K3 | awk '{print $7}' | sort -n | head -2 | tr '\n' ' ')"
  done
done
