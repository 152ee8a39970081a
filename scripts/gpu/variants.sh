# A/B of library variants built by scripts/build_variant.py: TAG, VARIANTS="a b c", ARGS (profile_k1 args)
set -x
if [ -n "$PYTEST" ]; then timeout 420 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_pytest.log; fi
for v in $VARIANTS; do
  lib=paper_2208_09985_b200/_lib/variants/$v.so; [ "$v" = default ] && lib=""
  for a in "${ARGS[@]:---cfg 3 --pairs 100000 --runs 3 --phases}"; do :; done
  SG_LIB_OVERRIDE=$lib timeout 150 python scripts/profile_k1.py ${ARGS:---cfg 3 --pairs 100000 --runs 3 --phases} > gpurun_out/${TAG}_$v.log 2>&1
  SG_LIB_OVERRIDE=$lib timeout 150 python scripts/profile_k1.py ${ARGS2:---cfg 3 --pairs 400000 --runs 2} >> gpurun_out/${TAG}_$v.log 2>&1
  echo "== $v"; cat gpurun_out/${TAG}_$v.log
done
