# traceback-batching / C4 variants of the full-frame K1: parity (default build), then cfg5 / cfg4 W128 / cfg2 per variant
set -x
timeout 600 python -m pytest tests/test_gpu_digests.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
tail -3 gpurun_out/r2e_pytest.log
for v in default old t8 t16 t16m8 t20m8; do
  lib=paper_2208_09985_b200/_lib/variants/$v.so; [ "$v" = default ] && lib=""
  SG_LIB_OVERRIDE=$lib timeout 200 python scripts/profile_k1.py --cfg 5 --pairs 500000 --runs 2 --phases > gpurun_out/r2e_cfg5_$v.log 2>&1
  SG_LIB_OVERRIDE=$lib timeout 200 python scripts/profile_k1.py --cfg 4 --pairs 20000 --W 128 --O 48 --runs 2 --phases > gpurun_out/r2e_cfg4w128_$v.log 2>&1
  SG_LIB_OVERRIDE=$lib timeout 200 python scripts/profile_k1.py --cfg 2 --pairs 1000000 --runs 3 > gpurun_out/r2e_cfg2_$v.log 2>&1
  SG_LIB_OVERRIDE=$lib timeout 200 python scripts/profile_k1.py --cfg 5 --pairs 500000 --runs 2 --kernel mixed > gpurun_out/r2e_cfg5mixed_$v.log 2>&1
  echo "== $v"; grep -h "K1-K3\|^full:\|lanes in DC" gpurun_out/r2e_cfg5_$v.log gpurun_out/r2e_cfg4w128_$v.log gpurun_out/r2e_cfg2_$v.log gpurun_out/r2e_cfg5mixed_$v.log
done
