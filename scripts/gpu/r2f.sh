# HEAD check (re-entry 5): GPU suite, driver-style bench, launch list, ncu --set full of K1 mixed on cfg3
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gpu_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
timeout 300 python scripts/profile_k1.py --cfg 3 --pairs 100000 --runs 3 --phases > gpurun_out/r2f_cfg3.log 2>&1
TAG=r2f bash scripts/gpu/ncu_k1.sh
TAG=r2f bash scripts/gpu/ncu_configs.sh
tail -n 3 gpurun_out/r2f_gpu_pytest.log gpurun_out/r2f_cfg3.log
