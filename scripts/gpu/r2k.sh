# HEAD after the pipelined one-shot path: driver-style bench, reference arm, launch list, ncu --set full of K1 mixed, per-config ncu metrics
set -x
timeout 900 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2k_bench_reference.json 2> gpurun_out/r2k_bench_reference.err; echo "ref rc=$?"
timeout 300 python scripts/profile_k1.py --cfg 3 --pairs 100000 --runs 3 --phases > gpurun_out/r2k_cfg3.log 2>&1
TAG=r2k bash scripts/gpu/launches.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches_e2e.csv python scripts/mini_call.py 100000 3 0 > gpurun_out/r2k_launches_e2e.log 2>&1
TAG=r2k bash scripts/gpu/ncu_k1.sh
TAG=r2k bash scripts/gpu/ncu_configs.sh
