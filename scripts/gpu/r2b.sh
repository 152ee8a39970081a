set -x
python scripts/profile_k1.py --cfg 3 --pairs 100000 --runs 3 --phases > gpurun_out/r2b_cfg3.log 2>&1
python scripts/profile_k1.py --cfg 3 --pairs 400000 --runs 2 --phases > gpurun_out/r2b_cfg3_400k.log 2>&1
python scripts/profile_k1.py --cfg 5 --pairs 500000 --runs 2 --phases > gpurun_out/r2b_cfg5.log 2>&1
python scripts/profile_k1.py --cfg 5 --pairs 500000 --runs 2 --phases --kernel mixed > gpurun_out/r2b_cfg5_mixed.log 2>&1
python scripts/profile_k1.py --cfg 2 --pairs 1000000 --runs 2 --phases > gpurun_out/r2b_cfg2.log 2>&1
python scripts/profile_k1.py --cfg 4 --pairs 20000 --W 128 --O 48 --runs 2 --phases > gpurun_out/r2b_cfg4_128.log 2>&1
python scripts/profile_k1.py --cfg 4 --pairs 20000 --W 32 --O 12 --runs 2 --phases > gpurun_out/r2b_cfg4_32.log 2>&1
tail -n 8 gpurun_out/r2b_*.log
