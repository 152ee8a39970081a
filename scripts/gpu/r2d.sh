# cfg5 / cfg2 / cfg4 W128 phase counters and per-launch K1 times, both kernels
set -x
for k in auto mixed; do
  timeout 300 python scripts/profile_k1.py --cfg 5 --pairs 500000 --runs 2 --phases --kernel $k > gpurun_out/r2d_cfg5_$k.log 2>&1
done
timeout 300 python scripts/profile_k1.py --cfg 2 --pairs 1000000 --runs 2 --phases > gpurun_out/r2d_cfg2.log 2>&1
timeout 300 python scripts/profile_k1.py --cfg 4 --pairs 20000 --W 128 --O 48 --runs 2 --phases > gpurun_out/r2d_cfg4_128.log 2>&1
timeout 300 python scripts/profile_k1.py --cfg 4 --pairs 20000 --W 32 --O 12 --runs 2 --phases > gpurun_out/r2d_cfg4_32.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k1_ --csv \
   --log-file gpurun_out/r2d_ncu_cfg5_mixed.csv python scripts/profile_k1.py --cfg 5 --pairs 500000 --runs 1 --kernel mixed > /dev/null 2>&1
tail -n 12 gpurun_out/r2d_*.log
