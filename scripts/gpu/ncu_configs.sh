# ncu metrics of every K1 launch (mixed, tail, full frame, wide) per BASELINE config: TAG
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,sm__warps_active.avg.per_cycle_active,launch__registers_per_thread
for spec in "1 10000 64 24" "2 1000000 64 24" "3 100000 64 24" "4 20000 32 12" "4 20000 64 24" "4 20000 64 33" "4 20000 128 48" "5 500000 64 24"; do
  set -- $spec
  timeout 600 ncu --metrics $M --clock-control none -k regex:k1_ --csv \
     --log-file gpurun_out/${TAG}_ncu_cfg$1_W$3_O$4.csv \
     python scripts/profile_k1.py --cfg $1 --pairs $2 --W $3 --O $4 --runs 1 > /dev/null 2>&1
  echo "cfg$1 W$3 O$4 rc=$?"
done
