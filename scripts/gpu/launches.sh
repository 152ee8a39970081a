# per-launch kernel times (ncu, serialised, cold) of one profile_k1 run: TAG, ARGS
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_k1.py ${ARGS:---cfg 3 --pairs 100000 --runs 2} \
    > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?"
