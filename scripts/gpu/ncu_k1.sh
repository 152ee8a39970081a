# one ncu --set full capture of K1 (mixed) on cfg3 100k pairs: TAG, CFG (default 3), PAIRS, KREGEX
CFG=${CFG:-3}; PAIRS=${PAIRS:-100000}; KREGEX=${KREGEX:-k1_mixed}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 \
    -o gpurun_out/${TAG}_k1 python scripts/profile_k1.py --cfg $CFG --pairs $PAIRS --runs 2 ${EXTRA} \
    > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
