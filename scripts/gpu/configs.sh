# K1 time per config, auto vs forced mixed: TAG
for spec in "2 1000000 64 24" "1 10000 64 24" "5 500000 64 24" "4 20000 64 24" "4 20000 64 33" "4 20000 32 12" "4 20000 128 48"; do
  set -- $spec
  for k in auto mixed; do
    echo "== cfg$1 n=$2 W=$3 O=$4 kernel=$k"
    timeout 120 python scripts/profile_k1.py --cfg $1 --pairs $2 --W $3 --O $4 --runs 2 --kernel $k 2>&1 | grep -E "K1-K3|rror" | tail -1
  done
done
