# quick GPU check: parity suites (digests + golden) and the cfg3 K1 time
set -x
timeout 420 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
python scripts/profile_k1.py --cfg 3 --pairs 100000 --runs 3 --phases > gpurun_out/${TAG}_cfg3.log 2>&1
python scripts/profile_k1.py --cfg 3 --pairs 400000 --runs 2 > gpurun_out/${TAG}_cfg3_400k.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_cfg3.log gpurun_out/${TAG}_cfg3_400k.log
