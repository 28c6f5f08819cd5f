mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/sweep69_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep69_pytest.log
for c in C2 C3 C4 C5; do python tools/time_stages.py $c 20 2>&1 | tail -1 >> gpurun_out/sweep69.txt; done
