mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/sweep70_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep70_pytest.log
for c in C1 C2; do python tools/time_stages.py $c 50 2>&1 | tail -1 >> gpurun_out/sweep70.txt; done
for s in 16 8 4; do TAT_STRIP_FWD=$s TAT_STRIP_ADJ=$s python tools/time_stages.py C1 50 2>&1 | tail -1 | sed "s|^|strip=$s |" >> gpurun_out/sweep70.txt; done
