mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/sweep55_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep55_pytest.log
for r in -1 0 15; do TAT_RING2=$r python tools/time_stages.py C5 20 2>&1 | tail -1 | sed "s|^|ring2=$r |" >> gpurun_out/sweep55.txt; done
