mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "inverse" > gpurun_out/sweep66_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep66_pytest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/inv_prof.py > gpurun_out/inv_launch2.csv 2>/dev/null
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/sweep66_bench.log 2>&1
