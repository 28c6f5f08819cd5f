mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "driver or lowk or autograd or inverse" > gpurun_out/sweep64_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep64_pytest.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-extras > gpurun_out/sweep64_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/nnls_prof.py > gpurun_out/nnls_launch2.csv 2>/dev/null
