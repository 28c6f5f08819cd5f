mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/sweep78_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep78_pytest.log
for rep in 1 2; do for c in C3 C4 C5; do python tools/time_stages.py $c 20 2>&1 | tail -1 >> gpurun_out/sweep78.txt; done; done
python bench.py --steps 20 --warmup 5 --no-cpu --no-loop --no-extras 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'])" >> gpurun_out/sweep78.txt
