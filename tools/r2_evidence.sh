#!/bin/bash
# Round evidence on one GPU (repo root, GPU box): all GPU tests, the default bench line, the ncu
# launch list of the same bench command, one ncu --set full of every C3 kernel (one launch each).
# usage: bash tools/r2_evidence.sh <tag>
tag=${1:-r2x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest_exit=$?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_C3.log 2>&1
echo "bench_exit=$?" >> gpurun_out/${tag}_bench_C3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-loop --no-extras \
  > gpurun_out/${tag}_launches_ncu.log 2>&1
echo "ncu_exit=$?" >> gpurun_out/${tag}_launches_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^(k|void k)" -c 11 \
  -o gpurun_out/${tag}_full python tools/time_stages.py C3 1 > gpurun_out/${tag}_full_ncu.log 2>&1
echo "ncu_exit=$?" >> gpurun_out/${tag}_full_ncu.log
