#!/bin/bash
# One gpurun round trip: GPU parity tests, a short bench (no CPU leg), a per-kernel launch list.
# usage (from the repo root, on the GPU box): bash tools/gpu_check.sh [tag] [pytest-args...]
tag=${1:-chk}; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest_exit=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > gpurun_out/${tag}_bench.log 2>&1
echo "bench_exit=$?" >> gpurun_out/${tag}_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 22 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu \
  > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu_exit=$?" >> gpurun_out/${tag}_ncu.log
