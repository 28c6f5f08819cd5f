#!/bin/bash
# Round-2 GPU round trip: all GPU tests (no -x), the default bench line, the FP32 ubench.
# usage (repo root, GPU box): bash tools/r2_check.sh <tag> [pytest-args...]
tag=${1:-chk}; shift
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_fp32 tools/ubench_fp32.cu && /tmp/ubench_fp32 > gpurun_out/${tag}_ubench_fp32.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q "$@" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest_exit=$?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo "bench_exit=$?" >> gpurun_out/${tag}_bench.log
