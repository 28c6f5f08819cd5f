#!/bin/bash
# Quick GPU iteration: selected GPU tests, a bench line without the slow legs.
# usage (repo root, GPU box): bash tools/r2_quick.sh <tag> "<pytest -k expr>"
tag=${1:-q}; k=${2:-parity}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "$k" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest_exit=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --no-cpu --no-loop --no-extras --steps 20 --warmup 5 > gpurun_out/${tag}_bench.log 2>&1
echo "bench_exit=$?" >> gpurun_out/${tag}_bench.log
