#!/bin/bash
# ncu --set full of selected kernels at C3 (one launch each), after a plain run exits 0.
# usage: bash tools/ncu_full.sh <tag> <kernel-regex> [count]
tag=$1; kre=$2; cnt=${3:-2}
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/${tag}_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${kre}" -c ${cnt} \
  -o gpurun_out/${tag} python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu_exit=$?" >> gpurun_out/${tag}_ncu.log
