#!/bin/bash
# Round-end evidence on one GPU (run from the repo root on the GPU box): parity tests, the default
# bench line, the ncu launch list of the same bench command, one ncu --set full of every C3
# kernel, and one of the dense-mode tcgen05 GEMMs.  usage: bash tools/profile_round.sh <tag>
tag=${1:-rX}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest_exit=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_C3.log 2>&1
echo "bench_exit=$?" >> gpurun_out/${tag}_bench_C3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-loop \
  > gpurun_out/${tag}_launches_ncu.log 2>&1
echo "ncu_exit=$?" >> gpurun_out/${tag}_launches_ncu.log
bash tools/ncu_full.sh ${tag} "^(k|void k|tat)" 11
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k5dt?_tc" -c 2 \
  -o gpurun_out/${tag}_dense python tools/time_dense.py > gpurun_out/${tag}_dense_ncu.log 2>&1
echo "ncu_exit=$?" >> gpurun_out/${tag}_dense_ncu.log
