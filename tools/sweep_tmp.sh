mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "full_size or small or other_grids or inverse or lowk or mixed" > gpurun_out/sweep20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep20_pytest.log
for c in C3 C5 C4; do
  python tools/time_stages.py $c 20 2>&1 | tail -1 >> gpurun_out/sweep20.txt
done
