mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "fused or full_batch" > gpurun_out/sweep9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep9_pytest.log
for c in C3 C4 C5; do for v in "TAT_K2S_IPC=2" "TAT_K2S_IPC=4" "TAT_K2S_IPC=8"; do
  env TAT_VERBOSE=1 $v python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/sweep9.txt
done; done
