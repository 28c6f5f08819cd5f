mkdir -p gpurun_out
for v in "TAT_K2S_IPC=4" "TAT_K2S_IPC=8" "TAT_K2S_IPC=16"; do
  for c in C3 C5 C4; do
    env $v python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|$v |" >> gpurun_out/sweep19.txt
  done
done
