mkdir -p gpurun_out
for v in "TAT_STRIP_ADJ=16" "TAT_STRIP_ADJ=15" "TAT_STRIP_ADJ=12" "TAT_STRIP_ADJ=10" "TAT_STRIP_ADJ=8" "TAT_STRIP_FWD=15" "TAT_STRIP_FWD=14" "TAT_STRIP_FWD=18"; do for c in C3 C4; do
  env $v python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|$v |" >> gpurun_out/sweep28.txt
done; done
