mkdir -p gpurun_out
for rep in 1 2; do
python tools/time_stages.py C3 20 2>&1 | tail -1 | sed "s|^|base |" >> gpurun_out/sweep54.txt
TAT_RING2=15 TAT_LIB=variants/k5m3.so python tools/time_stages.py C3 20 2>&1 | tail -1 | sed "s|^|k5m3 r15 |" >> gpurun_out/sweep54.txt
TAT_LIB=variants/k5m3.so python tools/time_stages.py C4 20 2>&1 | tail -1 | sed "s|^|k5m3 C4 |" >> gpurun_out/sweep54.txt
python tools/time_stages.py C4 20 2>&1 | tail -1 | sed "s|^|base C4 |" >> gpurun_out/sweep54.txt
done
