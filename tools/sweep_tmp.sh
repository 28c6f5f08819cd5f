mkdir -p gpurun_out
for lib in "" variants/nostore.so; do for c in C3 C5; do
  TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep32.txt
done; done
