mkdir -p gpurun_out
for rep in 1 2 3; do for lib in "" variants/l2h1.so; do
  TAT_LIB=$lib python tools/time_stages.py C3 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep81.txt
done; done
