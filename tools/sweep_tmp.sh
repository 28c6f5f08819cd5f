mkdir -p gpurun_out
for lib in variants/k4a.so variants/k4c.so variants/k4d.so; do
  for c in C3 C5 C4; do
    TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep11.txt
  done
done
TAT_LIB=variants/k4c.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size or small or other_grids or inverse" >> gpurun_out/sweep11.txt 2>&1
