mkdir -p gpurun_out
TAT_LIB=variants/p0s3.so timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or small or other_grids" > gpurun_out/sweep56_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep56_pytest.log
for rep in 1 2; do for lib in "" variants/p0s3.so variants/p0s2.so variants/p1s3.so; do
  TAT_LIB=$lib python tools/time_stages.py C3 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep56.txt
done; done
for lib in "" variants/p0s3.so; do for c in C4 C5; do TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep56.txt; done; done
