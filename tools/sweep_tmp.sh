mkdir -p gpurun_out
TAT_LIB=variants/u8sq.so timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or small or adjoint_identity or inverse" > gpurun_out/sweep60_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep60_pytest.log
for rep in 1 2; do for lib in "" variants/u8.so variants/sq.so variants/u8sq.so variants/u2.so; do
  TAT_LIB=$lib python tools/time_stages.py C3 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep60.txt
done; done
