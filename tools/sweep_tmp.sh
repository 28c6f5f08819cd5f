mkdir -p gpurun_out
TAT_LIB=variants/red128.so timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or small or adjoint_identity or determinism" > gpurun_out/sweep85_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep85_pytest.log
for rep in 1 2; do for lib in "" variants/red128.so; do for c in C3 C4 C5; do
  TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep85.txt
done; done; done
