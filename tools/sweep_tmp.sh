mkdir -p gpurun_out
TAT_LIB=variants/g4.so timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or small or driver" > gpurun_out/sweep83_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep83_pytest.log
for rep in 1 2; do for lib in "" variants/g2.so variants/g4.so; do for c in C3 C5; do
  TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep83.txt
done; done; done
