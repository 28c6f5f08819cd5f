mkdir -p gpurun_out
TAT_LIB=variants/stg.so timeout 600 python -m pytest tests -m gpu -q -x -k "full_size" > gpurun_out/sweep34_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep34_pytest.log
for lib in "" variants/stg.so; do for c in C3 C5 C4; do
  TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep34.txt
done; done
