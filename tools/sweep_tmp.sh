mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "fused or full_batch or full_size" > gpurun_out/sweep33_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep33_pytest.log
for lib in "" variants/s2.so variants/s4.so; do for c in C3 C5 C4; do
  TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep33.txt
done; done
