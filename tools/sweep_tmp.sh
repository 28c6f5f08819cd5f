mkdir -p gpurun_out
TAT_LIB=variants/sA.so timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or fused_adjoint or adjoint_identity" > gpurun_out/sweep67_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sweep67_pytest.log
for c in C3 C5 C4; do for lib in "" variants/sA.so variants/sB.so variants/sC.so variants/sD.so; do
  TAT_LIB=$lib python tools/time_stages.py $c 20 2>&1 | tail -1 | sed "s|^|lib=$lib |" >> gpurun_out/sweep67.txt
done; done
