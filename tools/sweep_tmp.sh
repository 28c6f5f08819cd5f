mkdir -p gpurun_out
for rep in 1 2; do for lib in "" variants/head.so; do
  TAT_LIB=$lib python bench.py --steps 20 --warmup 5 --no-cpu --no-loop --no-extras 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('lib=$lib', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])" >> gpurun_out/sweep77.txt
done; done
