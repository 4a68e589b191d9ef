# every build/variants/*.so: Euler GPU parity tests + config-4 sweep (base twice)
for lib in build/variants/*.so build/variants/*.so; do
  t=$(SFB_LIB=$lib timeout 600 python -m pytest tests/test_gpu_euler.py -x -q 2>&1 | tail -1)
  SFB_LIB=$lib python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw4.json 2>gpurun_out/sw4.err
  echo "$lib | $t | $(python -c "import json,sys; d=json.load(open('gpurun_out/sw4.json')); print(' '.join('n%d:%.3f'%(p['n'],p['ms_per_step']) for p in d['sweep']))" 2>&1)"
done
