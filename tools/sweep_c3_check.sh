# every build/variants/*.so: Euler GPU parity tests + config-3 timing (twice for the base)
for lib in build/variants/*.so build/variants/a_base.so; do
  t=$(SFB_LIB=$lib timeout 600 python -m pytest tests/test_gpu_euler.py -x -q 2>&1 | tail -1)
  SFB_LIB=$lib python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/s3.json 2>gpurun_out/s3.err
  echo "$lib | $t | $(python -c "import json; a=json.load(open('gpurun_out/s3.json')); print('c3 %.4f ms' % a['ms_per_step'])" 2>&1)"
done
