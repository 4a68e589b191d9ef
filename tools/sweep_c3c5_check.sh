# every build/variants/*.so: Euler + modal GPU parity tests, config-3 and config-5 timings
for lib in build/variants/*.so build/variants/a_base.so; do
  echo "== $lib $(SFB_LIB=$lib timeout 600 python -m pytest tests/test_gpu_euler.py tests/test_gpu_modal.py -x -q 2>&1 | tail -1)"
  SFB_LIB=$lib python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/s3.json 2>gpurun_out/s3.err
  SFB_LIB=$lib python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s5.json 2>gpurun_out/s5.err
  python -c "import json; a=json.load(open('gpurun_out/s3.json')); b=json.load(open('gpurun_out/s5.json')); print('c3 %.4f ms  c5 %.3f ms' % (a['ms_per_step'], b['ms_per_step']))" || tail -3 gpurun_out/s3.err gpurun_out/s5.err
done
