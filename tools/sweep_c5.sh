# every build/variants/*.so: modal GPU parity tests and the config-5 timing (gated)
for lib in build/variants/*.so; do
  echo "== $lib $(SFB_LIB=$lib timeout 600 python -m pytest tests/test_gpu_modal.py -x -q 2>&1 | tail -1)"
  SFB_LIB=$lib python bench.py --config 5 --steps ${STEPS:-8} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s5.json 2>gpurun_out/s5.err
  python -c "import json; b=json.load(open('gpurun_out/s5.json')); print('c5 %.3f ms frac %.3f gate %.1e' % (b['ms_per_step'], b['roofline']['frac'], b['gate']['max_rel']))" || tail -3 gpurun_out/s5.err
done
