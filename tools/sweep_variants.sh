# time every prebuilt variant library in build/variants with bench.py $BENCH_ARGS
for lib in build/variants/*.so; do
  SFB_LIB=$lib python bench.py --steps ${STEPS:-30} --warmup 3 --no-e2e --no-cpu-baseline --no-extras $BENCH_ARGS > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sw.json')); print(sys.argv[1], round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" $lib || tail -3 gpurun_out/sw.err
done
