# time every prebuilt variant library in build/variants with the default bench
for lib in build/variants/*.so; do
  SFB_LIB=$lib python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/sw.json')); print(sys.argv[1], round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" $lib
done
