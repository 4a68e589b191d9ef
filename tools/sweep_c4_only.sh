for lib in build/variants/*.so build/variants/*.so; do
  SFB_LIB=$lib python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw4.json 2>gpurun_out/sw4.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sw4.json')); print(sys.argv[1], ' '.join('n%d:%.3f'%(p['n'],p['ms_per_step']) for p in d['sweep']))" $lib || tail -3 gpurun_out/sw4.err
done
