# quick correctness + timing loop: euler tests, then the default bench
timeout 600 python -m pytest tests/test_gpu_euler.py -x -q 2>&1 | tail -3
python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'fp64', d['roofline_fp64']['frac'], d['clocks'])"
