# all bench modes on one GPU (each prints one JSON line)
for c in 3 2 5 4; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"
  tail -2 gpurun_out/bench_c$c.err
done
