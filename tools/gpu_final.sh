# round-end evidence in one call: GPU tests, smoke, default bench line, reference arm,
# config 2/4/5 lines, launch list of the default bench
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
for c in 2 4 5; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
