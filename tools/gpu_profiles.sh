# Round profile artefacts: bench line, launch list of the same command, full ncu of the top kernel.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/prof_euler.py 4 262144 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:euler_cart -s 1 -c 1 -o gpurun_out/euler_full python tools/prof_euler.py 4 262144 3 > gpurun_out/ncu_full.log 2>&1
echo done
