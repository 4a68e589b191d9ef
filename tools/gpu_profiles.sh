# Round profile artefacts, part 1: bench line + launch list of the same command.
# (part 2, the full ncu capture of the top kernel, is tools/gpu_prof.sh: one ncu per call)
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
echo done
