# full-size config-5 ncu capture (one replayed launch) + the default bench line
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
python tools/prof_modal.py 6 2097152 > gpurun_out/pm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:euler_modal -s 1 -c 1 -o gpurun_out/modal_full python tools/prof_modal.py 6 2097152 > gpurun_out/ncu_mf.log 2>&1
echo ncu rc=$?
