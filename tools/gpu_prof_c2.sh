python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/c2p.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hadamard_rowsum -s 3 -c 1 -o gpurun_out/had_v2 python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_h2.log 2>&1
echo rc=$?
