# Round evidence in one call: GPU tests, smoke, the default bench line (config 3 +
# configs 2/4/5 summaries with gates, CPU baselines, e2e legs), the reference arm,
# the launch list of the default bench command, and a 2-rank functional run of the
# multi-rank line (gloo: both ranks on the one GPU; functional only).
set -x
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/round_bench.json 2> gpurun_out/round_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/round_ref.json 2> gpurun_out/round_ref.err; echo "ref rc=$?"
python tools/pcie_bw.py > gpurun_out/round_pcie.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/round_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/round_ncu_launch.log 2>&1
echo "launch list rc=$?"
SFB_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/round_tr2.json 2> gpurun_out/round_tr2.err
echo "tr2 rc=$?"
