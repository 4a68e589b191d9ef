# round-2 measurement check: GPU tests, default bench line (gates, cpu baselines,
# e2e legs), the reference arm, and a functional 2-rank (gloo, one GPU) run of the
# multi-rank default line with its config-5 sharded object
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_default.json 2> gpurun_out/r2_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"
SFB_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2_tr2.json 2> gpurun_out/r2_tr2.err; echo "tr2 rc=$?"
tail -3 gpurun_out/r2_default.err gpurun_out/r2_tr2.err
