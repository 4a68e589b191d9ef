SFB_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --no-extras > gpurun_out/tr2.json 2> gpurun_out/tr2.err; echo "torchrun2 rc=$?"
SFB_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --config 5 --gpus 2 --steps 3 --warmup 3 > gpurun_out/tr2c5.json 2> gpurun_out/tr2c5.err; echo "torchrun2 c5 rc=$?"
# (NCCL refuses two ranks on one GPU: gloo for this functional check only)
