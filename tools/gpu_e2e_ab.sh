# host-buffer entry A/B: chunk sizes (SFB_HOST_CHUNK_MB) on the default library
timeout 300 python -m pytest tests/test_gpu_euler.py -x -q -k "host" 2>&1 | tail -2
for cm in 8 16 32 64; do
  echo "chunk=$cm $(SFB_HOST_CHUNK_MB=$cm python tools/e2e_ab.py 2>&1 | tail -1)"
done
