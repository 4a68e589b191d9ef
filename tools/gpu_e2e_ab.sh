timeout 300 python -m pytest tests/test_gpu_euler.py -x -q -k "host" 2>&1 | tail -2
for cm in 16 32 64; do for tp in 0 1; do
  echo "chunk=$cm taper=$tp $(SFB_HOST_CHUNK_MB=$cm SFB_HOST_TAPER=$tp python tools/e2e_ab.py 2>&1 | tail -1)"
done; done
for tp in 0 1; do echo "streams3 taper=$tp $(SFB_LIB=build/variants/s3.so SFB_HOST_TAPER=$tp python tools/e2e_ab.py 2>&1 | tail -1)"; done
echo "sync n6 tests"; timeout 300 python -m pytest tests/test_gpu_euler.py -x -q 2>&1 | tail -2
