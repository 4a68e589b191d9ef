set -x
python tools/prof_euler.py 4 262144 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:euler_cart_own -s 1 -c 1 -o gpurun_out/euler_warp python tools/prof_euler.py 4 262144 3 > gpurun_out/ncu_warp.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_warp.log
