# ncu --set full of the n = 6 config-4 kernel (barrier-synchronised CTA kernel)
python tools/prof_euler.py 6 77672 3 > gpurun_out/p6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:euler_cart_sync -s 1 -c 1 -o gpurun_out/euler_sync_n6 python tools/prof_euler.py 6 77672 3 > gpurun_out/ncu_n6.log 2>&1
echo ncu_rc=$?
