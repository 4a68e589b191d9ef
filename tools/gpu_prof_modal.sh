python tools/prof_modal.py 6 65536 > gpurun_out/pm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:euler_modal -s 1 -c 1 -o gpurun_out/modal_v1 python tools/prof_modal.py 6 65536 > gpurun_out/ncu_m1.log 2>&1
echo rc=$?
