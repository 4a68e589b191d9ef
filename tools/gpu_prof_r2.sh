# round 2: ncu --set full (with source) of the config-4 n = 5..8 kernels and the config-5 kernel
for n in 5 6 7 8; do
  E=$(python -c "print(round(2**24/$n**3))")
  python tools/prof_euler.py $n $E 3 > /dev/null 2>&1 || echo "plain run n=$n failed"
  ncu --set full --clock-control none --import-source on -k regex:euler_cart -s 1 -c 1 \
      -o gpurun_out/r2_c4_n$n python tools/prof_euler.py $n $E 3 > gpurun_out/r2_c4_n$n.log 2>&1
  echo "n=$n ncu rc=$?"
done
python tools/prof_modal.py 6 65536 > /dev/null 2>&1 || echo "plain modal failed"
ncu --set full --clock-control none --import-source on -k regex:euler_modal -s 1 -c 1 \
    -o gpurun_out/r2_c5_n6 python tools/prof_modal.py 6 65536 > gpurun_out/r2_c5.log 2>&1
echo "modal ncu rc=$?"
