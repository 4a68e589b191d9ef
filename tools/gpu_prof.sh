# One `ncu --set full` capture (with source) of a hot kernel, after a plain run of the
# same driver exited 0.  usage: bash tools/gpu_prof.sh {c2|c3|c4 N|c5 [E]} [tag]
# (one ncu per call: it replays the kernel ~40 times; never on a multi-rank command)
what=$1; shift
case $what in
  c3) drv="tools/prof_euler.py 4 262144 3"; k=euler_cart_own; tag=${1:-c3} ;;
  c4) n=$1; E=$(python -c "print(round(2**24/$n**3))"); drv="tools/prof_euler.py $n $E 3"; k=euler_cart; tag=${2:-c4_n$n} ;;
  c5) drv="tools/prof_modal.py 6 ${1:-2097152}"; k=euler_modal; tag=${2:-c5} ;;
  c2) drv="bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"; k=hadamard_rowsum; tag=${1:-c2} ;;
esac
python $drv > gpurun_out/prof_$tag.plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$tag \
    python $drv > gpurun_out/prof_$tag.ncu.log 2>&1
echo "ncu rc=$?"
