# DFMA peak with the SM clocks sampled while it runs (nvidia-smi every 50 ms):
# the roofline denominator bench.py uses, with its clock record.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/peaks/fp64_peak.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw \
    --format=csv,noheader,nounits -lms 50 > /tmp/fp64_clocks.csv &
SMI=$!
sleep 0.5
for i in 1 2 3; do /tmp/fp64_peak; done
kill $SMI
python - <<'PY'
import statistics
rows = [l.strip().split(", ") for l in open("/tmp/fp64_clocks.csv") if l.strip()]
sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
print({"clock_samples": len(sm), "sm_mhz_median": statistics.median(sm), "sm_mhz_min": min(sm),
       "sm_max_mhz": max(float(r[1]) for r in rows), "reasons_active": sorted({r[2] for r in rows}),
       "power_w_max": max(pw)})
PY
