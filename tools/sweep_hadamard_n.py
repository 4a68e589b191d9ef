import json, os, sys, subprocess
for lib in sorted(os.listdir("build/variants")):
    env = dict(os.environ, SFB_LIB="build/variants/" + lib)
    out = subprocess.run([sys.executable, "bench.py", "--config", "2", "--steps", "5", "--warmup", "3"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(lib, [(p["n"], round(p["ms_per_step"], 3), round(p["hbm_frac"], 2)) for p in d["n_sweep"]["points"]], round(d["n_sweep"]["slope_time_per_element_vs_n"], 2))
    except Exception as e:
        print(lib, "failed", out.stderr[-500:])
