"""bench.py's own code paths on the GPU at small sizes: the driver contract keys,
the correctness gate, the CPU baseline and the e2e legs of configs 2, 3 and 5."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def run_bench(*args):
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--cpu-seconds", "0.2", "--cpu-seconds-extra", "0.2",
                          *args], capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_config3_line_small():
    line = run_bench("--elements", "4096", "--no-extras", "--cpu-sample", "512")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "gpu_launches", "clocks", "roofline", "cpu_baseline", "e2e", "gate"):
        assert key in line, key
    assert line["gate"]["passed"] and line["gate"]["max_rel"] <= 1e-12
    assert line["gpu_launches"] == 3
    assert line["e2e"]["h2d_bytes_per_step"] == 4096 * 5 * 64 * 8
    assert line["cpu_baseline"]["kind"] == "port"


def test_config2_and_config5_lines_small():
    c2 = run_bench("--config", "2", "--elements", "2048")
    assert c2["gate"]["bitwise"] and c2["e2e"]["d2h_bytes_per_step"] == 2048 * 64 * 8
    assert "n_sweep" in c2
    c5 = run_bench("--config", "5", "--elements", "8192", "--cpu-sample-c5", "32",
                   "--e2e-sample-c5", "256")
    assert c5["gate"]["passed"] and c5["scaling"] == "strong"
    assert c5["e2e"]["sample_elements"] == 256 and c5["cpu_baseline"]["value"] > 0
    assert c5["residual_norm"] > 0
