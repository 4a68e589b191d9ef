"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line (the C oracle on the host cores) and the algorithmic work counts."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_algorithmic_counts():
    # n = 4: 288 unique pairs, 5120 bytes per element
    assert 3 * 4**3 * 3 // 2 == 288
    assert bench.euler_bytes_per_element(4) == 5120
    assert bench.euler_flops_per_element(4) == 288 * 73 + 192 * 18 + 64 * 16
    assert bench.modal_bytes_per_element(6) == 19 * 216 * 8 + 8


def test_reference_arm_line_on_cpu():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
         "--warmup", "1", "--elements", "3000"],
        capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the reference arm never maps the product library (oracle/workload.py)
    assert not any("libsumfac_b200" in x for x in line["native_libraries_mapped"])


@pytest.mark.parametrize("config,extra", [(2, ["--elements", "2000"]),
                                          (5, ["--cpu-sample-c5", "16"])])
def test_reference_arm_other_configs(config, extra):
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0", "--config", str(config), *extra],
        capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["impl"] == "reference"
    assert line["unit"] == ("element-DOF/s" if config == 5 else "entries/s")
    assert not any("libsumfac_b200" in x for x in line["native_libraries_mapped"])


def test_cpu_dense_vs_sumfac_slopes():
    cd = bench.cpu_dense_vs_sumfac(2, budget_s=0.05, ns=(3, 7))
    # dense per DOF grows ~n^3, sum-factorized ~n: between n = 3 and 7 the dense
    # route's disadvantage grows ~(7/3)^2 ~ 5x (2x leaves room for timing noise)
    r = cd["dense_over_sumfac"]
    assert r[7] > 2.0 * r[3] and r[3] > 1.0


def test_dense_oracle_equals_sum_factorized_oracle():
    from oracle import c_oracle, euler_oracle, workload

    syn = workload.synth()
    for n in (2, 3, 4, 5):
        U = syn.euler_states(3, n, seed=4)
        D = workload.gll_operators(n)[1]
        a = c_oracle.euler_volume_cartesian(U, D)
        b = c_oracle.euler_volume_dense(U, D)
        assert euler_oracle.max_rel(b, a) <= 1e-14


def test_gate_sample_and_failure():
    idx = bench.gate_sample(1000)
    assert idx[0] == 0 and idx[-1] == 999 and len(idx) <= 64 and np.all(np.diff(idx) > 0)
    assert list(bench.gate_sample(5)) == [0, 1, 2, 3, 4]
    with pytest.raises(bench.CorrectnessGateError):
        bench._gate_result("x", idx, 1e-9, 1e-12)
    assert bench._gate_result("x", idx, 1e-15, 1e-12)["passed"]


def test_reference_arm_non_zero_ranks_exit_quietly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--elements", "100"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0 and out.stdout.strip() == ""
