#!/usr/bin/env python
"""Benchmark of the B200 flux-differencing volume term (BASELINE.json metric).

Default workload (BASELINE config 3, the config the metric names): 3-D
compressible Euler, Chandrashekar two-point flux, GLL n = 4 (p = 3),
262,144 affine Cartesian elements, FP64, inputs seeded and generated on the
device.  One "step" = one pass of the fused volume-term kernel over the whole
element batch.  With N GPUs (torchrun) every rank owns its own 262,144
elements (distinct global element ids; weak scaling, no data-path
collective; timing is the max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3|2|4|5]

  --config 2   generic batched Hadamard + row sum + direction sum (n=4, 262,144 el.),
               plus the reference's sumfac-bench shape (n = 3..15) as "n_sweep"
  --config 4   config 3 swept over n = 2..8 with ~2^24 nodes each (one line, "sweep")
  --config 5   curvilinear modal Euler, n = 6, 2^21 elements sharded over the
               ranks (strong scaling) + the deterministic NCCL residual norm

Under torchrun (N > 1) the default line keeps config 3 as `value` (weak
scaling, comparable across N) and adds "config5_sharded": the north star's
sharded config at N ranks (2^21 elements split in whole norm blocks, NCCL
all_gather of the block partials, norm checked bitwise against the 1-rank
value, comm_nranks from a collective over the group).

Correctness gate (the reference's bench.py:134-164 _gate_point): before any
config is timed, sampled elements of the device result are compared with the
C oracle at max_rel <= 1e-12 (bitwise for config 2); a failure raises
CorrectnessGateError and the run exits non-zero without a line.

Rank 0 prints ONE JSON line.  Keys beyond the driver contract:
  element_dof_per_s     nodes / s (x5 for conserved DOF / s)
  roofline              dominant kernel vs measured HBM copy bandwidth
  roofline_fp64         same kernel's algorithmic FP64 rate vs measured DFMA peak
  cpu_baseline          the oracle's C port on the host cores (N=1, rank 0)
  e2e                   through the C-ABI host-buffer entry point (pinned
                        host buffers; H2D + kernel + D2H inside the timed region)
  gate                  the correctness gate's result for the timed config
  other_configs         configs 2, 4, 5 at N=1, each with gate, cpu_baseline
                        and e2e (config 4: CPU sum-factorized vs dense O(n^{2d})
                        per DOF)

The reference arm (--impl reference) never imports the product package: its
inputs come from oracle/workload.py (synth.py loaded by file path, operators
recorded from the reference itself) and it asserts that libsumfac_b200.so is
not mapped into the process before timing.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
DFMA_MEASURED_TFLOPS = 34.214  # tools/peaks/run_fp64_peak.sh, round 2, 1965 MHz (profiles/r02/)
METRIC = "FP64 Hadamard entries/s (3D Euler Chandrashekar flux differencing)"

# Algorithmic work per element: unique off-diagonal pairs
# x (C_pair flux + 20 accumulate) + diagonal entries x 18 + nodes x 16; bytes =
# 2 x 5 x n^3 x 8.  C_pair = 53 is the restated flux as written
# (oracle/euler_oracle.py chandrashekar + logmean) in SURVEY 8(d)'s convention
# (+, -, x, / = 1 flop), with the logarithms per node (2 per node, in NODE):
# two log means 2 x 6, vbar 6, rhobar 2, betabar 2, p_hat 2, v.n 5, F1 1,
# F_{1+m} 9, |v|^2 average 2, F5 12.  Cross-check, SASS of the config-3 kernel
# (ncu, FMA = 2 flops): ~56 flops per flux.  (Round 1 used 43, the kernel's own
# FP64 instruction count per flux with an FMA counted once.)
FLUX_FLOPS, ACC_FLOPS, DIAG_FLOPS, NODE_FLOPS = 53, 20, 18, 16
CURV_EXTRA_FLOPS = 6  # contravariant: the metric average n = (Ja_a + Ja_b) / 2, 3 x (add + mul)


def euler_flops_per_element(n):
    pairs = 3 * n * n * n * (n - 1) // 2
    return pairs * (FLUX_FLOPS + ACC_FLOPS) + 3 * n**3 * DIAG_FLOPS + n**3 * NODE_FLOPS


def euler_bytes_per_element(n):
    return 2 * 5 * n**3 * 8


def modal_flops_per_element(n):
    pairs = 3 * n * n * n * (n - 1) // 2
    transforms = 2 * 2 * 5 * 3 * n ** 4  # V^3 and Pi^3, FMA = 2
    return (transforms + pairs * (FLUX_FLOPS + CURV_EXTRA_FLOPS + ACC_FLOPS)
            + 3 * n**3 * DIAG_FLOPS + n**3 * NODE_FLOPS + 2 * 5 * n**3)


def modal_bytes_per_element(n):
    return (5 + 9 + 5) * n**3 * 8 + 8


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.samples = []
        self.proc = None
        self.dev = device_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        window = [s for t, s in self.samples if t0 - 0.15 <= t <= t1 + 0.15]
        if not window:
            window = [s for _, s in self.samples[-5:]]
        if not window:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in window if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in window if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in window for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(window)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_config(args, world):
    if args.config == 2:
        return {"workload": f"config2: batched generic Hadamard + row sum + direction sum, "
                            f"(D x I x I + I x D x I + I x I x D) o F, GLL n=4, {args.elements} "
                            f"elements per GPU",
                "n": 4, "elements_per_gpu": args.elements, "total_elements": args.elements * world,
                "l2": "inputs (%.0f MB) larger than the 126 MB L2" % (args.elements * 6144 / 1e6),
                "parallelism": f"element shards x{world}"}
    if args.config == 5:
        return {"workload": f"config5: curvilinear modal Euler (V^3 -> contravariant "
                            f"Chandrashekar flux differencing -> Pi^3), GLL n={args.n}, "
                            f"{args.elements} elements total, sharded, deterministic NCCL "
                            f"residual norm",
                "n": args.n, "total_elements": args.elements,
                "elements_per_gpu": args.elements // world, "gamma": 1.4, "vars": 5,
                "l2": "inputs (%.1f GB) larger than the 126 MB L2"
                      % (args.elements * modal_bytes_per_element(args.n) / 1e9),
                "parallelism": f"element shards x{world} (strong scaling)"}
    return {"workload": f"config3: 3-D Euler Chandrashekar volume term, GLL n={args.n} "
                        f"(p={args.n - 1}), {args.elements} Cartesian elements per GPU",
            "n": args.n, "elements_per_gpu": args.elements, "total_elements": args.elements * world,
            "gamma": 1.4, "vars": 5, "layout": "U[E][5][n^3] fp64 SoA",
            "l2": "inputs (%.0f MB) larger than the 126 MB L2" % (args.elements * 5 * args.n**3 * 8 / 1e6),
            "parallelism": f"element shards x{world}"}


# ---------------------------------------------------------------------------
# reference arm: the oracle's C port on the host cores (rank 0 only)
# ---------------------------------------------------------------------------
def assert_product_not_loaded(where):
    from oracle import workload

    libs = workload.loaded_native_libraries()
    bad = [x for x in libs if "libsumfac_b200" in x]
    if bad:
        raise RuntimeError(f"{where}: the product library is mapped into this process ({bad})")
    return libs


def cpu_dense_vs_sumfac(threads, budget_s=1.0, ns=range(2, 9)):
    """Config 4's CPU comparison: the C port of the sum-factorized route and of
    the dense O(n^{2d}) route (oracle.py:54-112 with the Chandrashekar operand:
    every entry of the n^d x n^d factor and flux matrices formed), per DOF, on
    fixed element samples (config-4 inputs, seed 4)."""
    from oracle import c_oracle, workload

    syn = workload.synth()
    pts = []
    for n in ns:
        D = workload.gll_operators(n)[1]
        row = {"n": n}
        # DOF per thread and call: ~50-100 ms of work, so thread start-up is noise
        for route, fn, dof in (("sumfac", c_oracle.euler_volume_cartesian, 1 << 16),
                               ("dense", c_oracle.euler_volume_dense, 1 << 12)):
            sample = threads * max(1, -(-dof // n**3))
            U = syn.euler_states(sample, n, seed=4)
            fn(U[:threads], D, threads=threads)
            t, reps = time.perf_counter(), 0
            while True:
                fn(U, D, threads=threads)
                reps += 1
                if time.perf_counter() - t > budget_s:
                    break
            sec = (time.perf_counter() - t) / reps
            row[f"{route}_ns_per_dof"] = sec * 1e9 / (sample * n**3)
            row[f"{route}_sample_elements"] = sample
        pts.append(row)
    ns_ = np.array([p["n"] for p in pts], dtype=float)
    out = {"points": pts, "threads": threads, "cpu": cpu_model()}
    hi = ns_ >= 5
    for route, exp in (("sumfac", "1 (O(n^{d+1}) per element)"), ("dense", "3 (O(n^{2d}))")):
        t = np.array([p[f"{route}_ns_per_dof"] for p in pts])
        out[f"{route}_slope_per_dof_vs_n"] = {
            "all_n": float(np.polyfit(np.log(ns_), np.log(t), 1)[0]), "expected": exp,
            "n5_to_8": float(np.polyfit(np.log(ns_[hi]), np.log(t[hi]), 1)[0])
            if hi.sum() >= 2 else None}
    out["dense_over_sumfac"] = {p["n"]: p["dense_ns_per_dof"] / p["sumfac_ns_per_dof"]
                                for p in pts}
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import c_oracle, workload

    syn = workload.synth()
    threads = os.cpu_count() or 1
    extra = {}
    unit = "entries/s"
    metric = METRIC
    if args.config == 2:
        n, E = 4, args.elements
        basis = workload.config2_basis(n)
        F = syn.uniform_array(E * 768, 2, -1.0, 1.0).reshape(E, 3, 64, 4)
        run = lambda: c_oracle.hadamard_rowsum_batched(basis, F, threads=threads)  # noqa: E731
        units = E * 768
        sample = f"full workload ({E} elements) per step"
        metric = "FP64 Hadamard entries/s (generic batched)"
    elif args.config == 5:
        n = args.n
        E = min(args.elements, args.cpu_sample_c5)
        nodes, D, V, Pi = workload.gll_operators(n)
        Uh = syn.modal_states(E, n, seed=5)
        Ja = syn.metric_cofactors(E, n, seed=6, nodes=nodes)
        run = lambda: c_oracle.euler_volume_curvilinear_modal(  # noqa: E731
            Uh, Ja, V, Pi, D, threads=threads)
        units = E * n**3
        unit = "element-DOF/s"
        metric = "FP64 element-DOF/s (3D curvilinear modal Euler flux differencing)"
        sample = (f"first {E} of the {args.elements} config-5 elements per step (per-DOF rate "
                  f"of the sample; the full job would take {args.elements / E:.0f}x longer)")
    else:
        n, E = args.n, args.elements
        D = workload.gll_operators(n)[1]
        U = syn.euler_states(E, n, seed=3)
        run = lambda: c_oracle.euler_volume_cartesian(U, D, threads=threads)  # noqa: E731
        units = E * 3 * n**4
        sample = f"full workload ({E} elements) per step"
        if args.config == 4:
            extra["cpu_dense_vs_sumfac"] = cpu_dense_vs_sumfac(threads)
    libs = assert_product_not_loaded("reference arm")
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        run()
        times.append(time.perf_counter() - t)
    sec = sum(times) / len(times)
    value = units / sec
    libs = assert_product_not_loaded("reference arm (after timing)")
    line = {
        "metric": metric,
        "impl": "reference",
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "port",
                         "sample": f"{sample}, C port of the oracle (oracle/euler_oracle.c), "
                                   f"{threads} threads on {cpu_model()}"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_libraries_mapped": libs,
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def timed_loop(step, steps, warmup, world, dist, stream, sampler):
    """W untimed steps, then K steps between barrier+sync pairs; per-step events."""
    import torch

    from paper_2306_11665_b200 import _lib

    for _ in range(max(warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    t0 = time.time()
    for a, b in ev:
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize()
    t1 = time.time()
    launches = _lib.launch_count() - launches0
    per = [a.elapsed_time(b) for a, b in ev]
    ms_total = ev[0][0].elapsed_time(ev[-1][1])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    return ms_total / steps, per, launches, (t0, t1)


GATE_RTOL = 1e-12  # north star's FP64 tolerance (the reference gate: bench.py:63-64, 1e-13)


class CorrectnessGateError(RuntimeError):
    """A sampled element of the device result disagrees with the oracle (bench.py:134-164)."""


def gate_sample(E, k=64, seed=0):
    """First, last and seeded-random element ids (sorted, unique), at most k."""
    if E <= k:
        return np.arange(E)
    rng = np.random.default_rng(seed)
    idx = np.concatenate([np.arange(4), np.arange(E - 4, E), rng.choice(E, k - 8, replace=False)])
    return np.unique(idx)


def _gate_result(what, idx, err, tol, bitwise=None):
    res = {"checked_elements": int(len(idx)), "max_rel": err, "tol": tol,
           "oracle": "C port of the oracle (oracle/euler_oracle.c)", "passed": err <= tol}
    if bitwise is not None:
        res["bitwise"] = bitwise
    if not res["passed"]:
        raise CorrectnessGateError(f"{what}: max_rel {err:.3e} > {tol:.0e} on sampled elements")
    return res


def gate_cartesian(U, R, n, threads):
    from oracle import c_oracle, euler_oracle, workload

    import torch

    idx = gate_sample(U.shape[0])
    ti = torch.from_numpy(idx).to(U.device)
    Us, Rs = U[ti].cpu().numpy(), R[ti].cpu().numpy()
    ref = c_oracle.euler_volume_cartesian(Us, workload.gll_operators(n)[1], threads=threads)
    return _gate_result(f"config 3/4 n={n}", idx, euler_oracle.max_rel(Rs, ref), GATE_RTOL)


def gate_hadamard(F, out, n, threads):
    from oracle import c_oracle, euler_oracle, workload

    import torch

    idx = gate_sample(F.shape[0])
    ti = torch.from_numpy(idx).to(F.device)
    ref = c_oracle.hadamard_rowsum_batched(workload.config2_basis(n), F[ti].cpu().numpy(),
                                           threads=threads)
    got = out[ti].cpu().numpy()
    return _gate_result("config 2", idx, euler_oracle.max_rel(got, ref), 1e-13,
                        bitwise=bool(np.array_equal(got, ref)))


def gate_modal(Uh, Ja, Rh, ss, n, threads):
    from oracle import c_oracle, euler_oracle, workload

    import torch

    idx = gate_sample(Uh.shape[0], k=32)
    ti = torch.from_numpy(idx).to(Uh.device)
    _, D, V, Pi = workload.gll_operators(n)
    ref, ref_ss = c_oracle.euler_volume_curvilinear_modal(Uh[ti].cpu().numpy(),
                                                          Ja[ti].cpu().numpy(), V, Pi, D,
                                                          threads=threads)
    err = max(euler_oracle.max_rel(Rh[ti].cpu().numpy(), ref),
              euler_oracle.max_rel(ss[ti].cpu().numpy(), ref_ss))
    return _gate_result("config 5", idx, err, GATE_RTOL)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2306_11665_b200 import euler as eu

    world, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        # SFB_DIST_BACKEND=gloo only for functional checks of the multi-rank
        # path on a one-GPU box (never for reported numbers)
        backend = os.environ.get("SFB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's init lines (communicator size, transport) on stderr: the
            # rank count stays observable outside the JSON line too
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)

    cpu = world == 1 and not args.no_cpu_baseline
    if args.config == 4:
        line = run_sweep(args, world, rank, dev, stream, sampler, dist, cpu=cpu)
    elif args.config == 5:
        line = run_modal(args, world, rank, dev, stream, sampler, dist, cpu=cpu,
                         e2e=world == 1 and not args.no_e2e)
    elif args.config == 2:
        line = run_hadamard(args, world, rank, dev, stream, sampler, dist, cpu=cpu,
                            e2e=world == 1 and not args.no_e2e)
    else:
        n, E = args.n, args.elements
        U = eu.generate_states(E, n, seed=3, e0=rank * E, device=dev)
        R = torch.empty_like(U)

        def step():
            eu.volume_cartesian(U, n, out=R)

        step()
        gate = gate_cartesian(U, R, n, os.cpu_count() or 1)
        ms_step, per, launches, (t0, t1) = timed_loop(step, args.steps, args.warmup, world, dist,
                                                      stream, sampler)
        line = finish_line(args, world, dev, dist, ms_step, per, launches, sampler, t0, t1,
                           units=E * 3 * n**4, unit="entries/s",
                           bytes_launch=euler_bytes_per_element(n) * E,
                           flops_launch=euler_flops_per_element(n) * E,
                           extra={"element_dof_per_s": None, "dof_per_element": n**3},
                           traffic=ncu_traffic(args, n, E))
        line["gate"] = gate
        line["element_dof_per_s"] = world * E * n**3 / (line["ms_per_step"] / 1e3)
        if not args.no_e2e:  # every rank its own host buffers; max over ranks
            line["e2e"] = measure_e2e(args, U, world, dist, dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = measure_cpu_baseline(args, U)
        del U, R
        torch.cuda.empty_cache()
        if world == 1 and not args.no_extras:
            line["other_configs"] = measure_other_configs(args, dev, stream, sampler, dist)
        elif world > 1 and not args.no_extras:
            line["config5_sharded"] = sharded_config5(args, world, rank, dev, stream, sampler,
                                                      dist)
            line["comm_nranks"] = line["config5_sharded"]["comm_nranks"]
    sampler.stop()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# residual norm of the default config 5 (n = 6, 2^21 elements, seeds 5/6),
# bitwise invariant in the rank count (shard.global_norm_tensor); measured on
# one B200 (profiles/r01/bench_config5.json, gpurun_out/tr2c5.json)
CONFIG5_NORM_1RANK = 0.0037271219456293993


def sharded_config5(args, world, rank, dev, stream, sampler, dist):
    """The north star's sharded config at this job's N ranks (strong scaling)."""
    import copy

    import torch

    a = copy.copy(args)
    a.config, a.n, a.elements, a.steps, a.warmup, a.traffic = 5, 6, 2**21, 5, 3, None
    ln = run_modal(a, world, rank, dev, stream, sampler, dist)
    ones = torch.ones(1, dtype=torch.float64, device=dev)
    dist.all_reduce(ones)
    out = {k: ln[k] for k in ("metric", "value", "unit", "ms_per_step", "scaling", "config",
                              "roofline", "residual_norm", "per_rank_kernel_ms", "gate")}
    out["comm_nranks"] = int(ones.item())
    out["comm_backend"] = dist.get_backend()
    out["norm_bitwise_equal_1rank"] = ln["residual_norm"] == CONFIG5_NORM_1RANK
    out["norm_1rank"] = CONFIG5_NORM_1RANK
    return out


def ncu_traffic(args, n, elements):
    """DRAM bytes per launch of the top kernel from an ncu --set full capture of the
    same kernel (profiles/ncu_traffic.json, per round), scaled to this launch's
    element count; None when no capture of this config and order n exists.
    --traffic overrides it."""
    if args.traffic is not None:
        return args.traffic
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f).get(f"config{args.config}")
    except (OSError, ValueError):
        return None
    if not isinstance(rec, dict) or rec.get("n") != n or not rec.get("elements"):
        return None
    return rec["bytes"] * elements / rec["elements"]


def finish_line(args, world, dev, dist, ms_step, per, launches, sampler, t0, t1, units, unit,
                bytes_launch, flops_launch, extra=None, metric=METRIC, traffic=None):
    import torch

    if world > 1:
        t = torch.tensor([ms_step], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    kernel_ms = float(np.mean(per))
    hbm_gbs, peak_kind = measured_peaks()
    achieved = bytes_launch / (kernel_ms / 1e3) / 1e9
    achieved_tf = flops_launch / (kernel_ms / 1e3) / 1e12
    line = {
        "metric": metric,
        "value": world * units / (ms_step / 1e3), "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if args.config == 5 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-hash inputs, device-generated)",
        "config": workload_config(args, world),
        "gpu_launches": launches,
        "clocks": sampler.summary(t0, t1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": achieved / hbm_gbs, "traffic": traffic,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "algorithmic_bytes_per_launch": bytes_launch, "kernel_ms": kernel_ms},
        "roofline_fp64": {"achieved": achieved_tf, "peak": DFMA_MEASURED_TFLOPS,
                          "unit": "TFLOP/s", "frac": achieved_tf / DFMA_MEASURED_TFLOPS,
                          "algorithmic_flops_per_launch": flops_launch,
                          "peak_source": "tools/peaks/fp64_peak.cu DFMA burst at 1965 MHz (profiles/r02/fp64_peak_with_clocks.txt)"},
    }
    if args.config == 5 or flops_launch / bytes_launch > DFMA_MEASURED_TFLOPS * 1e3 / hbm_gbs:
        # compute-bound by the algorithmic count: the FP64 roofline is the binding one
        line["roofline"], line["roofline_hbm"] = dict(line["roofline_fp64"], bound="fp64",
                                                      traffic=traffic,
                                                      kernel_ms=kernel_ms), line["roofline"]
        del line["roofline_fp64"]
    if line["roofline"]["frac"] > 1.0:
        # the denominator is MEASURED_PEAKS' copy rate (read + write); a
        # read-dominated stream (config 2: 1.61 GB read, 0.13 GB written) runs
        # above a copy, so the fraction is not comparable across configs
        line["roofline"]["note"] = ("frac > 1: read-dominated traffic against the measured "
                                    "copy (read+write) peak; not a bound violation")
    if extra:
        line.update({k: v for k, v in extra.items() if v is not None})
    return line


def run_hadamard(args, world, rank, dev, stream, sampler, dist, cpu=False, e2e=False):
    import torch

    import paper_2306_11665_b200 as sf
    from paper_2306_11665_b200 import euler as eu
    from paper_2306_11665_b200 import kernel

    n, d, E = 4, 3, args.elements
    D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
    pattern = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(pattern, D, np.ones(n))
    F = eu.generate_uniform(E * 768, 2, -1.0, 1.0, i0=rank * E * 768, device=dev).reshape(
        E, d, 64, n)
    out = torch.empty((E, 64), dtype=torch.float64, device=dev)
    B = basis.device

    def step():
        kernel.hadamard_rowsum_batched(B, F, out=out)

    step()
    gate = gate_hadamard(F, out, n, os.cpu_count() or 1)
    ms_step, per, launches, (t0, t1) = timed_loop(step, args.steps, args.warmup, world, dist,
                                                  stream, sampler)
    line = finish_line(args, world, dev, dist, ms_step, per, launches, sampler, t0, t1,
                       units=E * 768, unit="entries/s", bytes_launch=8 * (768 + 64) * E,
                       flops_launch=2 * 768 * E, metric="FP64 Hadamard entries/s (generic batched)",
                       traffic=ncu_traffic(args, n, E))
    line["gate"] = gate
    if cpu:
        line["cpu_baseline"] = cpu_baseline_hadamard(args, F)
    if e2e:
        line["e2e"] = e2e_hadamard(basis, F, out)
    del F, out
    torch.cuda.empty_cache()
    if world == 1:
        line["n_sweep"] = hadamard_n_sweep(dev, stream, sampler)
    return line


def cpu_baseline_hadamard(args, F):
    from oracle import c_oracle, workload

    threads = os.cpu_count() or 1
    basis = workload.config2_basis(4)
    sample = min(F.shape[0], 65536)
    Fs = F[:sample].cpu().numpy()
    c_oracle.hadamard_rowsum_batched(basis, Fs[:1024], threads=threads)
    t, reps = time.perf_counter(), 0
    while True:
        c_oracle.hadamard_rowsum_batched(basis, Fs, threads=threads)
        reps += 1
        if time.perf_counter() - t > args.cpu_seconds_extra:
            break
    sec = (time.perf_counter() - t) / reps
    return {"value": sample * 768 / sec, "unit": "entries/s", "cores": threads, "kind": "port",
            "sample": f"{sample} of the {F.shape[0]} config-2 elements x {reps} reps, C port of "
                      f"the reference pipeline (oracle/euler_oracle.c), {threads} threads on "
                      f"{cpu_model()}"}


def e2e_hadamard(basis, F_dev, out_dev, steps=5):
    """Config 2 through the host-buffer C-ABI entry (pinned F in, pinned sums out)."""
    import torch

    from paper_2306_11665_b200 import kernel

    E = F_dev.shape[0]
    Fh = torch.empty(tuple(F_dev.shape), dtype=torch.float64, pin_memory=True)
    Fh.copy_(F_dev.cpu())
    Oh = torch.empty((E, 64), dtype=torch.float64, pin_memory=True)
    kernel.hadamard_rowsum_batched_host(basis, Fh, out=Oh)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        kernel.hadamard_rowsum_batched_host(basis, Fh, out=Oh)
        times.append(time.perf_counter() - t)
    sec = float(np.mean(times))
    assert torch.equal(Oh, out_dev.cpu()), "config-2 e2e result differs from the device path"
    return {"value": E * 768 / sec, "unit": "entries/s", "h2d_bytes_per_step": Fh.numel() * 8,
            "d2h_bytes_per_step": Oh.numel() * 8, "ms_per_step": sec * 1e3, "steps": steps,
            "path": "sfb_hadamard_rowsum_batched_host (pinned host buffers, 3-stream chunked "
                    "H2D/kernel/D2H pipeline), wall clock per call; result bitwise equal to the "
                    "device path"}


def hadamard_n_sweep(dev, stream, sampler, steps=5):
    """The reference's own benchmark shape (sumfac-bench --dim 3 --n-min 3 --n-max 15:
    time of the sum-factorized Hadamard region vs n, expected slope d+1 = 4) on
    the fused batched kernel: ~2^26 Hadamard entries per point."""
    import torch

    import paper_2306_11665_b200 as sf
    from paper_2306_11665_b200 import _lib
    from paper_2306_11665_b200 import euler as eu

    d, pts = 3, []
    for n in range(3, 16):
        ent = d * n ** (d + 1)
        E = max(1, int(round(2**26 / ent)))
        D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
        basis = sf.assemble_basis_factors(sf.build_sparsity_pattern(n, n, d), D, np.ones(n)).device
        F = eu.generate_uniform(E * ent, 7, -1.0, 1.0, device=dev)
        out = torch.empty((E, n**d), dtype=torch.float64, device=dev)

        def step():
            _lib.call("sfb_hadamard_rowsum_batched", E, n, n, d, _lib.ptr(basis), _lib.ptr(F),
                      None, _lib.ptr(out), _lib.stream_ptr())

        ms, _, _, _ = timed_loop(step, steps, 3, 1, None, stream, sampler)
        pts.append({"n": n, "elements": E, "ms_per_step": ms, "us_per_element": ms * 1e3 / E,
                    "entries_per_s": E * ent / (ms / 1e3),
                    "hbm_frac": 8 * (ent + n**d) * E / (ms / 1e3) / 1e9 / measured_peaks()[0]})
        del F, out
        torch.cuda.empty_cache()
    ns = np.array([p["n"] for p in pts], dtype=float)
    t = np.array([p["us_per_element"] for p in pts])
    return {"workload": "fused Hadamard + row sum + direction sum, d=3, n=3..15, ~2^26 entries "
                        "per point (the reference's sumfac-bench shape, batched)",
            "points": pts,
            "slope_time_per_element_vs_n": float(np.polyfit(np.log(ns), np.log(t), 1)[0]),
            "expected_slope": "d+1 = 4 (the reference's own CPU run: 3.66, BASELINE.md)"}


def run_sweep(args, world, rank, dev, stream, sampler, dist, cpu=False):
    import torch

    from paper_2306_11665_b200 import euler as eu

    points = []
    gates = {}
    t_first = None
    for n in range(2, 9):
        E = int(round(2**24 / n**3))
        U = eu.generate_states(E, n, seed=4, e0=rank * E, device=dev)
        R = torch.empty_like(U)

        def step():
            eu.volume_cartesian(U, n, out=R)

        step()
        gates[n] = gate_cartesian(U, R, n, os.cpu_count() or 1)
        ms_step, per, launches, (t0, t1) = timed_loop(step, args.steps, args.warmup, world, dist,
                                                      stream, sampler)
        t_first = t_first or t0
        kernel_ms = float(np.mean(per))
        dof = E * n**3
        points.append({"n": n, "p": n - 1, "elements": E, "ms_per_step": ms_step,
                       "ns_per_dof": ms_step * 1e6 / dof,
                       "entries_per_s": world * E * 3 * n**4 / (ms_step / 1e3),
                       "hbm_frac": euler_bytes_per_element(n) * E / (kernel_ms / 1e3) / 1e9
                       / measured_peaks()[0],
                       "fp64_frac": euler_flops_per_element(n) * E / (kernel_ms / 1e3) / 1e12
                       / DFMA_MEASURED_TFLOPS})
        del U, R
        torch.cuda.empty_cache()
    # O(n^{d+1}) per element  <=>  time per DOF ~ n  (slope 1 in log-log)
    ns = np.array([p["n"] for p in points], dtype=float)
    t = np.array([p["ns_per_dof"] for p in points])
    slope_all = float(np.polyfit(np.log(ns), np.log(t), 1)[0])
    slope_cb = float(np.polyfit(np.log(ns[3:]), np.log(t[3:]), 1)[0])
    best = min(points, key=lambda p: p["ms_per_step"])
    line = finish_line(args, world, dev, dist, points[2]["ms_per_step"], [points[2]["ms_per_step"]],
                       launches, sampler, t_first, time.time(),
                       units=points[2]["elements"] * 3 * 4**4, unit="entries/s",
                       bytes_launch=euler_bytes_per_element(4) * points[2]["elements"],
                       flops_launch=euler_flops_per_element(4) * points[2]["elements"])
    line["config"] = {"workload": "config4: config-3 kernel swept over n = 2..8, ~2^24 nodes each",
                      "points": len(points)}
    line["sweep"] = points
    line["slope_time_per_dof_vs_n"] = {"all_n": slope_all, "n5_to_8": slope_cb,
                                       "expected": "1 (O(n^{d+1}) per element / n^d DOF)"}
    line["gate"] = {"passed": all(g["passed"] for g in gates.values()),
                    "max_rel": max(g["max_rel"] for g in gates.values()), "tol": GATE_RTOL,
                    "per_n": {n: g["max_rel"] for n, g in gates.items()}}
    if cpu:
        cd = cpu_dense_vs_sumfac(os.cpu_count() or 1)
        for p in points:
            q = next(x for x in cd["points"] if x["n"] == p["n"])
            p["cpu_sumfac_ns_per_dof"] = q["sumfac_ns_per_dof"]
            p["cpu_dense_ns_per_dof"] = q["dense_ns_per_dof"]
        line["cpu_dense_vs_sumfac"] = cd
        p4 = next(x for x in cd["points"] if x["n"] == 4)
        line["cpu_baseline"] = {"value": 3 * 4 / (p4["sumfac_ns_per_dof"] * 1e-9), "unit":
                                "entries/s", "cores": cd["threads"], "kind": "port",
                                "sample": f"{p4['sumfac_sample_elements']} config-4 elements at "
                                          f"n=4, C port of the oracle, {cd['threads']} threads "
                                          f"on {cd['cpu']}"}
    del best
    return line


def run_modal(args, world, rank, dev, stream, sampler, dist, cpu=False, e2e=False):
    import torch

    from paper_2306_11665_b200 import euler as eu
    from paper_2306_11665_b200 import shard

    n = args.n
    total = args.elements
    block = shard.job_block(total)  # one block size for the whole job
    e0, E = shard.block_shard(total, rank, world, block)  # whole blocks per rank
    Uh = eu.generate_modal_states(E, n, seed=5, e0=e0, device=dev)
    Ja = eu.generate_metric(E, n, seed=6, e0=e0, device=dev)
    Rh = torch.empty_like(Uh)
    ss = torch.empty(E, dtype=torch.float64, device=dev)
    norm = [None]

    def step():
        eu.volume_curvilinear_modal(Uh, Ja, n, out=Rh, sumsq=ss)
        # device scalar: partials, NCCL all_gather, fixed tree; no host sync
        norm[0] = shard.global_norm_tensor(ss, block=block, total=total)

    step()
    gate = gate_modal(Uh, Ja, Rh, ss, n, os.cpu_count() or 1)
    ms_step, per, launches, (t0, t1) = timed_loop(step, args.steps, args.warmup, world, dist,
                                                  stream, sampler)
    line = finish_line(args, world, dev, dist, ms_step, per, launches, sampler, t0, t1,
                       units=E * n**3, unit="element-DOF/s",
                       bytes_launch=modal_bytes_per_element(n) * E,
                       flops_launch=modal_flops_per_element(n) * E,
                       metric="FP64 element-DOF/s (3D curvilinear modal Euler flux differencing)",
                       traffic=ncu_traffic(args, n, E))
    line["value"] = total * n**3 / (line["ms_per_step"] / 1e3)  # strong scaling: total DOF
    line["residual_norm"] = float(norm[0].item())
    line["hadamard_entries_per_s"] = total * 3 * n**4 / (line["ms_per_step"] / 1e3)
    line["gate"] = gate
    step_ms = torch.tensor([float(np.mean(per))], dtype=torch.float64, device=dev)
    if world > 1:
        allk = [torch.empty_like(step_ms) for _ in range(world)]
        dist.all_gather(allk, step_ms)
        line["per_rank_kernel_ms"] = [float(x.item()) for x in allk]
    else:
        line["per_rank_kernel_ms"] = [float(step_ms.item())]
    line["elements_per_rank"] = E
    if cpu:
        line["cpu_baseline"] = cpu_baseline_modal(args, Uh, Ja)
    if e2e:
        line["e2e"] = e2e_modal(args, Uh, Ja, Rh, ss)
    del Uh, Ja, Rh, ss
    torch.cuda.empty_cache()
    return line


def cpu_baseline_modal(args, Uh, Ja):
    from oracle import c_oracle, workload

    n = args.n
    threads = os.cpu_count() or 1
    sample = min(Uh.shape[0], args.cpu_sample_c5)
    Us, Js = Uh[:sample].cpu().numpy(), Ja[:sample].cpu().numpy()
    _, D, V, Pi = workload.gll_operators(n)
    c_oracle.euler_volume_curvilinear_modal(Us[:threads], Js[:threads], V, Pi, D, threads=threads)
    t, reps = time.perf_counter(), 0
    while True:
        c_oracle.euler_volume_curvilinear_modal(Us, Js, V, Pi, D, threads=threads)
        reps += 1
        if time.perf_counter() - t > args.cpu_seconds_extra:
            break
    sec = (time.perf_counter() - t) / reps
    return {"value": sample * n**3 / sec, "unit": "element-DOF/s", "cores": threads,
            "kind": "port",
            "sample": f"first {sample} of the {args.elements} config-5 elements x {reps} reps "
                      f"(per-DOF rate of the sample, extrapolated: the full job would take "
                      f"{args.elements * sec / sample:.0f} s), C port of the oracle "
                      f"(oracle/euler_oracle.c), {threads} threads on {cpu_model()}"}


def e2e_modal(args, Uh_dev, Ja_dev, Rh_dev, ss_dev, steps=3):
    """Config 5 through the host-buffer C-ABI entry on an element sample (the whole
    job's inputs are 51 GB: pinned host buffers of that size are not a sane test)."""
    import torch

    from paper_2306_11665_b200 import euler as eu

    n = args.n
    E = min(Uh_dev.shape[0], args.e2e_sample_c5)
    Uh = eu.pinned_empty((E, 5, n**3))
    Uh.copy_(Uh_dev[:E].cpu())
    Ja = eu.pinned_empty((E, 3, 3, n**3))
    Ja.copy_(Ja_dev[:E].cpu())
    Rh = eu.pinned_empty((E, 5, n**3))
    ss = eu.pinned_empty((E,))
    eu.volume_curvilinear_modal_host(Uh, Ja, n, out=Rh, sumsq=ss)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        eu.volume_curvilinear_modal_host(Uh, Ja, n, out=Rh, sumsq=ss)
        times.append(time.perf_counter() - t)
    sec = float(np.mean(times))
    assert torch.equal(Rh, Rh_dev[:E].cpu()) and torch.equal(ss, ss_dev[:E].cpu()), \
        "config-5 e2e result differs from the device path"
    return {"value": E * n**3 / sec, "unit": "element-DOF/s",
            "h2d_bytes_per_step": (Uh.numel() + Ja.numel()) * 8,
            "d2h_bytes_per_step": (Rh.numel() + ss.numel()) * 8, "ms_per_step": sec * 1e3,
            "steps": steps, "sample_elements": E,
            "path": f"sfb_euler_volume_curvilinear_modal_host on the first {E} elements "
                    "(pinned host buffers, 3-stream chunked H2D/kernel/D2H pipeline), wall "
                    "clock per call; result bitwise equal to the device path"}


def measure_other_configs(args, dev, stream, sampler, dist):
    """Configs 2, 4, 5 in the same run (N=1), summarised; full lines via --config."""
    import copy

    import torch

    out = {}
    keep = ("workload", "metric", "value", "unit", "ms_per_step")
    for cfg in (2, 4, 5):
        a = copy.copy(args)
        a.config = cfg
        a.steps = 10 if cfg != 5 else 5
        a.warmup = 3
        a.n = 6 if cfg == 5 else 4
        a.elements = 2**21 if cfg == 5 else 262144
        a.traffic = None
        with_cpu = not args.no_cpu_baseline
        if cfg == 2:
            ln = run_hadamard(a, 1, 0, dev, stream, sampler, dist, cpu=with_cpu,
                              e2e=not args.no_e2e)
        elif cfg == 4:
            ln = run_sweep(a, 1, 0, dev, stream, sampler, dist, cpu=with_cpu)
        else:
            ln = run_modal(a, 1, 0, dev, stream, sampler, dist, cpu=with_cpu,
                           e2e=not args.no_e2e)
        summary = {k: (ln["config"]["workload"] if k == "workload" else ln[k]) for k in keep}
        summary["roofline"] = {k: ln["roofline"][k] for k in ("bound", "achieved", "peak", "unit",
                                                              "frac", "note") if k in ln["roofline"]}
        for k in ("gate", "cpu_baseline", "e2e", "cpu_dense_vs_sumfac", "residual_norm"):
            if k in ln:
                summary[k] = ln[k]
        if cfg == 4:
            summary["sweep"] = [{k: p[k] for k in ("n", "elements", "ms_per_step", "ns_per_dof",
                                                   "hbm_frac", "fp64_frac", "cpu_sumfac_ns_per_dof",
                                                   "cpu_dense_ns_per_dof") if k in p}
                                for p in ln["sweep"]]
            summary["slope_time_per_dof_vs_n"] = ln["slope_time_per_dof_vs_n"]
        if cfg == 2 and "n_sweep" in ln:
            summary["n_sweep_slope_time_per_element"] = ln["n_sweep"]["slope_time_per_element_vs_n"]
            summary["n_sweep_us_per_element"] = {p["n"]: p["us_per_element"]
                                                 for p in ln["n_sweep"]["points"]}
        out[f"config{cfg}"] = summary
        torch.cuda.empty_cache()
    out["f3_burgers_rk4"] = measure_burgers_rk4(dev)
    return out


def measure_burgers_rk4(dev, E=1 << 20, d=2, n=5, steps=20):
    """RK4 on the periodic Burgers element, whole run in one launch."""
    import torch

    from paper_2306_11665_b200 import burgers as bg
    from paper_2306_11665_b200 import euler as eu

    u0 = eu.generate_uniform(E * n**d, 11, -1.0, 1.0, device=dev).reshape(E, n**d)
    bg.integrate_rk4(u0[:1024], d, n, 1e-3, 2, every=1)  # warm-up / operator cache
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    u, ent, mass = bg.integrate_rk4(u0, d, n, 1e-3, steps, every=steps)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    drift = float(((ent[:, -1] - ent[:, 0]).abs() / ent[:, 0]).max())
    return {"workload": f"periodic Burgers d={d} n={n}, {E} elements, {steps} RK4 steps "
                        f"(4 time derivatives each), entropy monitored on device",
            "value": E * steps / (ms / 1e3), "unit": "element-steps/s", "ms": ms,
            "launches": 1, "max_rel_entropy_drift_ec": drift}


def measure_e2e(args, U_dev, world=1, dist=None, dev=None):
    """Through the C-ABI host-buffer entry: pinned host U in, pinned host R out.

    Every rank runs its own shard; the step time is the max over ranks and the
    value the whole job's entries per second."""
    import torch

    from paper_2306_11665_b200 import euler as eu

    n, E = args.n, args.elements
    Uh = eu.pinned_empty(tuple(U_dev.shape))
    Uh.copy_(U_dev.cpu())
    Rh = eu.pinned_empty(tuple(U_dev.shape))
    steps = max(3, min(args.steps, 10))
    for _ in range(2):
        eu.volume_cartesian_host(Uh, n, out=Rh)
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        eu.volume_cartesian_host(Uh, n, out=Rh)
        times.append(time.perf_counter() - t)
    sec = float(np.mean(times))
    if world > 1:
        t = torch.tensor([sec], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    # the result is read on the host: cross-check one element against the device path
    Rd = eu.volume_cartesian(U_dev[:1].contiguous(), n).cpu()
    assert torch.equal(Rd[0], Rh[0]), "e2e result differs from the device path"
    nbytes = Uh.numel() * 8
    ceil_ms = pcie_ceiling_ms(Uh, Rh, U_dev)
    return {"value": world * E * 3 * n**4 / sec, "unit": "entries/s",
            "h2d_bytes_per_step": world * nbytes, "d2h_bytes_per_step": world * nbytes,
            "ms_per_step": sec * 1e3, "steps": steps, "n_ranks": world,
            "pcie_ceiling_ms": ceil_ms, "frac_of_pcie_ceiling": ceil_ms / (sec * 1e3),
            "pcie_ceiling": "same box, same buffers: pinned H2D of U and D2H of R as two "
                            "concurrent plain copies (no kernel), CUDA events",
            "path": "sfb_euler_volume_cartesian_host (pinned host buffers, 3-stream "
                    "chunked H2D/kernel/D2H pipeline), wall clock per call"}


def pcie_ceiling_ms(Uh, Rh, U_dev, reps=5):
    """Time of the e2e step's copies alone (pinned U -> device, device -> pinned
    R, concurrently on two streams): the link ceiling the e2e leg is read against."""
    import torch

    D = torch.empty_like(U_dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            D.copy_(Uh, non_blocking=True)
        with torch.cuda.stream(s2):
            Rh.copy_(U_dev, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    both()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        both()
    e1.record()
    torch.cuda.synchronize()
    del D
    return e0.elapsed_time(e1) / reps


def measure_cpu_baseline(args, U_dev):
    from oracle import c_oracle, workload

    n = args.n
    threads = os.cpu_count() or 1
    sample = min(args.elements, args.cpu_sample)
    Us = U_dev[:sample].cpu().numpy()
    D = workload.gll_operators(n)[1]
    c_oracle.euler_volume_cartesian(Us[: max(1, sample // 10)], D, threads=threads)
    t = time.perf_counter()
    reps = 0
    while True:
        c_oracle.euler_volume_cartesian(Us, D, threads=threads)
        reps += 1
        if time.perf_counter() - t > args.cpu_seconds:
            break
    sec = (time.perf_counter() - t) / reps
    return {"value": sample * 3 * n**4 / sec, "unit": "entries/s", "cores": threads,
            "kind": "port",
            "sample": f"{sample} of the {args.elements} config-3 elements x {reps} reps, C port "
                      f"of the oracle (oracle/euler_oracle.c), {threads} threads on {cpu_model()}"}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--elements", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the configs 2/4/5 summaries appended to the default line")
    ap.add_argument("--cpu-sample", type=int, default=262144)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)  # ~10-30 s of CPU work
    ap.add_argument("--cpu-seconds-extra", type=float, default=4.0,
                    help="CPU work per cpu_baseline of the configs 2/5 summaries")
    ap.add_argument("--cpu-sample-c5", type=int, default=8192,
                    help="config-5 elements in a CPU sample (reference arm / cpu_baseline)")
    ap.add_argument("--e2e-sample-c5", type=int, default=131072,
                    help="config-5 elements in the host-buffer e2e leg")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the top kernel (default: profiles/)")
    args = ap.parse_args(argv)
    if args.n is None:
        args.n = 6 if args.config == 5 else 4
    if args.elements is None:
        args.elements = 2**21 if args.config == 5 else 262144
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and argv is None:
        # plain `python bench.py --gpus N`: relaunch as N ranks (what the driver
        # does itself with torch.distributed.run)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", os.environ.get("MASTER_PORT", "29511"),
               os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    raise SystemExit(main())
