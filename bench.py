"""Benchmark: realization·timesteps/s of the noisy-CTQW hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the configuration the metric is quoted on
that fits one GPU): 2 particles on an N = 256 ring (D = 65 536, 1 MiB complex128
state per realization), R = 1000 realizations PER GPU (weak scaling), static
tunnelling noise (levels +-0.1, seeds (1234, r)), Taylor order 4, dt = 0.02,
the per-step norm policy, and one collection point (diagonal observables:
populations, position moments, participation ratio) at the end of the timed
region (post_rate = K).  A "step" advances every realization by one dt.

Lines printed by rank 0 (one JSON object):
  value       realization·steps/s over all ranks, device-timed (CUDA events,
              max over ranks), states resident in HBM (1 GiB per buffer >> L2)
  e2e         the same metric through the public API ``run(config)``: host
              initial state uploaded, noise drawn, K steps, observable rows
              copied back to the host, wall-timed (after one untimed run())
  roofline    the streaming step kernel: algorithmic bytes 32*D per
              realization per launch / CUDA-event launch time, vs MEASURED_PEAKS
  cpu_baseline the NumPy oracle port on the host cores, bounded sample
``--impl reference`` runs the reference algorithm (oracle port of
``ctqw._evolve_segment``) on the host cores on a bounded sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "realization·timesteps/sec (2-particle, N-site lattice)"
UNIT = "realization·steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--m", type=int, default=2)
    ap.add_argument("--realizations", type=int, default=1000, help="per GPU")
    ap.add_argument("--backend", default="taylor", choices=("taylor", "rk4"))
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--dt", type=float, default=0.02)
    ap.add_argument("--rate", type=float, default=0.0,
                    help="telegraph switching rate (0 = static disorder, the BASELINE configs; the "
                         "reference's CLI default is 0.1)")
    ap.add_argument("--exact", action="store_true",
                    help="reference operation order without FMA (bit-identical to the reference between "
                         "renormalisations) for the headline value; default is the FMA-contracted stencil, "
                         "which the parity tests hold to <= 1e-12 of the reference (north-star bar 1e-10)")
    ap.add_argument("--fma", action="store_true", help=argparse.SUPPRESS)  # the default; kept for old scripts
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU side (oracle port = the reference's algorithm, NumPy)


_WORKER_STATE = {}


def _cpu_worker(args):
    """One task = ``count`` realizations advanced ``steps`` steps by the oracle.

    The realization stack persists in the worker process between tasks (like
    the reference's per-worker chunks), so only stepping is timed.
    """
    n, m, count, r0, steps, dt, backend, order = args
    import numpy as np

    from oracle import ctqw_oracle as orc

    key = (n, m, count, backend, order, dt)
    st_psi = _WORKER_STATE.get(key)
    if st_psi is None:
        noise = np.stack([np.random.default_rng((1234, r)).choice(np.array([-0.1, 0.1]), n)
                          for r in range(r0, r0 + count)])
        st = orc.make_stencil(m, n, 0.0, 1.0, 0.0, link=noise, batch=count)
        st_psi = (st, np.tile(orc.product_state(m, n), (count, 1)), 0)
    st, psi, done = st_psi
    t0 = time.perf_counter()
    psi, _ = orc.evolve_segment(st, psi, done, steps, dt, 1.0, backend, order)
    _WORKER_STATE[key] = (st, psi, done + steps)
    return time.perf_counter() - t0


class CpuPool:
    """Persistent spawn pool of ``cores`` processes (1 BLAS thread each)."""

    def __init__(self, cores):
        from concurrent.futures import ProcessPoolExecutor
        import multiprocessing as mp

        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        self.cores = cores
        self.pool = ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn"))

    def step(self, n, m, backend, order, dt, per_core, steps):
        jobs = [(n, m, per_core, 100000 + i * per_core, steps, dt, backend, order) for i in range(self.cores)]
        t0 = time.perf_counter()
        list(self.pool.map(_cpu_worker, jobs))
        return time.perf_counter() - t0

    def close(self):
        self.pool.shutdown(wait=True)


def cpu_rate(n, m, backend, order, dt, per_core, seconds, cores=None):
    """Wall rate of the oracle on ``cores`` processes: one calibration step,
    then as many steps as fill ~``seconds`` of wall time, timed as one round."""
    cores = cores or host_cores()
    pool = CpuPool(cores)
    try:
        pool.step(n, m, backend, order, dt, per_core, 1)  # imports + state set-up
        t1 = pool.step(n, m, backend, order, dt, per_core, 1)
        steps = max(1, min(500, int(round(seconds / max(t1, 1e-6)))))
        wall = pool.step(n, m, backend, order, dt, per_core, steps)
    finally:
        pool.close()
    return cores * per_core * steps / wall, cores, wall, steps


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample_size(n, m):
    """Realizations per core of the CPU sample (a few MiB of state per process)."""
    dim = n ** m
    return max(1, min(16, (8 << 20) // (16 * dim)))


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    per_core = 2 if a.n ** a.m >= 65536 else 8
    pool = CpuPool(cores)
    try:
        for _ in range(max(a.warmup, 1)):
            pool.step(a.n, a.m, a.backend, a.order, a.dt, per_core, 1)
        t_all = 0.0
        for _ in range(a.steps):
            t_all += pool.step(a.n, a.m, a.backend, a.order, a.dt, per_core, 1)
    finally:
        pool.close()
    value = a.steps * cores * per_core / t_all
    sample = (f"{cores} processes x {per_core} realizations advanced 1 step per timed step "
              f"(N={a.n}, m={a.m}; oracle port of ctqw._evolve_segment)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 * t_all / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (static tunnelling noise, seeds (1234, r))",
        "config": workload_config(a),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(a):
    state_gib = a.realizations * a.n ** a.m * 16 / 2**30
    label = "configs[1]: " if (a.m, a.n) == (2, 256) else ""
    noise = "static tunnelling noise" if a.rate == 0 else f"telegraph tunnelling noise (rate {a.rate})"
    return {
        "workload": f"{label}m={a.m} particles, N={a.n} ring (D={a.n ** a.m}), "
                    f"{a.realizations} realizations per GPU, {noise}, "
                    f"{a.backend}{'' if a.backend == 'rk4' else '-' + str(a.order)}, dt={a.dt}, "
                    f"norm policy every step, diagonal observables at the last step",
        "n_sites": a.n, "particles": a.m, "realizations_per_gpu": a.realizations,
        "backend": a.backend, "taylor_order": a.order, "dt": a.dt,
        "exact_order": bool(a.exact),
        "arithmetic": ("exact reference order (bit-identical between renormalisations)" if a.exact else
                       "FMA-contracted stencil (Horner-form Taylor), FP64, <= 1e-12 from the reference "
                       "(tests/test_gpu_parity.py)"),
        "l2_policy": (f"inputs larger than L2 (state stack {state_gib:.2f} GiB per buffer per GPU, L2 126 MB)"
                      if state_gib * 2**30 > 126e6 else
                      f"state stack {state_gib * 1024:.0f} MiB per GPU fits in L2: not an HBM measurement"),
    }


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~10 ms while
    the timed region runs (falls back to nvidia-smi if NVML is missing)."""

    REASONS = {  # nvmlClocksEventReason* bit -> name used in the JSON line
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            try:
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            return float(sm), float(mx), int(bits)
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        return float(out[0]), float(out[1]), int(out[2].strip(), 16)

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        bits = 0
        for _, _, b in self.samples:
            bits |= b
        reasons = sorted(name for bit, name in self.REASONS.items() if bits & bit)
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# GPU arm


def ours(a):
    import torch
    import torch.distributed as dist

    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import engine, sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    # launched by torchrun: one process per GPU over NCCL (also at world 1, so
    # the distributed path -- barriers, MAX reductions, run(group=...) -- runs)
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    # CTQW_DIST_BACKEND=gloo lets several ranks share one GPU, to exercise the
    # N > 1 code path (barriers, MAX reductions, sharded run()) on a one-GPU
    # box; measurements use NCCL with one GPU per rank
    backend = os.environ.get("CTQW_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if distributed:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    R_total = a.realizations * world
    obs = ("populations", "position_mean_variance", "participation_ratio")
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([a.n]), a.m),
                      noise=p.NoiseSpec(target="tunneling", levels=(-0.1, 0.1), rate=a.rate),
                      stepper=p.StepperConfig(backend=a.backend, dt=a.dt, taylor_order=a.order),
                      realizations=R_total, steps=a.steps, post_rate=a.steps, precision="double",
                      observables=obs, memory_budget=170 * 2**30, exact=bool(a.exact), device=local)
    lo, hi = sharding.shard_bounds(R_total, world, rank)
    ens = engine.EnsembleState(cfg, local, lo, hi)
    h = ens.handle
    dim = a.n ** a.m

    def barrier():
        if distributed:
            dist.barrier()

    # warm-up (includes one collection point)
    for k in range(a.warmup):
        ens.evolve(k, 1)
        ens.stats()
    engine.collect_observables(cfg, ens)
    torch.cuda.synchronize()

    # timed region: K steps + the collection point, device-timed
    ens.handle.kernel_timing(True)
    launches0 = h.launches
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start.record()
        ens.evolve(a.warmup, a.steps)
        stats = ens.stats()
        engine.collect_observables(cfg, ens)
        stop.record()
        torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(stop)
    kernel_ms, kernel_launches = h.kernel_time()
    kernel = h.step_kernel()
    h.kernel_timing(False)
    launches = h.launches - launches0
    # the other arithmetic mode on the same states (reported beside the headline)
    ens.stepper = cfg.stepper.native(not a.exact)
    ens.evolve(a.warmup + a.steps, 2)
    barrier()
    torch.cuda.synchronize()
    start.record()
    ens.evolve(a.warmup + a.steps + 2, a.steps)
    ens.stats()
    engine.collect_observables(cfg, ens)
    stop.record()
    torch.cuda.synchronize()
    ms_other = start.elapsed_time(stop)
    ens.stepper = cfg.stepper.native(bool(a.exact))
    t = torch.tensor([ms, ms_other], device=f"cuda:{local}")
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_other_max = float(t[1].item())
    ms_max = float(t[0].item())
    value = R_total * a.steps / (ms_max / 1000.0)
    assert stats["failure"] is None

    # roofline of the dominant kernel (streaming step / resident segment)
    avg_launch_ms = kernel_ms / max(kernel_launches, 1)
    bytes_per_launch = (hi - lo) * 32.0 * dim
    if kernel_launches == 1 and a.n <= 64:
        bytes_per_launch *= a.steps  # resident: one launch covers every step
    achieved = bytes_per_launch / (avg_launch_ms / 1000.0) / 1e9
    peak, peak_src = measured_peak_hbm()
    traffic = ncu_traffic()
    traffic_bytes = None
    if traffic and traffic.get("kernel") == kernel and a.n == 256 and a.m == 2:
        # ncu --set full capture (profiles/), per realization-step, scaled to this launch
        traffic_bytes = traffic["dram_bytes_per_realization_step"] * (hi - lo)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "frac_of_spec_8000": achieved / 8000.0, "traffic": traffic_bytes,
                "traffic_source": traffic.get("source") if traffic_bytes else None,
                "kernel": kernel,
                "kernel_ms_avg": avg_launch_ms, "kernel_launches": kernel_launches,
                "kernel_share_of_step": kernel_ms / ms if ms > 0 else None,
                "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_src,
                "flops_per_launch": (hi - lo) * dim * (22.0 * a.order if a.backend == "taylor" else 112.0)}
    roofline["achieved_fp64_tflops"] = roofline["flops_per_launch"] / (avg_launch_ms / 1000.0) / 1e12

    # e2e through the public API: run(config) with host I/O
    e2e = None
    if not a.no_e2e:
        sinks = p.MemorySinks(keep_densities=False)
        # one untimed run() first, as the device arm's warm-up steps: the
        # allocator then serves this run's buffers from its cache
        p.run(cfg, p.MemorySinks(keep_densities=False), group=dist.group.WORLD if distributed else None)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        p.run(cfg, sinks, group=dist.group.WORLD if distributed else None)
        torch.cuda.synchronize()
        t_e2e = torch.tensor([time.perf_counter() - t0], device=f"cuda:{local}")
        if distributed:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        e2e_s = float(t_e2e.item())
        h2d = dim * 16 + 16  # initial state + noise levels
        d2h = (a.n + 3) * 8 * len(cfg.schedule)  # observable rows per collection point
        e2e = {"value": R_total * a.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d / a.steps, "d2h_bytes_per_step": d2h / a.steps,
               "seconds": e2e_s, "api": "paper_1612_00746_b200.run(RunConfig, MemorySinks)"}

    cpu = None  # the host-core baseline is taken on rank 0 at N = 1 only
    if rank == 0 and world == 1 and not a.no_cpu:
        cores = host_cores()
        per_core = cpu_sample_size(a.n, a.m)
        rate, cores, wall, steps = cpu_rate(a.n, a.m, a.backend, a.order, a.dt, per_core, a.cpu_seconds, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{cores} processes x {per_core} realizations x {steps} steps of the same "
                         f"workload (oracle port of the reference algorithm), {wall:.1f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (static tunnelling noise drawn on device, seeds (1234, r))",
            "config": dict(workload_config(a), parallelism=f"realizations sharded over {world} GPU(s)"),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "other_arithmetic": {"exact_order": not a.exact,
                                 "value": R_total * a.steps / (ms_other_max / 1000.0),
                                 "ms_per_step": ms_other_max / a.steps},
            "clocks": clocks.summary(),
            "norm_events": stats["event_count"],
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    else:
        ours(a)


if __name__ == "__main__":
    main()
