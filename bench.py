"""Benchmark: realization·timesteps/s of the noisy-CTQW hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config I]

Workload (default ``--config 2``): BASELINE.json configs[2]'s per-GPU shard --
2 particles on an N = 1024 ring (D = 2^20, 16 MiB complex128 state per
realization), 1250 realizations PER GPU (configs[2]'s 10^4 over 8 GPUs; weak
scaling), static on-site + tunnelling noise (levels +-0.1, seeds (1234, r)),
Taylor order 4, dt = 0.02, the per-step norm policy, and one collection point
(diagonal observables: populations, position moments, participation ratio) at
the end of the timed region (post_rate = K).  A "step" advances every
realization by one dt.  ``--config 0..4`` selects the other BASELINE
configurations (the parity tests cover all of them).

``--gpus N`` with N > 1 launches N ranks itself (torch.distributed.run, NCCL,
127.0.0.1) unless it already runs under torchrun; one process per GPU.

Line printed by rank 0 (one JSON object):
  value        realization·steps/s over all ranks, device-timed (CUDA events,
               max over ranks), states resident in HBM (20 GiB per buffer >> L2)
  e2e          the same metric through the public API ``run(config)``: host
               initial state uploaded, noise drawn on the device, K steps,
               observable rows copied back to the host, wall-timed
  roofline     the dominant step kernel: algorithmic bytes 32*D per
               realization per launch / CUDA-event launch time, vs MEASURED_PEAKS
  cpu_baseline the reference's own CPU path (``ctqw`` installed under
               baseline/_ref, its worker pool ``_init_worker``/``_segment_task``)
               on the host cores, bounded sample
  secondary    configs[1] (N = 256, R = 1000) measured the same way, device-timed
``--impl reference`` times that reference path per step on the host cores.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

METRIC = "realization·timesteps/sec (2-particle, N-site lattice)"
UNIT = "realization·steps/s"

# BASELINE.json configs, per-GPU shapes (weak scaling: realizations per GPU)
PRESETS = {
    0: dict(n=64, m=2, realizations=100, target="tunneling", dt=0.02,
            label="configs[0]: N=64, 100 realizations, static tunnelling noise"),
    1: dict(n=256, m=2, realizations=1000, target="tunneling", dt=0.02,
            label="configs[1]: N=256, 1000 realizations per GPU, static tunnelling noise"),
    2: dict(n=1024, m=2, realizations=1250, target="both", dt=0.02,
            label="configs[2] per-GPU shard: N=1024, 1250 realizations per GPU (10^4 over 8 GPUs), "
                  "static on-site + tunnelling noise, streaming TMA path"),
    3: dict(n=512, m=2, realizations=1000, target="tunneling", dt=0.02,
            label="configs[3]: N=512, 1000 realizations per GPU, static tunnelling noise"),
    4: dict(n=128, m=3, realizations=5300, target="tunneling", dt=0.015,
            label="configs[4]: m=3, N=128 (D=2^21), 5300 realizations per GPU (largest that fits)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=2, choices=sorted(PRESETS))
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--realizations", type=int, default=None, help="per GPU")
    ap.add_argument("--target", default=None, choices=("tunneling", "onsite", "both"))
    ap.add_argument("--backend", default="taylor", choices=("taylor", "rk4"))
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--dt", type=float, default=None)
    ap.add_argument("--post-rate", type=int, default=0, help="collection every P steps (0: once, at the end)")
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
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-other", action="store_true", help="skip the other-arithmetic measurement")
    a = ap.parse_args()
    pre = PRESETS[a.config]
    for key in ("n", "m", "realizations", "target", "dt"):
        if getattr(a, key) is None:
            setattr(a, key, pre[key])
    a.custom = any(getattr(a, k) != pre[k] for k in ("n", "m", "realizations", "target", "dt"))
    return a


# ---------------------------------------------------------------------------
# CPU side: the reference's own code (baseline/_ref), through its worker pool


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def physical_cores():
    try:
        import psutil

        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:
        pass
    try:
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        pairs = {ln for ln in out.splitlines() if ln and not ln.startswith("#")}
        return len(pairs) or None
    except Exception:
        return None


def import_reference():
    """The unmodified reference package installed under baseline/_ref (pip --target)."""
    if os.path.isdir(os.path.join(REF_DIR, "ctqw")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import ctqw  # noqa: F401
        from ctqw import ensemble

        if os.path.dirname(os.path.dirname(os.path.abspath(ensemble.__file__))) == os.path.abspath(REF_DIR):
            return ensemble
    return None


def _oracle_segment(args):
    """Fallback worker (baseline/_ref missing): the oracle port of _evolve_segment."""
    chunk, start, steps, dt, backend, order = args
    from oracle import ctqw_oracle as orc

    st, psi = chunk
    psi, _ = orc.evolve_segment(st, psi, start, steps, dt, 1.0, backend, order)
    return (st, psi)


class ReferencePool:
    """The reference's own parallel harness (ensemble.py:672-731): a spawn
    pool initialised with ``_init_worker(ctx)``; each round submits
    ``_segment_task(chunk, start, n_steps)`` for every chunk and collects the
    chunks back, exactly as ``run`` does between two collection points.
    One chunk of ``per_worker`` realizations per worker, 1 BLAS thread each.
    """

    def __init__(self, a, workers, per_worker):
        from concurrent.futures import ProcessPoolExecutor
        import multiprocessing as mp

        import numpy as np

        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        os.environ["MKL_NUM_THREADS"] = "1"
        self.workers = workers
        self.per_worker = per_worker
        self.ens = import_reference()
        self.kind = "reference" if self.ens is not None else "port"
        ctx_mp = mp.get_context("spawn")
        r0 = 100000
        if self.ens is not None:
            import ctqw

            space = ctqw.JointSpace(ctqw.build_lattice([a.n]), a.m)
            cfg = ctqw.RunConfig(space=space,
                                 noise=ctqw.NoiseSpec(target=a.target, levels=(-0.1, 0.1), rate=a.rate),
                                 stepper=ctqw.StepperConfig(backend=a.backend, dt=a.dt, taylor_order=a.order),
                                 realizations=workers * per_worker, steps=1, post_rate=1, precision="double")
            topology = ctqw.build_topology(space)
            psi0 = ctqw.build_initial_state(cfg.initial, space).astype(np.complex128)
            self.chunks = []
            for w in range(workers):
                lo = r0 + w * per_worker
                self.chunks.append(self.ens._ChunkState(
                    r0=lo, psi=np.tile(psi0, (per_worker, 1)),
                    noise=[ctqw.init_process(cfg.noise, topology, seed=(cfg.master_seed, r))
                           for r in range(lo, lo + per_worker)]))
            ctx = self.ens._WorkerContext(topology=topology, model=cfg.model, stepper=cfg.stepper,
                                          dtype_name="complex128", dense_cap=cfg.dense_cap)
            self.pool = ProcessPoolExecutor(max_workers=workers, mp_context=ctx_mp,
                                            initializer=self.ens._init_worker, initargs=(ctx,))
            list(self.pool.map(self.ens._ping, range(2 * workers)))
        else:
            from oracle import ctqw_oracle as orc

            self.chunks = []
            for w in range(workers):
                lo = r0 + w * per_worker
                nl = a.n if a.target in ("tunneling", "both") else 0
                ns = a.n if a.target in ("onsite", "both") else 0
                noise = np.stack([np.random.default_rng((1234, r)).choice(np.array([-0.1, 0.1]), nl + ns)
                                  for r in range(lo, lo + per_worker)])
                st = orc.make_stencil(a.m, a.n, 0.0, 1.0, 0.0, link=noise[:, :nl] if nl else None,
                                      site=noise[:, nl:] if ns else None, batch=per_worker)
                self.chunks.append((st, np.tile(orc.product_state(a.m, a.n), (per_worker, 1))))
            self.pool = ProcessPoolExecutor(max_workers=workers, mp_context=ctx_mp)
            self.a = a
        self.step_no = 0

    def round(self, steps):
        """Advance every chunk by ``steps`` steps; wall seconds of the round."""
        t0 = time.perf_counter()
        if self.ens is not None:
            futs = [self.pool.submit(self.ens._segment_task, c, self.step_no, steps) for c in self.chunks]
            self.chunks = [f.result()[0] for f in futs]
        else:
            a = self.a
            futs = [self.pool.submit(_oracle_segment, (c, self.step_no, steps, a.dt, a.backend, a.order))
                    for c in self.chunks]
            self.chunks = [f.result() for f in futs]
        self.step_no += steps
        return time.perf_counter() - t0

    @property
    def realizations(self):
        return self.workers * self.per_worker

    def describe(self):
        what = ("the reference's own ctqw (baseline/_ref) worker pool: _init_worker + _segment_task per chunk "
                "(ensemble.py:672-731)" if self.kind == "reference" else
                "oracle port of ctqw._evolve_segment (baseline/_ref not installed)")
        return f"{self.workers} workers x {self.per_worker} realizations, {what}"

    def close(self):
        self.pool.shutdown(wait=True)


def cpu_workers():
    return physical_cores() or host_cores()


def cpu_sample_size(n, m):
    """Realizations per worker: a few MiB of state per process."""
    dim = n ** m
    return max(1, min(8, (4 << 20) // (16 * dim)))


def pool_rate(a):
    """Wall rate of the reference's own pool on this workload: one W-step
    warm segment (spawn, imports, first touch), then the K timed steps as one
    segment per chunk, as run() does between two collection points (the
    values are assembled once per segment).  Both arms report this same
    measurement, so a run carries one CPU number."""
    workers = cpu_workers()
    pool = ReferencePool(a, workers, cpu_sample_size(a.n, a.m))
    try:
        pool.round(max(a.warmup, 1))
        t_all = pool.round(a.steps)
    finally:
        pool.close()
    sample = f"{pool.describe()}, the K timed steps as one {a.steps}-step segment per chunk ({t_all:.1f} s wall)"
    return a.steps * pool.realizations / t_all, pool, t_all, sample


def cores_info(workers):
    return {"cores": workers, "os_cpu_count": os.cpu_count(), "affinity_cpus": host_cores(),
            "physical_cores": physical_cores()}


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    value, pool, t_all, sample = pool_rate(a)
    workers = pool.workers
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 * t_all / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": data_label(a),
        "config": dict(workload_config(a), parallelism=f"realizations sharded over {a.gpus} GPU(s)"),
        "cpu_baseline": dict({"value": value, "unit": UNIT, "kind": pool.kind, "sample": sample},
                             **cores_info(workers)),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def data_label(a):
    noise = {"tunneling": "tunnelling", "onsite": "on-site", "both": "on-site + tunnelling"}[a.target]
    kind = "static" if a.rate == 0 else f"telegraph (rate {a.rate})"
    return f"synthetic ({kind} {noise} noise, levels +-0.1, seeds (1234, r), drawn on the device)"


def workload_config(a):
    state_gib = a.realizations * a.n ** a.m * 16 / 2**30
    label = PRESETS[a.config]["label"] if not a.custom else "custom"
    noise = {"tunneling": "tunnelling", "onsite": "on-site", "both": "on-site + tunnelling"}[a.target]
    noise = f"static {noise} noise" if a.rate == 0 else f"telegraph {noise} noise (rate {a.rate})"
    post = "diagonal observables at the last step" if a.post_rate <= 0 else f"diagonal observables every {a.post_rate} steps"
    return {
        "workload": f"{label} | m={a.m} particles, N={a.n} ring (D={a.n ** a.m}), "
                    f"{a.realizations} realizations per GPU, {noise}, "
                    f"{a.backend}{'' if a.backend == 'rk4' else '-' + str(a.order)}, dt={a.dt}, "
                    f"norm policy every step, {post}",
        "baseline_config": None if a.custom else a.config,
        "n_sites": a.n, "particles": a.m, "realizations_per_gpu": a.realizations, "noise_target": a.target,
        "backend": a.backend, "taylor_order": a.order, "dt": a.dt, "post_rate": a.post_rate or None,
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


def fp64_flops_per_amplitude_step(a):
    """Algorithmic FP64 flops per amplitude and step of the FMA-form kernels:
    per stencil application 2m neighbour terms (complex x real, 4 flops each)
    plus the diagonal (2, +1 per on-site noise add; none when eps0 = U = 0
    without site noise, where the first neighbour term is a multiply: -2), and
    the Horner / RK4 combination (4 flops; RK4 adds the accumulation, 4)."""
    site = a.target in ("onsite", "both")
    zd = not site  # the bench's model: eps0 = U = 0
    per_app = 8 * a.m + 4 + (-2 if zd else 2 + (1 if site else 0))
    napp = 4 if a.backend == "rk4" else a.order
    return float(per_app * napp + (4 * 4 if a.backend == "rk4" else 0))


def measured_peak_fp64(torch, n=8192):
    x = torch.randn(n, n, dtype=torch.float64, device="cuda")
    y = torch.randn(n, n, dtype=torch.float64, device="cuda")
    best = float("inf")
    for _ in range(4):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        x @ y
        s1.record()
        torch.cuda.synchronize()
        best = min(best, s0.elapsed_time(s1))
    del x, y
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def traffic_key(m, n, target, backend, order, exact):
    integ = "rk4" if backend == "rk4" else f"taylor{order}"
    return f"m{m}_n{n}_{target}_{integ}_{'exact' if exact else 'fma'}"


def ncu_traffic(key):
    """DRAM bytes per realization-step of the kernel from a committed
    ``ncu --set full`` capture (profiles/traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get("entries", {}).get(key)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# GPU arm


def make_config(p, a, R_total, steps, local, n=None, m=None, target=None, dt=None):
    n = a.n if n is None else n
    m = a.m if m is None else m
    target = a.target if target is None else target
    dt = a.dt if dt is None else dt
    obs = ("populations", "position_mean_variance", "participation_ratio")
    post = steps if a.post_rate <= 0 else a.post_rate
    return p.RunConfig(space=p.JointSpace(p.build_lattice([n]), m),
                       noise=p.NoiseSpec(target=target, levels=(-0.1, 0.1), rate=a.rate),
                       stepper=p.StepperConfig(backend=a.backend, dt=dt, taylor_order=a.order),
                       realizations=R_total, steps=steps, post_rate=post, precision="double",
                       observables=obs, memory_budget=176 * 2**30, exact=bool(a.exact), device=local)


def enqueue_schedule(engine, cfg, ens, first, steps, torch, group=None):
    """Enqueue ``steps`` steps from global step ``first`` with the
    collection points of cfg's schedule, the way run() does them
    (engine._fused_groups: ctqw_evolve_observe per group of points, one
    all-reduce of the point limbs, ctqw_observe_points).  Returns the last
    group's (out, diag) device buffers."""
    out = diag = None
    for start, targets in engine._fused_groups(cfg):
        if targets[-1] > steps:
            break
        out, diag, _ = engine.enqueue_group(cfg, ens, first + start, [first + t for t in targets], group)
    return out, diag


def timed_segment(engine, cfg, ens, first, steps, post_rate, torch, group=None):
    """Device time (ms) of ``steps`` steps with the collection points of the
    schedule (every post_rate steps, and at the end)."""
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record()
    enqueue_schedule(engine, cfg, ens, first, steps, torch, group)
    stats = ens.stats()
    stop.record()
    torch.cuda.synchronize()
    return start.elapsed_time(stop), stats


def secondary_line(p, engine, a, local, world, torch, barrier, all_max, group):
    """configs[1] (N=256, R=1000 per GPU, tunnelling, Taylor-4): device-timed."""
    R = 1000 * world
    rank = int(os.environ.get("RANK", "0"))
    from paper_1612_00746_b200 import sharding

    cfg = make_config(p, a, R, a.steps, local, n=256, m=2, target="tunneling", dt=0.02)
    lo, hi = sharding.shard_bounds(R, world, rank)
    ens = engine.EnsembleState(cfg, local, lo, hi)
    for k in range(a.warmup):
        ens.evolve(k, 1)
    ens.stats()
    torch.cuda.synchronize()
    ens.handle.kernel_timing(True)
    barrier()
    ms, _ = timed_segment(engine, cfg, ens, a.warmup, a.steps, 0, torch, group)
    kms, kl = ens.handle.kernel_time()
    ens.handle.kernel_timing(False)
    ms = all_max(ms)
    kavg = kms / max(kl, 1)
    peak, _ = measured_peak_hbm()
    achieved = (hi - lo) * 32.0 * 65536 / (kavg / 1000.0) / 1e9
    kernel = ens.handle.step_kernel()
    del ens
    torch.cuda.empty_cache()
    return {"workload": PRESETS[1]["label"] + " | Taylor-4, dt=0.02, FMA stencil, one collection point",
            "value": R * a.steps / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms / a.steps,
            "roofline": {"bound": "hbm", "kernel": kernel, "kernel_ms_avg": kavg, "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak}}


def resident_line(p, engine, a, local, world, torch, barrier, all_max, group):
    """configs[0] (N=64, R=100 per GPU, tunnelling, Taylor-4, 1500 steps with a
    collection point every 10 steps, diagonal observables): the resident64
    kernel with the collection fused in, against its FP64 roofline (cuBLAS
    DGEMM measured here)."""
    import dataclasses

    R, steps, post = 100 * world, 1500, 10
    rank = int(os.environ.get("RANK", "0"))
    from paper_1612_00746_b200 import sharding

    cfg = make_config(p, a, R, steps, local, n=64, m=2, target="tunneling", dt=0.02)
    cfg = dataclasses.replace(cfg, post_rate=post)
    lo, hi = sharding.shard_bounds(R, world, rank)
    ens = engine.EnsembleState(cfg, local, lo, hi)
    enqueue_schedule(engine, cfg, ens, 0, steps, torch, group)  # warm: allocations, first launches
    ens.stats()
    torch.cuda.synchronize()
    ens.handle.kernel_timing(True)
    barrier()
    ms, _ = timed_segment(engine, cfg, ens, steps, steps, post, torch, group)
    kms, kl = ens.handle.kernel_time()
    ens.handle.kernel_timing(False)
    ms = all_max(ms)
    kernel = ens.handle.step_kernel()
    del ens
    torch.cuda.empty_cache()
    flops = (hi - lo) * 4096 * fp64_flops_per_amplitude_step(argparse.Namespace(
        m=2, target="tunneling", backend="taylor", order=4)) * steps
    achieved = flops / (kms / 1000.0) / 1e12
    fpeak = measured_peak_fp64(torch)
    return {"workload": PRESETS[0]["label"] + " | Taylor-4, dt=0.02, FMA stencil, 1500 steps, diagonal observables "
                                               "every 10 steps (fused into the step kernel)",
            "value": R * steps / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms / steps,
            "roofline": {"bound": "fp64", "kernel": kernel, "kernel_ms_total": kms, "kernel_launches": kl,
                         "achieved": achieved, "peak": fpeak, "unit": "TFLOP/s", "frac": achieved / fpeak,
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run",
                         "sm_fill": min(1.0, (hi - lo) / 148.0),
                         "note": "one CTA per realization: 100 realizations occupy 100 of 148 SMs; state on chip "
                                 "for the whole segment, HBM only at segment ends; ncu FP64 pipe 50-54 % on the "
                                 "busy SMs (profiles/r02c, r02h)"}}


def ours(a):
    # the JSON line is the only thing on stdout: libraries that print there
    # (NCCL's version banner at communicator init, ...) go to stderr
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    import torch
    import torch.distributed as dist

    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import engine, sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
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
    elif local >= torch.cuda.device_count():
        print(f"bench.py: rank {rank} needs cuda:{local} but only {torch.cuda.device_count()} GPU(s)",
              file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    if distributed:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    group = dist.group.WORLD if distributed else None
    R_total = a.realizations * world
    cfg = make_config(p, a, R_total, a.steps, local)
    lo, hi = sharding.shard_bounds(R_total, world, rank)
    ens = engine.EnsembleState(cfg, local, lo, hi)
    h = ens.handle
    dim = a.n ** a.m

    def barrier():
        if distributed:
            dist.barrier()

    def all_max(*vals):
        t = torch.tensor(list(vals), dtype=torch.float64, device=f"cuda:{local}")
        if distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out = [float(v) for v in t.tolist()]
        return out[0] if len(out) == 1 else out

    # warm-up (includes collection points): the last warm-up step goes
    # through evolve_observe, and the point reduction's scratch is sized for
    # the largest group of the timed schedule
    for k in range(a.warmup - 1):
        ens.evolve(k, 1)
        ens.stats()
    engine.collect_observables(cfg, ens, group)
    max_pts = max(len(t) for _, t in engine._fused_groups(cfg))
    wacc = torch.zeros((max_pts, 3, dim), dtype=torch.int64, device=ens.dev)
    ens.evolve_observe(a.warmup - 1, 1, 1, wacc[:1])
    wout = torch.empty((max_pts, a.n + 3), dtype=torch.float64, device=ens.dev)
    wdiag = torch.empty((max_pts, dim), dtype=torch.float64, device=ens.dev)
    ens.handle.observe_points(wacc, max_pts, float(R_total), wout, wdiag)
    ens.stats()
    del wacc, wout, wdiag
    torch.cuda.synchronize()

    # timed region: K steps + the collection point(s), device-timed
    h.kernel_timing(True)
    launches0 = h.launches
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record()
        out, _ = enqueue_schedule(engine, cfg, ens, a.warmup, a.steps, torch, group)
        stats = ens.stats()
        stop.record()
        torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(stop)
    kernel_ms, kernel_launches = h.kernel_time()
    kernel = h.step_kernel()
    h.kernel_timing(False)
    launches = h.launches - launches0
    assert stats["failure"] is None
    assert abs(float(out[-1, : a.n].sum()) - a.m) < 4 * a.m * 1e-6  # within the norm policy tol_norm

    ms_other = None
    if not a.no_other:
        # the other arithmetic mode on the same states (reported beside the headline)
        ens.stepper = cfg.stepper.native(not a.exact)
        ens.evolve(a.warmup + a.steps, 2)
        barrier()
        torch.cuda.synchronize()
        ms_other, _ = timed_segment(engine, cfg, ens, a.warmup + a.steps + 2, a.steps, a.post_rate, torch, group)
        ens.stepper = cfg.stepper.native(bool(a.exact))
    ms_max, ms_other_max = all_max(ms, ms_other if ms_other is not None else 0.0)
    value = R_total * a.steps / (ms_max / 1000.0)

    # roofline of the dominant kernel (streaming step / resident segment)
    avg_launch_ms = kernel_ms / max(kernel_launches, 1)
    steps_per_launch = 1
    if kernel.startswith("resident"):
        steps_per_launch = a.steps // max(kernel_launches, 1)  # one launch covers a whole segment
    bytes_per_launch = (hi - lo) * 32.0 * dim * steps_per_launch
    achieved = bytes_per_launch / (avg_launch_ms / 1000.0) / 1e9
    peak, peak_src = measured_peak_hbm()
    tr = ncu_traffic(traffic_key(a.m, a.n, a.target, a.backend, a.order, a.exact))
    traffic_bytes = None
    if tr and tr.get("kernel") == kernel:
        # ncu --set full capture (profiles/), per realization-step, scaled to this launch
        traffic_bytes = tr["dram_bytes_per_realization_step"] * (hi - lo) * steps_per_launch
    flops_unit = fp64_flops_per_amplitude_step(a)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "frac_of_spec_8000": achieved / 8000.0, "traffic": traffic_bytes,
                "traffic_source": tr.get("source") if traffic_bytes else None,
                "kernel": kernel,
                "kernel_ms_avg": avg_launch_ms, "kernel_launches": kernel_launches,
                "kernel_share_of_step": kernel_ms / ms if ms > 0 else None,
                "algorithmic_bytes_per_unit": 32.0 * dim, "units_per_launch": (hi - lo) * steps_per_launch,
                "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_src,
                "flops_per_launch": (hi - lo) * dim * flops_unit * steps_per_launch}
    roofline["achieved_fp64_tflops"] = roofline["flops_per_launch"] / (avg_launch_ms / 1000.0) / 1e12
    if kernel.startswith("resident"):
        # the resident kernel touches HBM only at segment ends: its roofline
        # is the FP64 pipe (with shared memory beside it, ncu in profiles/)
        fpeak = measured_peak_fp64(torch)
        hbm_equiv = {k: roofline[k] for k in ("bound", "achieved", "peak", "unit", "frac")}
        hbm_equiv["note"] = "bytes a streaming kernel would move per step; the resident kernel keeps the state on chip"
        roofline.update({"bound": "fp64", "achieved": roofline["achieved_fp64_tflops"], "peak": fpeak,
                         "unit": "TFLOP/s", "frac": roofline["achieved_fp64_tflops"] / fpeak,
                         "peak_source": "measured in this run: cuBLAS DGEMM 8192^3 (torch float64 matmul, best of 3)",
                         "hbm_equivalent": hbm_equiv, "traffic": None})
    del ens, out
    torch.cuda.empty_cache()

    # e2e through the public API: run(config) with host I/O
    e2e = None
    if not a.no_e2e:
        sinks = p.MemorySinks(keep_densities=False)
        # one untimed run() first, as the device arm's warm-up steps: the
        # allocator then serves this run's buffers from its cache
        warm = make_config(p, a, R_total, max(a.warmup, 1), local)
        p.run(warm, p.MemorySinks(keep_densities=False), group=group)
        gc.collect()
        torch.cuda.synchronize()
        barrier()
        prof = None
        if os.environ.get("CTQW_E2E_PROFILE"):
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        # three full end-to-end runs, the median reported (each one a complete
        # run(): host upload, noise, K steps, collection, rows to the host)
        walls = []
        for _ in range(3):
            sinks = p.MemorySinks(keep_densities=False)
            barrier()
            t0 = time.perf_counter()
            rep = p.run(cfg, sinks, group=group)
            torch.cuda.synchronize()
            walls.append(all_max(time.perf_counter() - t0))
            del rep
            gc.collect()
        e2e_s = statistics.median(walls)
        if prof is not None:
            import pstats

            prof.disable()
            pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(12)
        n_points = len(cfg.schedule)
        h2d = dim * 16 + 16  # initial state + noise levels
        d2h = (a.n + 4) * 8 * n_points + 48 * n_points  # observable rows + segment statistics per point
        e2e = {"value": R_total * a.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d / a.steps, "d2h_bytes_per_step": d2h / a.steps,
               "seconds": e2e_s, "seconds_all_runs": walls, "collection_points": n_points, "rows": len(sinks.rows),
               "api": "paper_1612_00746_b200.run(RunConfig, MemorySinks)",
               "includes": "initial-state H2D, device noise draw + coefficient build, K steps with the norm "
                           "policy, collection point(s), observable rows D2H, run() bookkeeping; median of 3 runs"}
        torch.cuda.empty_cache()

    secondary = None
    if not a.no_secondary and a.config == 2 and not a.custom:
        secondary = [secondary_line(p, engine, a, local, world, torch, barrier, all_max, group),
                     resident_line(p, engine, a, local, world, torch, barrier, all_max, group)]

    cpu = None  # the host-core baseline is taken on rank 0 at N = 1 only
    if rank == 0 and world == 1 and not a.no_cpu:
        rate, pool, wall, sample = pool_rate(a)
        cpu = dict({"value": rate, "unit": UNIT, "kind": pool.kind, "sample": sample}, **cores_info(pool.workers))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": data_label(a),
            "config": dict(workload_config(a), parallelism=f"realizations sharded over {world} GPU(s)"),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "other_arithmetic": None if ms_other is None else {
                "exact_order": not a.exact, "value": R_total * a.steps / (ms_other_max / 1000.0),
                "ms_per_step": ms_other_max / a.steps},
            "secondary": secondary,
            "clocks": clocks.summary(),
            "norm_events": stats["event_count"],
        }
        print(json.dumps(line), file=json_out, flush=True)
    if distributed:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(a):
    """``--gpus N`` outside torchrun: one process per GPU via torch.distributed.run."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only the JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    return subprocess.call(cmd + sys.argv[1:], env=env)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(a))
    if a.impl == "reference":
        reference_arm(a)
    else:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only the JSON line
        ours(a)


if __name__ == "__main__":
    main()
