"""Throughput sweep over the BASELINE.json configurations (one GPU).

    python scripts/sweep.py [--quick]

Prints one JSON line per case: realization·steps/s of K steps (device-timed
with CUDA events, states resident in HBM) plus, where the case has a
collection cadence, the same with the observable reduction at every
post_rate-th step, so the post-processing cost is visible (configs[3]).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as _f:
        PEAK = float(json.load(_f)["hbm_gbs"]) * 1e9
except Exception:
    PEAK = 6544e9
ONLY = ""


def timed(ens, cfg, steps, post_rate, engine, torch):
    """Device seconds of ``steps`` steps with a collection point every
    ``post_rate`` steps, the way run() schedules them: the batched path
    (ctqw_evolve_observe + ctqw_observe_points, bench.enqueue_schedule;
    with purity, one evolve_observe per segment plus the overlap kernel)."""
    import dataclasses

    import bench

    c = dataclasses.replace(cfg, steps=steps, post_rate=post_rate)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    bench.enqueue_schedule(engine, c, ens, 0, steps, torch)
    stop.record()
    torch.cuda.synchronize()
    st = ens.stats()
    assert st["failure"] is None, st["failure"]
    return start.elapsed_time(stop) / 1000.0


def run_case(name, m, n, R, steps, backend="taylor", dt=0.02, target="tunneling", post_rates=(None,), rate=0.0,
             observables=("populations", "position_mean_variance", "participation_ratio")):
    if ONLY and ONLY not in name:
        return
    import torch

    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import engine

    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), m),
                      noise=p.NoiseSpec(target=target, levels=(-0.1, 0.1), rate=rate),
                      stepper=p.StepperConfig(backend=backend, dt=dt), realizations=R, steps=steps,
                      post_rate=steps, precision="double", observables=observables,
                      memory_budget=175 * 2**30, exact=False, device=0)
    ens = engine.EnsembleState(cfg, 0, 0, R)
    ens.evolve(0, 2)
    ens.stats()
    engine.collect_observables(cfg, ens)
    out = []
    for ex in (False, True):  # FMA-contracted, then exact reference order
        ens.stepper = cfg.stepper.native(ex)
        ens.evolve(0, 1)
        for pr in post_rates:
            prate = steps if pr is None else pr
            timed(ens, cfg, steps, prate, engine, torch)  # untimed: allocator, scratch, first launches
            secs = timed(ens, cfg, steps, prate, engine, torch)
            thr = R * steps / secs
            line = {"case": name, "m": m, "n": n, "realizations": R, "steps": steps, "backend": backend,
                    "post_rate": prate, "exact": ex, "seconds": secs, "r_steps_per_s": thr, "noise_rate": cfg.noise.rate,
                    "kernel": ens.handle.step_kernel(),
                    "hbm_frac_of_measured": thr * 32.0 * n ** m / PEAK}
            print(json.dumps(line), flush=True)
            out.append(line)
    del ens
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="", help="run only the cases whose name contains this")
    a = ap.parse_args()
    q = a.quick
    global ONLY
    ONLY = a.only
    # configs[0]: N=64, 100 realizations (resident kernel), Taylor, post every 10 steps
    run_case("configs[0] N=64 R=100", 2, 64, 100, 300 if q else 1500, post_rates=(10, None),
             observables=("populations", "position_mean_variance", "purity", "participation_ratio"))
    run_case("configs[0] N=64 R=100 diag observables", 2, 64, 100, 300 if q else 1500, post_rates=(10, None))
    run_case("N=64 R=1000", 2, 64, 1000, 300 if q else 1500)
    # configs[1]: N=256, 1000 realizations, Taylor vs RK4
    for backend in ("taylor", "rk4"):
        run_case(f"configs[1] N=256 R=1000 {backend}", 2, 256, 1000, 50 if q else 200, backend=backend)
    # configs[2]: N=1024, on-site + tunnelling noise, 1250 realizations per GPU (10^4 over 8)
    run_case("configs[2] N=1024 R=1250 both", 2, 1024, 1250, 10 if q else 40, target="both")
    # configs[3]: N=512, post-processing frequency sweep
    run_case("configs[3] N=512 R=1000 post sweep", 2, 512, 1000, 100 if q else 1000,
             post_rates=(1, 10, 100, None) if not q else (1, 10, None))
    # the reference's CLI default noise: dynamic telegraph switching at rate 0.1
    run_case("configs[1] N=256 R=1000 telegraph rate=0.1", 2, 256, 1000, 50 if q else 200, rate=0.1)
    # configs[4]: m=3, N=128 (D=2^21), 16-CTA cluster kernel; the largest ensemble that fits
    # (one 32 MiB buffer per realization: the kernel marches in place) is ~5300 per GPU
    run_case("configs[4] m=3 N=128 R=5300 (in place)", 3, 128, 5300, 3 if q else 10, dt=0.015)


if __name__ == "__main__":
    main()
