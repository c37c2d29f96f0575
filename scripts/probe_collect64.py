"""Probe: where the configs[0] collection cost goes (resident64 fused
collection vs the point reductions), device-timed per group of 100 steps."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1612_00746_b200 as p
from paper_1612_00746_b200 import engine

R, n = 100, 64
cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), 2), noise=p.NoiseSpec(target="tunneling", levels=(-0.1, 0.1), rate=0.0),
                  stepper=p.StepperConfig(backend="taylor", dt=0.02), realizations=R, steps=300, post_rate=10,
                  precision="double", observables=("populations", "position_mean_variance", "participation_ratio"),
                  exact=False, device=0)
ens = engine.EnsembleState(cfg, 0, 0, R)
ens.evolve(0, 2); ens.stats()
dim = n * n
print(ens.handle.step_kernel(), ens.handle.step_variant(), file=sys.stderr)
import time
t0 = time.time()
while time.time() - t0 < 3.0:  # let the clocks ramp up
    ens.evolve(0, 100)
    torch.cuda.synchronize()
ens.stats()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); ens.evolve(0, 100); e1.record(); torch.cuda.synchronize()
    print("evolve 100 steps us", e0.elapsed_time(e1) * 1e3, file=sys.stderr)
ens.stats()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
out = {}
for post in (100, 10, 1):
    P = 100 // post
    acc = torch.zeros((P, 3, dim), dtype=torch.int64, device="cuda:0")
    o = torch.empty((P, n + 3), dtype=torch.float64, device="cuda:0")
    dg = torch.empty((P, dim), dtype=torch.float64, device="cuda:0")
    for rep in range(3):
        torch.cuda.synchronize()
        ev[0].record()
        ens.evolve_observe(0, 100, post, acc)
        ev[1].record()
        ens.handle.observe_points(acc, P, float(R), o, dg)
        ev[2].record()
        torch.cuda.synchronize()
    ens.stats()
    out[post] = (ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3)
    print(json.dumps({"post": post, "points": P, "evolve_observe_us": out[post][0], "observe_points_us": out[post][1]}))
