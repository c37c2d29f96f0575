"""Probe: can the SMs plane3's 16-CTA clusters leave idle (148 - 112) do
useful m=3 work concurrently?  Times plane3 alone, the generic per-application
kernels alone, and both on two streams at once (configs[4] shape, N=128).

    python scripts/probe_m3_fill.py [RA] [RB] [steps]
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import engine

    ra = int(sys.argv[1]) if len(sys.argv) > 1 else 112
    rb = int(sys.argv[2]) if len(sys.argv) > 2 else 36
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2

    def cfg(R):
        return p.RunConfig(space=p.JointSpace(p.build_lattice([128]), 3),
                           noise=p.NoiseSpec(target="tunneling", levels=(-0.1, 0.1)),
                           stepper=p.StepperConfig(backend="taylor", dt=0.02), realizations=R, steps=steps,
                           post_rate=steps, precision="double", observables=("populations",),
                           memory_budget=175 * 2**30, exact=False, device=0)

    os.environ.pop("CTQW_STREAM", None)
    ea = engine.EnsembleState(cfg(ra), 0, 0, ra)
    os.environ["CTQW_STREAM"] = "generic"
    eb = engine.EnsembleState(cfg(rb), 0, 0, rb)
    os.environ.pop("CTQW_STREAM", None)
    for e in (ea, eb):
        e.evolve(0, 1)
        e.stats()
    print("kernels:", ea.handle.step_kernel(), eb.handle.step_kernel(), file=sys.stderr)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

    def run(which):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if "a" in which:
            with torch.cuda.stream(sa):
                ea.evolve(1, steps)
        if "b" in which:
            with torch.cuda.stream(sb):
                eb.evolve(1, steps)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    out = {}
    for which in ("a", "b", "ab", "a", "b", "ab"):
        out[which] = run(which)
    ta, tb, tab = out["a"], out["b"], out["ab"]
    print(json.dumps({"ra": ra, "rb": rb, "steps": steps, "t_a": ta, "t_b": tb, "t_ab": tab,
                      "a_rate": ra * steps / ta, "b_rate": rb * steps / tb,
                      "ab_rate": (ra + rb) * steps / tab}))


if __name__ == "__main__":
    main()
