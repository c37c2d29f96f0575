"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck):  compute-sanitizer --tool racecheck python scripts/sanitize.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1612_00746_b200 as p  # noqa: E402


def run(m, n, R, steps, backend="taylor", rate=0.0, target="both", lattice=None, stream=None):
    if stream:
        os.environ["CTQW_STREAM"] = stream
    else:
        os.environ.pop("CTQW_STREAM", None)
    lat = lattice or p.build_lattice([n])
    cfg = p.RunConfig(space=p.JointSpace(lat, m), model=p.CouplingModel(onsite_energy=0.1, interaction=0.3),
                      noise=p.NoiseSpec(target=target, rate=rate), stepper=p.StepperConfig(backend=backend, dt=0.05),
                      realizations=R, steps=steps, post_rate=steps, precision="double",
                      observables=("populations", "participation_ratio"))
    sinks = p.MemorySinks()
    p.run(cfg, sinks)
    print(m, n, R, backend, rate, stream, "rows", len(sinks.rows), "ok", flush=True)


def gram():
    import torch

    from paper_1612_00746_b200 import density

    rng = np.random.default_rng(3)
    stack = torch.as_tensor(rng.normal(size=(5, 70)) + 1j * rng.normal(size=(5, 70)), device="cuda:0")
    density.packed_density_device(stack, 5)
    torch.cuda.synchronize()
    print("packed_gram ok", flush=True)


def run_posts(m, n, R, steps, post, backend="taylor", rate=0.0, dt=0.05):
    """run() on the batched schedule: evolve_observe (fused on resident64),
    observe_points, segment events."""
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), m), model=p.CouplingModel(onsite_energy=0.1),
                      noise=p.NoiseSpec(target="both", rate=rate), stepper=p.StepperConfig(backend=backend, dt=dt),
                      realizations=R, steps=steps, post_rate=post, precision="double",
                      observables=("populations", "participation_ratio", "joint_distribution"))
    sinks = p.MemorySinks()
    p.run(cfg, sinks)
    print(m, n, R, backend, "post", post, "rows", len(sinks.rows), "events", len(sinks.events), "ok", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["band4", "resident", "generic", "telegraph", "lattice", "plane3", "resident64",
                             "gram", "points"]
    if "resident64" in which:
        run(2, 64, 2, 3)
        run(2, 64, 2, 3, "rk4")
        run_posts(2, 64, 2, 9, 3, dt=0.12)  # fused collection, with renormalisations
    if "gram" in which:
        gram()
    if "points" in which:
        run_posts(2, 96, 2, 6, 2)
    if "band4" in which:
        run(2, 96, 3, 3)
        run(2, 256, 2, 2, "rk4")
    if "band4split" in which:  # N = 1024: the split-phase row barrier
        run(2, 1024, 2, 2)
        run(2, 1024, 2, 2, "rk4")
    if "resident" in which:
        run(2, 32, 3, 4)
    if "generic" in which:
        run(3, 10, 2, 3)
    if "telegraph" in which:
        run(2, 96, 2, 3, rate=2.0)
    if "lattice" in which:
        run(2, 12, 2, 2, lattice=p.build_lattice([3, 4], boundary="open"))
    if "plane3" in which:
        run(3, 128, 1, 2)
