"""Generate golden fixtures from the REFERENCE package (run in the build container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports ``ctqw`` read-only from ``/root/reference/pkg/src`` and stores its own
outputs (noise draws, apply/step results, segment stats, ``run()`` observable
rows) as small ``.npz`` fixtures.  Nothing on the GPU box reads
``/root/reference``; the tests read only these committed files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from ctqw.ensemble import (  # noqa: E402
    InitialStateSpec,
    MemorySinks,
    RunConfig,
    _ChunkState,
    _evolve_segment,
    _WorkerContext,
    run,
)
from ctqw.errors import NormFailureError  # noqa: E402
from ctqw.hamiltonian import CouplingModel, apply_values, assemble_values  # noqa: E402
from ctqw.hilbert import JointSpace, build_lattice, build_topology  # noqa: E402
from ctqw.noise import NoiseSpec, init_process  # noqa: E402
from ctqw.propagators import (  # noqa: E402
    StepperConfig,
    check_norm_stack,
    step_rk4_values,
    step_taylor_values,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def noise_fixture():
    cases = []
    arrays = {}
    k = 0
    for target, levels, n in (
        ("tunneling", (-0.1, 0.1), 64),
        ("both", (-0.1, 0.1), 16),
        ("onsite", (-0.3, 0.0, 0.3), 12),
        ("both", (0.25,), 10),
        ("both", (-1.0, -0.5, 0.5, 1.0, 2.0), 9),
    ):
        spec = NoiseSpec(target=target, levels=levels, rate=0.0)
        lat = build_lattice([n])
        for seed in (1234, 7, 2**33 + 5):
            for r in (0, 1, 5, 99, 4097):
                proc = init_process(spec, lat, seed=(seed, r))
                arrays[f"v{k}"] = proc.values
                cases.append(dict(key=f"v{k}", target=target, levels=list(levels), n=n,
                                  seed=seed, r=r, n_links=proc.n_links, n_sites=proc.n_sites))
                k += 1
    np.savez_compressed(os.path.join(HERE, "noise_draws.npz"), meta=json.dumps(cases), **arrays)


def stencil_fixture():
    """apply / Taylor / RK4 single steps on random noisy instances (m = 1, 2, 3)."""
    rng = np.random.default_rng(20261017)
    arrays = {}
    meta = []
    for idx, (n, m, b) in enumerate(((9, 1, 3), (7, 2, 2), (12, 2, 3), (5, 3, 2), (6, 3, 1))):
        space = JointSpace(lattice=build_lattice([n]), m=m)
        topo = build_topology(space)
        model = CouplingModel(onsite_energy=float(rng.uniform(-1, 1)),
                              tunneling=float(rng.uniform(0.5, 1.5)),
                              interaction=float(rng.uniform(0, 2)), hbar=1.3)
        link = 0.3 * rng.normal(size=(b, n))
        site = 0.3 * rng.normal(size=(b, n))
        values = assemble_values(topo, model, link_values=link, site_values=site)
        psi = rng.normal(size=(b, space.dim)) + 1j * rng.normal(size=(b, space.dim))
        psi /= np.linalg.norm(psi, axis=1, keepdims=True)
        dt = 0.05
        arrays[f"link{idx}"] = link
        arrays[f"site{idx}"] = site
        arrays[f"psi{idx}"] = psi
        arrays[f"apply{idx}"] = apply_values(topo, values, psi)
        arrays[f"taylor4_{idx}"] = step_taylor_values(topo, values, psi, dt, hbar=model.hbar, order=4)
        arrays[f"taylor7_{idx}"] = step_taylor_values(topo, values, psi, dt, hbar=model.hbar, order=7)
        arrays[f"rk4_{idx}"] = step_rk4_values(topo, values, psi, dt, hbar=model.hbar)
        # tunnelling-only assembly (site noise absent)
        values_t = assemble_values(topo, model, link_values=link)
        arrays[f"taylor4t_{idx}"] = step_taylor_values(topo, values_t, psi, dt, hbar=model.hbar, order=4)
        meta.append(dict(n=n, m=m, b=b, onsite=model.onsite_energy, tunneling=model.tunneling,
                         interaction=model.interaction, hbar=model.hbar, dt=dt))
    np.savez_compressed(os.path.join(HERE, "stencil_steps.npz"), meta=json.dumps(meta), **arrays)


def segment_fixture():
    """Reference ``_evolve_segment`` with renormalisation events (dt large)."""
    arrays = {}
    meta = []
    cases = (
        dict(n=8, m=2, b=5, backend="taylor", order=4, dt=0.05, steps=60, target="both"),
        dict(n=8, m=2, b=4, backend="rk4", order=4, dt=0.05, steps=60, target="tunneling"),
        dict(n=6, m=3, b=3, backend="taylor", order=4, dt=0.04, steps=40, target="both"),
        dict(n=16, m=1, b=4, backend="taylor", order=3, dt=0.1, steps=50, target="onsite"),
        dict(n=10, m=2, b=3, backend="taylor", order=4, dt=0.02, steps=80, target="both"),
    )
    for idx, c in enumerate(cases):
        space = JointSpace(lattice=build_lattice([c["n"]]), m=c["m"])
        topo = build_topology(space)
        model = CouplingModel(onsite_energy=0.2, tunneling=1.0, interaction=0.7)
        stepper = StepperConfig(backend=c["backend"], dt=c["dt"], taylor_order=c["order"])
        spec = NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=0.0)
        noise = [init_process(spec, topo, seed=(1234, r)) for r in range(c["b"])]
        start = (c["n"] - c["m"]) // 2
        psi0 = np.zeros(space.dim, dtype=np.complex128)
        j = 0
        for x in range(start, start + c["m"]):
            j = j * c["n"] + x
        psi0[j] = 1.0
        chunk = _ChunkState(r0=0, psi=np.tile(psi0, (c["b"], 1)), noise=noise)
        ctx = _WorkerContext(topology=topo, model=model, stepper=stepper,
                             dtype_name="complex128", dense_cap=4096)
        chunk, stats = _evolve_segment(ctx, chunk, 0, c["steps"])
        arrays[f"psi{idx}"] = chunk.psi
        arrays[f"ev{idx}"] = np.array([[e.deviation, float(e.corrected), e.realization, e.step]
                                       for e in stats.events]).reshape(-1, 4)
        meta.append(dict(c, onsite=0.2, tunneling=1.0, interaction=0.7, seed=1234,
                         event_count=stats.event_count, corrections=stats.corrections,
                         max_deviation=stats.max_deviation))
    # a norm failure: huge dt, no renormalisation (test_ensemble.py:359-370 style)
    space = JointSpace(lattice=build_lattice([9]), m=2)
    topo = build_topology(space)
    model = CouplingModel()
    stepper = StepperConfig(dt=0.6, renormalize=False)
    spec = NoiseSpec(target="both", levels=(-0.4, 0.4), rate=0.0)
    noise = [init_process(spec, topo, seed=(99, r)) for r in range(4)]
    psi0 = np.zeros(space.dim, dtype=np.complex128)
    psi0[3 * 9 + 4] = 1.0
    chunk = _ChunkState(r0=0, psi=np.tile(psi0, (4, 1)), noise=noise)
    ctx = _WorkerContext(topology=topo, model=model, stepper=stepper,
                         dtype_name="complex128", dense_cap=4096)
    fail = None
    try:
        _evolve_segment(ctx, chunk, 0, 50)
    except NormFailureError as exc:
        fail = dict(realization=exc.realization, step=exc.step, deviation=exc.deviation)
    np.savez_compressed(os.path.join(HERE, "segments.npz"), meta=json.dumps(meta),
                        failure=json.dumps(fail), **arrays)


def run_fixture():
    """Reference ``run()`` observable rows (dense-rho path, small sizes)."""
    arrays = {}
    meta = []
    cases = (
        dict(n=10, m=2, R=6, steps=30, post_rate=10, backend="taylor", dt=0.05, target="both",
             observables=None, initial="auto"),
        dict(n=12, m=2, R=5, steps=25, post_rate=7, backend="rk4", dt=0.04, target="tunneling",
             observables=("populations", "position_mean_variance", "purity",
                          "participation_ratio", "joint_distribution"), initial="auto"),
        dict(n=6, m=3, R=4, steps=12, post_rate=4, backend="taylor", dt=0.03, target="onsite",
             observables=None, initial="auto"),
        dict(n=9, m=2, R=3, steps=20, post_rate=20, backend="taylor", dt=0.05, target="tunneling",
             observables=None, initial="antisymmetrized_pair"),
        dict(n=11, m=1, R=4, steps=15, post_rate=5, backend="taylor", dt=0.05, target="both",
             observables=None, initial="auto"),
    )
    for idx, c in enumerate(cases):
        space = JointSpace(lattice=build_lattice([c["n"]]), m=c["m"])
        cfg = RunConfig(
            space=space,
            model=CouplingModel(onsite_energy=0.1, tunneling=1.0, interaction=0.5),
            noise=NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=0.0),
            stepper=StepperConfig(backend=c["backend"], dt=c["dt"]),
            initial=InitialStateSpec(kind=c["initial"]),
            realizations=c["R"], steps=c["steps"], post_rate=c["post_rate"],
            master_seed=1234, workers=1, precision="double",
            observables=c["observables"],
        )
        sinks = MemorySinks()
        report = run(cfg, sinks)
        arrays[f"rows{idx}"] = np.array([r[3] for r in sinks.rows], dtype=np.float64)
        meta.append(dict(c, rows=[(r[0], r[1], r[2]) for r in sinks.rows],
                         onsite=0.1, tunneling=1.0, interaction=0.5,
                         observables_resolved=list(cfg.observables),
                         corrections=report.norm_corrections, norm_events=report.norm_events,
                         max_norm_deviation=report.max_norm_deviation))
    np.savez_compressed(os.path.join(HERE, "run_rows.npz"), meta=json.dumps(meta), **arrays)


def telegraph_fixture():
    """Reference dynamic (telegraph) noise: process states after k advances
    (noise.py:128-206) and ``run()`` rows/switch counts with rate > 0."""
    from ctqw.noise import advance

    arrays = {}
    meta = {"trajectories": [], "runs": []}
    traj = (
        dict(n=12, target="both", levels=(-0.1, 0.1, 0.3), rate=0.7, seed=1234, r0=5, count=3, dt=0.05,
             checkpoints=(0, 1, 7, 40)),
        dict(n=20, target="tunneling", levels=(-0.2, 0.2), rate=2.5, seed=99, r0=0, count=2, dt=0.13,
             checkpoints=(3, 25)),
    )
    for ti, c in enumerate(traj):
        spec = NoiseSpec(target=c["target"], levels=c["levels"], rate=c["rate"])
        lat = build_lattice([c["n"]])
        procs = [init_process(spec, lat, seed=(c["seed"], r)) for r in range(c["r0"], c["r0"] + c["count"])]
        done = 0
        for k in c["checkpoints"]:
            for _ in range(k - done):
                for pr in procs:
                    advance(pr, c["dt"])
            done = k
            arrays[f"traj{ti}_values_{k}"] = np.stack([pr.values for pr in procs])
            arrays[f"traj{ti}_next_{k}"] = np.stack([pr.next_switch for pr in procs])
            arrays[f"traj{ti}_time_{k}"] = np.array([pr.time for pr in procs])
            arrays[f"traj{ti}_switches_{k}"] = np.array([pr.switch_count for pr in procs])
        meta["trajectories"].append(dict(c, n_links=procs[0].n_links, n_sites=procs[0].n_sites))
    runs = (
        dict(n=10, m=2, R=5, steps=40, post_rate=10, backend="taylor", dt=0.05, target="both", rate=0.8),
        dict(n=9, m=2, R=4, steps=30, post_rate=15, backend="rk4", dt=0.05, target="tunneling", rate=2.0),
    )
    for idx, c in enumerate(runs):
        space = JointSpace(lattice=build_lattice([c["n"]]), m=c["m"])
        cfg = RunConfig(
            space=space,
            model=CouplingModel(onsite_energy=0.1, tunneling=1.0, interaction=0.5),
            noise=NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=c["rate"]),
            stepper=StepperConfig(backend=c["backend"], dt=c["dt"]),
            realizations=c["R"], steps=c["steps"], post_rate=c["post_rate"],
            master_seed=1234, workers=1, precision="double",
        )
        sinks = MemorySinks()
        report = run(cfg, sinks)
        arrays[f"run{idx}_rows"] = np.array([r[3] for r in sinks.rows], dtype=np.float64)
        meta["runs"].append(dict(c, rows=[(r[0], r[1], r[2]) for r in sinks.rows], onsite=0.1, tunneling=1.0,
                                 interaction=0.5, switch_count=report.switch_count,
                                 corrections=report.norm_corrections, norm_events=report.norm_events))
    np.savez_compressed(os.path.join(HERE, "telegraph.npz"), meta=json.dumps(meta), **arrays)


def lattice_fixture():
    """General lattices (q > 1, k_half > 1, open boundaries; hilbert.py:189-359):
    apply / Taylor-4 / RK4 steps on noisy instances, and run() rows."""
    rng = np.random.default_rng(4242)
    arrays = {}
    meta = {"steps": [], "runs": []}
    cases = (
        dict(dims=[3, 4], k_half=[1, 1], boundary="periodic", m=2, b=2, tunneling=1.0),
        dict(dims=[8], k_half=[1], boundary="open", m=1, b=3, tunneling=1.0),
        dict(dims=[7], k_half=[1], boundary="open", m=2, b=2, tunneling=0.9),
        dict(dims=[9], k_half=[2], boundary="periodic", m=2, b=2, tunneling=1.1),
        dict(dims=[4, 3], k_half=[1, 1], boundary="open", m=2, b=2, tunneling=[1.0, 0.7]),
        dict(dims=[3, 3], k_half=[1, 1], boundary="periodic", m=3, b=1, tunneling=[0.8, 1.2]),
        dict(dims=[3, 5], k_half=[1, 2], boundary="open", m=2, b=2, tunneling=[1.0, 0.6]),
    )
    for idx, c in enumerate(cases):
        lat = build_lattice(c["dims"], k_half=c["k_half"], boundary=c["boundary"])
        space = JointSpace(lattice=lat, m=c["m"])
        topo = build_topology(space)
        model = CouplingModel(onsite_energy=0.3, tunneling=c["tunneling"], interaction=0.6, hbar=1.1)
        b, n, nl = c["b"], lat.n_sites, lat.n_sites * lat.moves_half
        link = 0.3 * rng.normal(size=(b, nl))
        site = 0.3 * rng.normal(size=(b, n))
        values = assemble_values(topo, model, link_values=link, site_values=site)
        psi = rng.normal(size=(b, space.dim)) + 1j * rng.normal(size=(b, space.dim))
        psi /= np.linalg.norm(psi, axis=1, keepdims=True)
        dt = 0.04
        arrays[f"link{idx}"] = link
        arrays[f"site{idx}"] = site
        arrays[f"psi{idx}"] = psi
        arrays[f"apply{idx}"] = apply_values(topo, values, psi)
        arrays[f"taylor4_{idx}"] = step_taylor_values(topo, values, psi, dt, hbar=model.hbar, order=4)
        arrays[f"rk4_{idx}"] = step_rk4_values(topo, values, psi, dt, hbar=model.hbar)
        meta["steps"].append(dict(c, onsite=0.3, interaction=0.6, hbar=1.1, dt=dt))
    runs = (
        dict(dims=[3, 4], k_half=[1, 1], boundary="periodic", m=2, R=3, steps=20, post_rate=10, rate=0.0,
             target="both", observables=None),
        dict(dims=[10], k_half=[1], boundary="open", m=2, R=4, steps=24, post_rate=8, rate=0.5,
             target="both", observables=None),
        dict(dims=[11], k_half=[2], boundary="periodic", m=1, R=3, steps=30, post_rate=10, rate=0.0,
             target="tunneling", observables=None),
    )
    for idx, c in enumerate(runs):
        lat = build_lattice(c["dims"], k_half=c["k_half"], boundary=c["boundary"])
        cfg = RunConfig(space=JointSpace(lattice=lat, m=c["m"]),
                        model=CouplingModel(onsite_energy=0.1, tunneling=1.0, interaction=0.5),
                        noise=NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=c["rate"]),
                        stepper=StepperConfig(backend="taylor", dt=0.05), realizations=c["R"], steps=c["steps"],
                        post_rate=c["post_rate"], master_seed=1234, workers=1, precision="double",
                        observables=c["observables"])
        sinks = MemorySinks()
        report = run(cfg, sinks)
        arrays[f"run{idx}_rows"] = np.array([r[3] for r in sinks.rows], dtype=np.float64)
        meta["runs"].append(dict(c, rows=[(r[0], r[1], r[2]) for r in sinks.rows],
                                 observables_resolved=list(cfg.observables), switch_count=report.switch_count,
                                 corrections=report.norm_corrections))
    np.savez_compressed(os.path.join(HERE, "lattices.npz"), meta=json.dumps(meta), **arrays)


def density_fixture():
    """Reference dense <rho>: accumulate_density on a random stack and the
    packed snapshots of a small run() (density.py:57-98)."""
    from ctqw.density import accumulate_density

    rng = np.random.default_rng(2024)
    stack = rng.normal(size=(7, 30)) + 1j * rng.normal(size=(7, 30))
    stack /= np.linalg.norm(stack, axis=1, keepdims=True)
    rho = accumulate_density(stack, time_tag=0.25)
    arrays = {"stack": stack, "packed": rho.packed}
    space = JointSpace(lattice=build_lattice([8]), m=2)
    cfg = RunConfig(space=space, model=CouplingModel(onsite_energy=0.1, tunneling=1.0, interaction=0.5),
                    noise=NoiseSpec(target="both", levels=(-0.1, 0.1), rate=0.5),
                    stepper=StepperConfig(backend="taylor", dt=0.05), realizations=5, steps=12, post_rate=4,
                    master_seed=1234, workers=1, precision="double")
    sinks = MemorySinks()
    run(cfg, sinks)
    meta = {"n": 8, "m": 2, "R": 5, "steps": 12, "post_rate": 4, "dt": 0.05, "rate": 0.5,
            "snapshots": [(d.time_tag, d.sample_count) for d in sinks.densities]}
    for i, d in enumerate(sinks.densities):
        arrays[f"snap{i}"] = d.packed
    np.savez_compressed(os.path.join(HERE, "density.npz"), meta=json.dumps(meta), **arrays)


def config0_fixture():
    """BASELINE configs[0] at full length through the reference's own ``run()``:
    N=64, m=2, R=100 realizations, static tunnelling noise (+-0.1), Taylor-4,
    dt=0.02, 1500 steps, post_rate=10 (150 snapshots), default observables
    (populations, position, purity, participation ratio), dense-rho path."""
    space = JointSpace(lattice=build_lattice([64]), m=2)
    cfg = RunConfig(
        space=space,
        noise=NoiseSpec(target="tunneling", levels=(-0.1, 0.1), rate=0.0),
        stepper=StepperConfig(backend="taylor", dt=0.02, taylor_order=4),
        realizations=100, steps=1500, post_rate=10,
        master_seed=1234, workers=int(os.environ.get("GOLDEN_WORKERS", "8")), precision="double",
    )
    sinks = MemorySinks(keep_densities=False)
    report = run(cfg, sinks)
    rows = np.array([r[3] for r in sinks.rows], dtype=np.float64)
    meta = dict(n=64, m=2, R=100, steps=1500, post_rate=10, backend="taylor", order=4, dt=0.02,
                target="tunneling", levels=[-0.1, 0.1], master_seed=1234,
                observables_resolved=list(cfg.observables),
                rows=[(r[0], r[1], r[2]) for r in sinks.rows],
                corrections=report.norm_corrections, norm_events=report.norm_events,
                max_norm_deviation=report.max_norm_deviation, wall_seconds=report.wall_seconds)
    np.savez_compressed(os.path.join(HERE, "config0_run.npz"), meta=json.dumps(meta), rows=rows)


if __name__ == "__main__":
    import sys as _sys

    only = _sys.argv[1:]
    for fn in (noise_fixture, stencil_fixture, segment_fixture, run_fixture, telegraph_fixture, density_fixture,
               lattice_fixture, config0_fixture):
        if not only or fn.__name__ in only:
            fn()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
