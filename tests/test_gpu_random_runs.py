"""Randomised run() sweep (fixed seed): m = 1..3 on rings of random size,
random ensemble sizes, schedules, integrators, couplings and noise targets,
static or telegraph noise.  Every observable row must match the oracle's
restatement of the reference's run() to 1e-10 relative (the north-star bar),
and the norm-correction and switch counts must be equal."""

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from oracle.noise_oracle import TelegraphOracle
from tests.test_gpu_parity import numpy_noise, pkg  # noqa: F401  (pkg: fixture)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

OBS = ("populations", "position_mean_variance", "purity", "participation_ratio", "joint_distribution")


def _runs(count=16, seed=2718):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.choice([1, 2, 2, 3]))
        n = int({1: rng.integers(5, 120), 2: rng.integers(5, 80), 3: rng.integers(4, 12)}[m])
        steps = int(rng.integers(4, 40))
        out.append(dict(m=m, n=n, R=int(rng.integers(1, 12)), steps=steps,
                        post_rate=int(rng.integers(1, steps + 1)),
                        backend=str(rng.choice(["taylor", "rk4"])), dt=round(float(rng.uniform(0.01, 0.05)), 4),
                        target=str(rng.choice(["tunneling", "onsite", "both"])),
                        onsite=round(float(rng.uniform(-0.3, 0.3)), 3), U=round(float(rng.uniform(0, 1)), 3),
                        rate=float(rng.choice([0.0, 0.0, round(float(rng.uniform(0.05, 2.0)), 3)]))))
    return out


CASES = _runs()


@pytest.mark.parametrize("c", CASES, ids=[f"m{c['m']}n{c['n']}R{c['R']}{c['backend']}{c['target']}r{c['rate']}"
                                          for c in CASES])
def test_random_run_matches_oracle(pkg, c):
    p = pkg
    m, n, R = c["m"], c["n"], c["R"]
    obs = OBS if m > 1 else tuple(o for o in OBS if o != "joint_distribution")
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), m),
                      model=p.CouplingModel(onsite_energy=c["onsite"], interaction=c["U"]),
                      noise=p.NoiseSpec(target=c["target"], rate=c["rate"]),
                      stepper=p.StepperConfig(backend=c["backend"], dt=c["dt"]),
                      realizations=R, steps=c["steps"], post_rate=c["post_rate"], precision="double",
                      observables=obs)
    sinks = p.MemorySinks(keep_densities=False)
    report = p.run(cfg, sinks)

    nl = n if c["target"] in ("tunneling", "both") else 0
    ns = n if c["target"] in ("onsite", "both") else 0
    tg = None
    if c["rate"] > 0:
        tg = TelegraphOracle(1234, 0, R, (-0.1, 0.1), nl, ns, c["rate"])
        link = tg.link_values() if nl else None
        site = tg.site_values().copy() if ns else None
    else:
        noise = numpy_noise(1234, 0, R, (-0.1, 0.1), nl + ns)
        link = noise[:, :nl] if nl else None
        site = noise[:, nl:] if ns else None
    st = orc.make_stencil(m, n, c["onsite"], 1.0, c["U"], link=link, site=site, batch=R)
    out, _, totals = orc.run_rows(st, orc.product_state(m, n), R, c["steps"], c["post_rate"], c["dt"],
                                  backend=c["backend"], observables=obs, noise=tg)
    ref = [(t, name, i, v) for t, rr in out for name, i, v in rr]
    assert [r[:3] for r in sinks.rows] == [r[:3] for r in ref]
    np.testing.assert_allclose([r[3] for r in sinks.rows], [r[3] for r in ref], rtol=1e-10, atol=1e-13)
    assert report.norm_corrections == totals.corrections
    if tg is not None:
        assert report.switch_count == int(tg.switches.sum())
